# dedup + checked parity tests, then rollout throughput with and without dedup (sum and critical path)
python -m pytest tests/test_gpu_parity.py -x -q -k "dedup or checked or search" > gpurun_out/pytest_dedup.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_dedup.log
for c in ${CONFIGS:-gpt24 unet gns16 llama80}; do for cm in sum cp; do for dd in 0 1; do
  timeout 300 python bench.py --config $c --cost-model $cm --dedup $dd --no-search --no-cpu-baseline --no-variants --steps 20 > gpurun_out/d_${c}_${cm}_$dd.json 2>gpurun_out/d_${c}_${cm}_$dd.err
  python -c "import json;d=json.loads(open('gpurun_out/d_${c}_${cm}_$dd.json').read().strip().splitlines()[-1]);print('$c $cm dedup=$dd', round(d['value']/1e6,1), 'M', 'ms', round(d['ms_per_step'],4))" || tail -3 gpurun_out/d_${c}_${cm}_$dd.err
done; done; done
