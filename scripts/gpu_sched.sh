# parity, then dynamic vs static batch scheduling (TOAST_STATIC_SCHED) on each config
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-gpt24 llama80 unet gns16}; do for S in dyn static; do
  if [ $S = static ]; then export TOAST_STATIC_SCHED=1; else unset TOAST_STATIC_SCHED; fi
  timeout 300 python bench.py --config $c --no-search --no-cpu-baseline --no-variants --steps 30 > gpurun_out/s_${c}_$S.json 2>gpurun_out/s_${c}_$S.err
  python -c "import json;d=json.loads(open('gpurun_out/s_${c}_$S.json').read().strip().splitlines()[-1]);print('$c $S', round(d['value']/1e6,1), 'M K', d['config']['warps_per_batch'], 'blocks', d['config']['blocks_per_sm'], 'ms', round(d['ms_per_step'],4), 'n', d['config']['rollouts_per_step_per_gpu'])"
done; done
unset TOAST_STATIC_SCHED
bash scripts/gpu_ncu.sh gpt24
