# critical-path rollout throughput vs the L2 budget for finish-slot scratch (TOAST_CP_L2_MB; 0 = no cap)
python -m pytest tests -m gpu -x -q -k "critical_path or cp" > gpurun_out/pytest_cp.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_cp.log
for MB in ${MBS:-0 32 64 96 128}; do for c in ${CONFIGS:-gpt24 llama80}; do
TOAST_CP_L2_MB=$MB timeout 300 python bench.py --config $c --cost-model cp --steps 10 --no-search --no-cpu-baseline > gpurun_out/bench_cp_${c}_$MB.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/bench_cp_${c}_$MB.json').read().strip().splitlines()[-1]); print('$c MB=$MB', '%.1fM'%(d['value']/1e6), 'K', d['config']['warps_per_batch'], 'wave', d['config']['wave'])"
done; done
