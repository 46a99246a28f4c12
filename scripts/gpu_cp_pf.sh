# critical-path rollout throughput vs prefetch distance / cold threshold
python -m pytest tests -m gpu -x -q -k "critical_path or cp" > gpurun_out/pytest_cp.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_cp.log
for PD in 0 3 6 12; do for c in ${CONFIGS:-gpt24 llama80}; do
TOAST_CP_PF_DIST=$PD timeout 300 python bench.py --config $c --cost-model cp --steps 10 --no-search --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('PD=$PD', '$c', '%.1fM'%(d['value']/1e6))"
done; done
TOAST_CP_PF_COLD=4 TOAST_CP_PF_DIST=6 timeout 300 python bench.py --config gpt24 --cost-model cp --steps 10 --no-search --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('cold4 PD=6 gpt24', '%.1fM'%(d['value']/1e6))"
