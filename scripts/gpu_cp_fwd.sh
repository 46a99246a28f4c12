python -m pytest tests -m gpu -x -q -k "critical_path or cp" > gpurun_out/pytest_cp.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_cp.log
for F in 1 0; do for c in gpt24 unet gns16 llama80; do
TOAST_CP_FWD=$F timeout 300 python bench.py --config $c --cost-model cp --steps 10 --no-search --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('FWD=$F', '$c', '%.1fM'%(d['value']/1e6))"
done; done
