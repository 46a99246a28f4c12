# critical-path lines with the measured K/residency vs the occupancy heuristic (TOAST_CP_NO_AUTOTUNE=1)
for T in 0 1; do for c in gpt24 unet gns16 llama80; do
if [ $T = 1 ]; then export TOAST_CP_NO_AUTOTUNE=1; else unset TOAST_CP_NO_AUTOTUNE; fi
timeout 300 python bench.py --config $c --cost-model cp --steps 10 --no-search --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('heuristic' if $T else 'measured', '$c', '%.1fM'%(d['value']/1e6), 'K', d['config']['warps_per_batch'], 'B', d['config']['blocks_per_sm'], 'nda %.2fs'%d['nda_s'])"
done; done
