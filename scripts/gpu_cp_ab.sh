# critical-path throughput: two builds (CP min blocks 2 / 3) x bundle widths
for L in paper_2508_15010_b200/lib/libtoast.so paper_2508_15010_b200/lib/libtoast_cp3.so; do for E in 8 6 4; do for c in ${CONFIGS:-gpt24 llama80}; do
TOAST_LIB=$L TOAST_CP_EMAX=$E timeout 300 python bench.py --config $c --cost-model cp --steps 10 --no-search --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('$L'.split('/')[-1], 'E=$E', '$c', '%.1fM'%(d['value']/1e6), 'K', d['config']['warps_per_batch'], 'wave', d['config']['wave'])"
done; done; done
