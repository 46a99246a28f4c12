for rep in 1 2; do for L in paper_2508_15010_b200/lib/libtoast.so paper_2508_15010_b200/lib/libtoast_loc.so; do for PD in 6 0; do for c in gpt24 unet; do
TOAST_LIB=$L TOAST_CP_PF_DIST=$PD timeout 300 python bench.py --config $c --cost-model cp --steps 10 --no-search --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('$L'.split('/')[-1], 'PD=$PD', '$c', '%.1fM'%(d['value']/1e6))"
done; done; done; done
