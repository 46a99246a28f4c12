# A/B of two library builds on the critical-path bench lines
A=${A:-paper_2508_15010_b200/lib/libtoast.so}; B=${B:-paper_2508_15010_b200/lib/libtoast_cp64.so}
for rep in 1 2; do for L in $A $B; do for c in ${CONFIGS:-gpt24 unet gns16 llama80}; do
  TOAST_LIB=$L timeout 300 python bench.py --config $c --cost-model cp --steps 10 --no-search --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$L'.split('/')[-1], '$c', round(d['value']/1e6,1), 'K', d['config']['warps_per_batch'], 'B', d['config']['blocks_per_sm'])"
done; done; done
