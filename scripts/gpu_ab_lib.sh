# A/B: two library builds on one box, the main bench line of one config, alternating
C=${C:-llama80}; A=${A:-paper_2508_15010_b200/lib/libtoast.so}; B=${B:-paper_2508_15010_b200/lib/libtoast_na3.so}
for rep in 1 2 3; do for L in $A $B; do
  TOAST_LIB=$L timeout 300 python bench.py --config $C --no-search --no-cpu-baseline --no-variants > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$L'.split('/')[-1], '$C', round(d['value']/1e6,1), 'K', d['config']['warps_per_batch'], d['config']['wave'])"
done; done
