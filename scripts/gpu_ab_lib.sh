# A/B of variant libraries (scripts/build_base.py or kernel_sweep.py) against the working tree's, alternating on one box:
# scripts/gpu_ab_lib.sh "<tag> [<tag> ...]" "configs" reps
VS=$1; CS=${2:-gpt24}; R=${3:-3}
for r in $(seq $R); do for c in $CS; do for L in default $VS; do
  if [ $L = default ]; then LIBV=""; else LIBV=paper_2508_15010_b200/lib/variants/libtoast_$L.so; fi
  TOAST_LIB=$LIBV python bench.py --config $c --no-search --no-cpu-baseline --no-variants --steps 50 > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$c $L', round(d['value']/1e6,1), d['config']['warps_per_batch'], d['config']['blocks_per_sm'])"
done; done; done
