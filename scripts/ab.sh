# A/B two library builds on the same box: scripts/ab.sh <config> <libA> <libB>
C=${1:-gpt24}; A=${2}; B=${3}
for rep in 1 2; do for L in $A $B; do
  TOAST_LIB=$L python bench.py --config $C --no-search --no-cpu-baseline --no-variants > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$L'.split('/')[-1], '$C', round(d['value']/1e6,1), d['config']['warps_per_batch'], d['config']['wave'], round(d['ms_per_step'],4))"
done; done
