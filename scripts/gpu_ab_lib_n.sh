# A/B of a variant library against the default at several step sizes: scripts/gpu_ab_lib_n.sh <variant> "n1 n2" reps
V=$1; NS=${2:-262144}; R=${3:-2}
for r in $(seq $R); do for n in $NS; do for L in default $V; do
  if [ $L = default ]; then LIBV=""; else LIBV=paper_2508_15010_b200/lib/variants/libtoast_$L.so; fi
  TOAST_LIB=$LIBV python bench.py --n $n --no-search --no-cpu-baseline --no-variants --steps 20 > gpurun_out/abn.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/abn.json').read().strip().splitlines()[-1]);print('$L n=$n', round(d['value']/1e6,1), 'e2e', round(d['e2e']['value']/1e6,1))"
done; done; done
