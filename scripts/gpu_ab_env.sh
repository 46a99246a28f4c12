# A/B of an environment knob on the same box, alternating: scripts/gpu_ab_env.sh VAR "configs" reps
V=$1; CS=${2:-gpt24}; R=${3:-3}
for r in $(seq $R); do for c in $CS; do for on in 0 1; do
  if [ $on = 1 ]; then export $V=1; else unset $V; fi
  python bench.py --config $c --no-search --no-cpu-baseline --no-variants --steps 50 > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$c $V=$on', round(d['value']/1e6,1), d['config']['blocks_per_sm'])"
done; done; done
