# throughput per forced K (warps sharing one batch) for each config
for c in ${CONFIGS:-gpt24 unet gns16 llama80}; do for K in 1 2 4; do
  TOAST_FORCE_K=$K python bench.py --config $c --no-search --no-cpu-baseline --no-variants --steps 30 > gpurun_out/k_${c}_$K.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/k_${c}_$K.json').read().strip().splitlines()[-1]);print('$c K=$K', round(d['value']/1e6,1), 'M', d['config']['rollouts_per_step_per_gpu'])"
done; done
