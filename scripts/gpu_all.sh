# every config: the main rollout line and the critical-path line (no search / CPU legs)
for c in gpt24 unet gns16 llama80; do for cm in sum cp; do
timeout 300 python bench.py --config $c --cost-model $cm --no-search --no-cpu-baseline --no-variants > gpurun_out/bench_${cm}_$c.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/bench_${cm}_$c.json').read().strip().splitlines()[-1]); print('$c $cm', '%.1fM'%(d['value']/1e6), 'e2e %.1fM'%(d['e2e']['value']/1e6), 'full %.1fM'%(d['e2e']['full_records']['value']/1e6), 'K', d['config']['warps_per_batch'], 'B', d['config'].get('blocks_per_sm'), 'ms', round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],4))"
done; done
