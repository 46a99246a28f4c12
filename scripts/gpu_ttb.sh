# time-to-best (GPU search vs the oracle's search) for the other configs
for c in ${CONFIGS:-unet gns16 llama80}; do
timeout 600 python bench.py --config $c --steps 10 --no-variants > gpurun_out/ttb_$c.json 2>gpurun_out/ttb_$c.err
python -c "
import json;d=json.loads(open('gpurun_out/ttb_$c.json').read().strip().splitlines()[-1]); t=d['time_to_best']
print('$c', 'S*', t['target_score'], 'gpu median', t['gpu_seeds']['median_s'], 'hit', t['gpu_seeds']['hit'], 'cpu', t.get('cpu_oracle'), 'speedup', t.get('speedup_vs_cpu_oracle'), t.get('speedup_lower_bound'), 'cpu_baseline', d['cpu_baseline']['value'])"
done
