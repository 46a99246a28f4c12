# host-buffer pipeline: streams x chunk size (e2e of the main bench line)
for PS in ${PSS:-4 6 8}; do for CD in ${CDS:-2 4 8}; do
TOAST_PIPE_STREAMS=$PS TOAST_PIPE_CHUNK_DIV=$CD timeout 300 python bench.py --config gpt24 --steps 20 --no-search --no-cpu-baseline --no-variants > gpurun_out/ab.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('PS=$PS CD=$CD', '%.1fM'%(d['value']/1e6), 'e2e %.1fM'%(d['e2e']['value']/1e6), 'full %.1fM'%(d['e2e']['full_records']['value']/1e6))"
done; done
