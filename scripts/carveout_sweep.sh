for cv in -1 100 90 80 70 60 50; do
  TOAST_CARVEOUT=$cv TOAST_LIB=paper_2508_15010_b200/lib/ab/libtoast_new.so python bench.py --config gpt24 --no-search --no-cpu-baseline --no-variants > gpurun_out/cv.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/cv.json').read().strip().splitlines()[-1]);print('cv $cv', round(d['value']/1e6,1), d['config']['warps_per_batch'], d['config']['wave'], round(d['ms_per_step'],4))"
done
