# parity suite on the default build, then every variant library of scripts/kernel_sweep.py on each config
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-gpt24 llama80 unet gns16}; do for L in default ${VARIANTS:-b3 b4 b5 b6}; do
  if [ $L = default ]; then LIBV=""; else LIBV=paper_2508_15010_b200/lib/variants/libtoast_$L.so; fi
  TOAST_LIB=$LIBV timeout 300 python bench.py --config $c --no-search --no-cpu-baseline --no-variants --steps 30 > gpurun_out/v_${c}_$L.json 2>gpurun_out/v_${c}_$L.err
  python -c "import json;d=json.loads(open('gpurun_out/v_${c}_$L.json').read().strip().splitlines()[-1]);print('$c $L', round(d['value']/1e6,1), 'M K', d['config']['warps_per_batch'], 'blocks', d['config']['blocks_per_sm'], 'ms', round(d['ms_per_step'],4))"
done; done
