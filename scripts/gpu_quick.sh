# quick GPU check: parity tests, smoke, bench lines for every config (no search / CPU legs)
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
rm -f gpurun_out/bench*.json
for c in gpt24 unet gns16 llama80; do timeout 300 python bench.py --config $c --no-search --no-cpu-baseline > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err; echo "$c rc=$?"; done
for K in 1 2 4; do for c in ${KCONFIGS:-gpt24 unet}; do TOAST_FORCE_K=$K timeout 300 python bench.py --config $c --no-search --no-cpu-baseline > gpurun_out/benchK${K}_$c.json 2>&1; done; done
