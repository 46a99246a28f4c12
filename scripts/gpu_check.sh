set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/bench_gpt24.json 2> gpurun_out/bench_gpt24.err; echo "bench rc=$?"
for c in unet gns16 llama80; do python bench.py --config $c --no-search --no-cpu-baseline > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err; done
python bench.py --steps 2 --warmup 1 --no-search --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-search --no-cpu-baseline > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?"
