# round-2 check: full GPU parity suite, smoke, quick bench lines
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
for c in gpt24 llama80; do timeout 300 python bench.py --config $c --no-search --no-cpu-baseline --no-variants --steps 20 > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err; echo "$c rc=$?"; done
