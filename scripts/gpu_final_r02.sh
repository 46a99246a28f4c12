# round-2 final evidence: GPU suite, smoke, default bench (all legs), reference arm, ncu captures of every config
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
T0=$(date +%s); python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$? wall $(( $(date +%s) - T0 )) s"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
bash scripts/gpu_ncu_r02.sh > gpurun_out/ncu_r02.log 2>&1; echo "ncu rc=$?"
