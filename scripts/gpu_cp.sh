# critical-path parity tests + the cp variant bench line
python -m pytest tests -m gpu -x -q -k "critical_path or cp" > gpurun_out/pytest_cp.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_cp.log
for c in ${CONFIGS:-gpt24 unet gns16 llama80}; do timeout 300 python bench.py --config $c --cost-model cp --steps 10 --no-search --no-cpu-baseline > gpurun_out/bench_cp_$c.json 2>gpurun_out/bench_cp_$c.err; echo "$c rc=$?"; done
