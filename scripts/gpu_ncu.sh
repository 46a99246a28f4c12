# ncu evidence for one config: the launch list of a short bench run and one --set full capture of the rollout kernel.
# The throughput K and residency measured by toast_nda are pinned (TOAST_FORCE_K, TOAST_FORCE_BLOCKS) for the profiled runs: under ncu's replay the
# measurement itself would be distorted.
C=${1:-gpt24}
CMD="python bench.py --config $C --steps 3 --warmup 3 --no-search --no-cpu-baseline --no-variants"
$CMD > gpurun_out/plain_$C.log 2>&1 && \
export TOAST_FORCE_K=$(python -c "import json;print(json.loads(open('gpurun_out/plain_$C.log').read().strip().splitlines()[-1])['config']['warps_per_batch'])") && \
export TOAST_FORCE_BLOCKS=$(python -c "import json;print(json.loads(open('gpurun_out/plain_$C.log').read().strip().splitlines()[-1])['config']['blocks_per_sm'])") && \
$CMD > gpurun_out/plain_forced_$C.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$C.csv $CMD > gpurun_out/ncu_launch_$C.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rollout -s 3 -c 1 -o gpurun_out/prof_$C -f $CMD > gpurun_out/ncu_full_$C.log 2>&1
echo "ncu rc=$?"
