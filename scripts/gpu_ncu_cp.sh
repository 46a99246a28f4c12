# ncu --set full of the critical-path rollout kernel (one config), source-level
C=${1:-gpt24}
CMD="python bench.py --config $C --cost-model cp --steps 3 --warmup 3 --no-search --no-cpu-baseline --no-variants"
$CMD > gpurun_out/plain_cp_$C.log 2>&1 && \
export TOAST_FORCE_K=$(python -c "import json;print(json.loads(open('gpurun_out/plain_cp_$C.log').read().strip().splitlines()[-1])['config']['warps_per_batch'])") && \
ncu --set full --clock-control none --import-source on -k regex:rollout -s 3 -c 1 -o gpurun_out/prof_cp_$C -f $CMD > gpurun_out/ncu_full_cp_$C.log 2>&1
echo "ncu rc=$?"
