# ncu --set full of the critical-path kernels (one config), source-level: the one-kernel path (--dedup 0,
# the rollout kernel's CP instantiation) and the dedup pipeline's back kernel (the default under this model)
C=${1:-gpt24}
for DD in 0 1; do
  CMD="python bench.py --config $C --cost-model cp --dedup $DD --steps 3 --warmup 3 --no-search --no-cpu-baseline --no-variants"
  $CMD > gpurun_out/plain_cp${DD}_$C.log 2>&1 || { echo "bench rc=$?"; continue; }
  export TOAST_FORCE_K=$(python -c "import json;print(json.loads(open('gpurun_out/plain_cp${DD}_$C.log').read().strip().splitlines()[-1])['config']['warps_per_batch'])")
  if [ $DD = 0 ]; then KR=regex:rollout; OUT=prof_cp_$C; else KR=regex:dedup_back; OUT=prof_cpdd_$C; fi
  ncu --set full --clock-control none --import-source on -k $KR -s 3 -c 1 -o gpurun_out/$OUT -f $CMD > gpurun_out/ncu_full_cp${DD}_$C.log 2>&1
  echo "ncu dedup=$DD rc=$?"
  unset TOAST_FORCE_K
done
