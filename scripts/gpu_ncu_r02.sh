# round-2 ncu evidence: per config a launch list + one --set full capture of the rollout kernel,
# summarised ON the box (profiles/ written there, copied to gpurun_out/profiles_r02/), reports kept only for gpt24
mkdir -p gpurun_out/profiles_r02
for c in ${CONFIGS:-gpt24 unet gns16 llama80}; do
  bash scripts/gpu_ncu.sh $c
  python scripts/ncu_summary.py $c gpurun_out/prof_$c.ncu-rep r02 > /dev/null 2>&1; echo "summary $c rc=$?"
  cp gpurun_out/launches_$c.csv gpurun_out/profiles_r02/r02_launches_$c.csv
  [ $c = gpt24 ] || rm -f gpurun_out/prof_$c.ncu-rep
done
if [ -z "$NO_CP" ]; then
  bash scripts/gpu_ncu_cp.sh gpt24
  python scripts/ncu_summary.py gpt24_cp gpurun_out/prof_cp_gpt24.ncu-rep r02 > /dev/null 2>&1; echo "summary cp rc=$?"
  python scripts/ncu_summary.py gpt24_cp_dedup_back gpurun_out/prof_cpdd_gpt24.ncu-rep r02 > /dev/null 2>&1; echo "summary cp dedup rc=$?"
  rm -f gpurun_out/prof_cp_gpt24.ncu-rep gpurun_out/prof_cpdd_gpt24.ncu-rep
fi
cp profiles/r02_ncu_* profiles/ncu_summary.json gpurun_out/profiles_r02/ 2>/dev/null   # (the launch lists were copied above)
ls -la gpurun_out/profiles_r02
