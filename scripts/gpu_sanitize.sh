# compute-sanitizer over every kernel instantiation (scripts/sanitize.py); logs under gpurun_out/
CS=/usr/local/cuda/bin/compute-sanitizer
python scripts/sanitize.py --quick mlp_c > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 $CS --tool $tool --kernel-name kns=toast_ --error-exitcode 3 --print-limit 50 python scripts/sanitize.py $SAN_ARGS > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/san_$tool.log
done
