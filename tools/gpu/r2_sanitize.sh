# compute-sanitizer, one tool per call: bash tools/gpu/r2_sanitize.sh racecheck
tool=$1
mkdir -p gpurun_out/sanitize
for c in fat cluster64 cluster128 cluster9 ip nlpr ssfm rx coeff; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py $c \
    > gpurun_out/sanitize/${tool}_$c.log 2>&1
  echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|finite=' gpurun_out/sanitize/${tool}_$c.log | tr '\n' ' ')"
done
