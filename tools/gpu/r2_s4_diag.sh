# persistent cluster kernel: run-to-run determinism on the configs[4] launch
# (bit for bit against one cluster per block), then the configs[4] parity test
mkdir -p gpurun_out
DIAG_REPS=${DIAG_REPS:-24} python tools/gpu/diag_persist.py > gpurun_out/diag_persist.log 2>&1; echo "diag rc=$?"
grep -c "persistent.* 0 differing samples" gpurun_out/diag_persist.log; grep "differing samples" gpurun_out/diag_persist.log | grep -v " 0 differing" | head
python -m pytest tests/test_gpu_configs.py -x -q -p no:cacheprovider -k "config4" > gpurun_out/p_tests2.log 2>&1; echo "tests2 rc=$?"; tail -3 gpurun_out/p_tests2.log
python -m pytest tests/test_gpu_parity.py tests/test_gpu_checked.py -x -q -p no:cacheprovider > gpurun_out/p_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/p_tests.log
for rep in 1 2; do
  a=$(python bench.py --steps 4 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],2), '%.3g'%d['value'], d['roofline']['frac'])")
  echo "rep$rep cfg5_c128 $a"
done
