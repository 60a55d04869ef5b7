mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_checked.py -x -q -p no:cacheprovider > gpurun_out/p_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/p_tests.log
for rep in 1 2 3; do
for k in cluster ""; do
  if [ -z "$k" ]; then unset CBESSFM_KERNEL; else export CBESSFM_KERNEL=$k; fi
  a=$(python bench.py --steps 4 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],2), d['kernel']['name'])")
  b=$(python bench.py --workload cfg2 --batch 8 --steps 10 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],3))")
  echo "rep$rep kernel=${k:-default} cfg5_c128 $a | cfg2x8_c128 $b"
done; done
unset CBESSFM_KERNEL
DIAG_REPS=8 python tools/gpu/diag_persist.py > gpurun_out/diag_persist.log 2>&1; echo "diag rc=$?"; grep -c "persistent.* 0 differing samples" gpurun_out/diag_persist.log; grep "differing" gpurun_out/diag_persist.log | grep -v " 0 differing" | head -5
