mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "persistent or golden_parity" > gpurun_out/p_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/p_tests.log
for rep in 1 2 3; do
for pair in 0 ""; do
  if [ -z "$pair" ]; then unset CBESSFM_PAIR; else export CBESSFM_PAIR=$pair; fi
  a=$(python bench.py --steps 4 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],2), d['kernel']['plan'])")
  b=$(python bench.py --workload cfg2 --batch 8 --steps 10 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],3))")
  echo "rep$rep pair=${pair:-default} cfg5_c128 $a | cfg2x8_c128 $b"
done; done
unset CBESSFM_PAIR
DIAG_REPS=6 python tools/gpu/diag_persist.py > gpurun_out/diag_persist.log 2>&1; echo "diag rc=$?"; grep -c "persistent.* 0 differing samples" gpurun_out/diag_persist.log; grep "differing" gpurun_out/diag_persist.log | grep -v " 0 differing" | head -5
