# persistent cluster kernel: parity (new bit-identity test + golden + configs), A/B vs one cluster per block
python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "persistent or golden_parity or full_size or block_ranges or run_host or both_block" > gpurun_out/p_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/p_tests.log
python -m pytest tests/test_gpu_configs.py -x -q -p no:cacheprovider -k "config4 or config3_full" > gpurun_out/p_tests2.log 2>&1; echo "tests2 rc=$?"; tail -3 gpurun_out/p_tests2.log
for rep in 1 2; do
for pers in 0 1; do
  if [ $pers = 0 ]; then export CBESSFM_PERSIST=0; else unset CBESSFM_PERSIST; fi
  a=$(python bench.py --steps 4 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],2), '%.3g'%d['value'], d['roofline']['frac'])")
  b=$(python bench.py --workload cfg2 --batch 8 --steps 10 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],3))")
  echo "rep$rep persist=$pers cfg5_c128 $a | cfg2x8_c128 $b"
done; done
