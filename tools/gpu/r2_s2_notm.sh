# c128: twiddle rows from L2 (CB_NO_TMEM) vs TMEM
python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "golden_parity" > gpurun_out/notm_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/notm_tests.log
for rep in 1 2; do
for lib in libcbessfm.so libcbessfm_notm.so; do
  export CBESSFM_LIB=$PWD/paper_2409_14489_b200/$lib
  a=$(python bench.py --steps 4 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],2), '%.3g'%d['value'], d['kernel']['name'])")
  b=$(python bench.py --workload cfg2 --batch 8 --steps 10 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],4))")
  c=$(python bench.py --workload cfg4 --dtype c128 --steps 5 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],4))")
  echo "rep$rep $lib cfg5_c128 $a | cfg2_b8_c128 $b | cfg4_c128 $c"
done; done
unset CBESSFM_LIB
timeout 600 python tools/bench_wide.py > gpurun_out/wide_bench.jsonl 2> gpurun_out/wide_bench.err; echo "wide bench rc=$?"; cat gpurun_out/wide_bench.jsonl
