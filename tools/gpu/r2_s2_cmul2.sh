# packed FP32 complex products (CB_CMUL2) vs base: c64 precision, parity, A/B; wide-path timing
python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "c64 or headroom" > gpurun_out/cmul2_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/cmul2_tests.log
python tools/c64_errors.py > gpurun_out/cmul2_c64_errors.txt 2>&1; tail -14 gpurun_out/cmul2_c64_errors.txt
for rep in 1 2; do
for lib in libcbessfm_base.so libcbessfm.so; do
  export CBESSFM_LIB=$PWD/paper_2409_14489_b200/$lib
  a=$(python bench.py --workload cfg2 --dtype c64 --steps 10 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],4))")
  b=$(python bench.py --workload cfg2 --dtype c64 --batch 8 --steps 10 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],4))")
  c=$(python bench.py --workload cfg4 --dtype c64 --steps 10 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],4))")
  echo "rep$rep $lib cfg2_c64 $a | cfg2_b8_c64 $b | cfg4_c64 $c"
done; done
unset CBESSFM_LIB
timeout 600 python tools/bench_wide.py > gpurun_out/wide_bench.jsonl 2> gpurun_out/wide_bench.err; echo "wide bench rc=$?"; cat gpurun_out/wide_bench.jsonl; tail -3 gpurun_out/wide_bench.err
