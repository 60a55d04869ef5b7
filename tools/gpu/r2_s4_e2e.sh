# host link of this box, e2e chunk sweep, and the parity suites on the build with the next-window prefetch
mkdir -p gpurun_out
python tools/exp_copy2.py 2>&1 | tee gpurun_out/copy2.log
python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_checked.py -x -q -p no:cacheprovider > gpurun_out/p_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/p_tests.log
for ch in 4 2 8 4; do
  a=$(BENCH_E2E_CHUNKS=$ch python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2), '%.3g'%d['e2e']['value'])")
  echo "chunks=$ch kernel $a"
done
