mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_checked.py -x -q -p no:cacheprovider > gpurun_out/p_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/p_tests.log
VARIANT=notab bash tools/gpu/r2_s4_ab.sh
for dt in c64; do a=$(python bench.py --dtype c64 --steps 4 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],2))"); echo "c64 cfg5 $a"; done
