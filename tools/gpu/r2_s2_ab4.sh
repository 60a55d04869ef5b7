# warp-uniform small-angle sincos (no reduction) vs HEAD: parity, A/B both dtypes
python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -p no:cacheprovider > gpurun_out/ab4_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/ab4_tests.log
for rep in 1 2; do
for lib in libcbessfm_head.so libcbessfm.so; do
  export CBESSFM_LIB=$PWD/paper_2409_14489_b200/$lib
  a=$(python bench.py --steps 4 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],2), '%.3g'%d['value'])")
  b=$(python bench.py --dtype c64 --steps 4 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],2), '%.3g'%d['value'])")
  echo "rep$rep $lib cfg5_c128 $a | cfg5_c64 $b"
done; done
