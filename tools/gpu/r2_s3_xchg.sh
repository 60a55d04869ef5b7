# outer exchange: register form (all remote loads, one barrier, direct writes) vs staged form
python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "persistent or golden_parity or full_size" > gpurun_out/x_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/x_tests.log
CBESSFM_LIB=paper_2409_14489_b200/libcbessfm_prof.so python tools/xchg_marks.py c128 > gpurun_out/x_marks_reg.txt 2>&1
CBESSFM_LIB=paper_2409_14489_b200/libcbessfm_profstaged.so python tools/xchg_marks.py c128 > gpurun_out/x_marks_staged.txt 2>&1
cat gpurun_out/x_marks_reg.txt gpurun_out/x_marks_staged.txt | grep "=="
for rep in 1 2; do
for lib in libcbessfm_staged.so libcbessfm.so; do
  export CBESSFM_LIB=$PWD/paper_2409_14489_b200/$lib
  a=$(python bench.py --steps 4 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],2), '%.3g'%d['value'], d['roofline']['frac'])")
  b=$(python bench.py --workload cfg2 --batch 8 --steps 10 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],3))")
  echo "rep$rep $lib cfg5_c128 $a | cfg2x8_c128 $b"
done; done
