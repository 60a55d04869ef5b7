# A/B: L2 prefetch of the next block's window in the persistent cluster kernel
mkdir -p gpurun_out
for rep in 1 2 3; do
for lib in "" "paper_2409_14489_b200/libcbessfm_pf.so"; do
  if [ -z "$lib" ]; then unset CBESSFM_LIB; else export CBESSFM_LIB=$PWD/$lib; fi
  a=$(python bench.py --steps 4 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],2))")
  b=$(python bench.py --workload cfg2 --batch 8 --steps 10 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],3))")
  echo "rep$rep lib=${lib:-main} cfg5_c128 $a | cfg2x8_c128 $b"
done; done
