# A/B of a library variant against the main build on the c64 workloads
mkdir -p gpurun_out
for rep in 1 2 3; do
for lib in "" "paper_2409_14489_b200/libcbessfm_${VARIANT}.so"; do
  if [ -z "$lib" ]; then unset CBESSFM_LIB; else export CBESSFM_LIB=$PWD/$lib; fi
  a=$(python bench.py --dtype c64 --steps 4 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],2))")
  b=$(python bench.py --dtype c64 --workload cfg2 --batch 1 --steps 20 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],4))")
  echo "rep$rep lib=${lib:-main} cfg5_c64 $a | cfg2x1_c64 $b"
done; done
