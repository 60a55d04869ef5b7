# A/B of a library variant against the main build on the c128 headline and the batched configs[1] launch
# usage: VARIANT=name bash tools/gpu/r2_s4_ab.sh
mkdir -p gpurun_out
for rep in 1 2 3; do
for lib in "" "paper_2409_14489_b200/libcbessfm_${VARIANT}.so"; do
  if [ -z "$lib" ]; then unset CBESSFM_LIB; else export CBESSFM_LIB=$PWD/$lib; fi
  a=$(python bench.py --steps 4 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],2))")
  b=$(python bench.py --workload cfg2 --batch 8 --steps 10 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],3))")
  echo "rep$rep lib=${lib:-main} cfg5_c128 $a | cfg2x8_c128 $b"
done; done
