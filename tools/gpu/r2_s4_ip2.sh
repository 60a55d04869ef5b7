# in-place-pass kernel vs the Stockham cluster kernel at equal features (no rotation table, one cluster per block)
export CBESSFM_LIB=$PWD/paper_2409_14489_b200/libcbessfm_notab.so CBESSFM_PERSIST=0
for rep in 1 2; do
for k in "" ip; do
  if [ -z "$k" ]; then unset CBESSFM_KERNEL; else export CBESSFM_KERNEL=$k; fi
  a=$(python bench.py --steps 3 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],2))")
  b=$(python bench.py --workload cfg2 --batch 8 --steps 10 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],3), d['kernel']['name'])")
  echo "rep$rep kernel=${k:-cluster} cfg5_c128 $a | cfg2x8_c128 $b"
done; done
