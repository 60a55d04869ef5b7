# timing stubs (wrong results): what the NLPR chain costs inside the c128 step
for rep in 1 2; do
for lib in "" nl1 nl2; do
  if [ -z "$lib" ]; then unset CBESSFM_LIB; else export CBESSFM_LIB=$PWD/paper_2409_14489_b200/libcbessfm_$lib.so; fi
  a=$(python bench.py --steps 4 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],2))")
  echo "rep$rep lib=${lib:-main} cfg5_c128 $a"
done; done
