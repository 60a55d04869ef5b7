# throughput of the c128 configs[4] launch vs the number of resident persistent clusters,
# single (5 CTAs, one block) and paired (10 CTAs, two blocks)
for cfg in "0 15" "0 29" "0 44" "0 59" "0 74" "1 7" "1 14" "1 22" "1 29" "1 37"; do
  set -- $cfg
  a=$(CBESSFM_PAIR=$1 CBESSFM_PERSIST=$2 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],2))")
  echo "pair=$1 clusters=$2 ms=$a"
done
