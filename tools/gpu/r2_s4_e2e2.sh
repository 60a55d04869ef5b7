# e2e leg: ring size x chunks on one box, next to the box's host link
python tools/exp_copy2.py | tail -1
for cfg in "3 4" "4 4" "6 4" "3 2" "4 2" "6 2" "4 1" "3 4"; do
  set -- $cfg
  a=$(BENCH_E2E_RING=$1 BENCH_E2E_CHUNKS=$2 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2), '%.3g'%d['e2e']['value'])")
  echo "ring=$1 chunks=$2 kernel $a"
done
