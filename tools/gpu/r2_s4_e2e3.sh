python tools/exp_copy2.py | tail -1
for cfg in "4 1 4" "4 1 10" "3 4 10" "4 1 10" "6 2 10" "4 1 20"; do
  set -- $cfg
  a=$(BENCH_E2E_RING=$1 BENCH_E2E_CHUNKS=$2 python bench.py --steps $3 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2), '%.3g'%d['e2e']['value'])")
  echo "ring=$1 chunks=$2 steps=$3 kernel $a"
done
