# e2e (C-ABI host-buffer path) chunk sweep on the default configs[4] c128 workload
for ch in 4 3 2 4 3; do
  a=$(BENCH_E2E_CHUNKS=$ch python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2), '%.3g'%d['e2e']['value'])")
  echo "chunks=$ch kernel $a"
done
