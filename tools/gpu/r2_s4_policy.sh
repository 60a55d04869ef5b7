# cluster scheduling policy preference (default / spread / load balancing) on the c128 headline
for rep in 1 2; do
for pol in 0 1 2; do
  a=$(CBESSFM_CLUSTER_POLICY=$pol python bench.py --steps 4 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],2))")
  b=$(CBESSFM_CLUSTER_POLICY=$pol python bench.py --workload cfg2 --batch 1 --steps 20 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],4))")
  echo "rep$rep policy=$pol cfg5_c128 $a | cfg2x1_c128 $b"
done; done
