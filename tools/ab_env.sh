#!/bin/bash
# A/B of environment settings on the bench workload:
#   tools/ab_env.sh "1 8" "" "CBESSFM_KERNEL=cluster" ...
# prints ms/step per (setting, batch), twice.
batches=$1; shift
for rep in 1 2; do
  for setting in "$@"; do
    for b in $batches; do
      ms=$(env $setting python bench.py --no-cpu-baseline --no-e2e --batch $b ${BENCH_ARGS} 2>/dev/null | tail -1 | python -c "import json,sys; print(round(json.load(sys.stdin)['ms_per_step'],4))")
      echo "rep$rep ${setting:-default} batch=$b ms=$ms"
    done
  done
done
