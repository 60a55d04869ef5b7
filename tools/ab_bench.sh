#!/bin/bash
# A/B of library variants on the bench workload: tools/ab_bench.sh "1 8" lib1 lib2 ...
# (lib "" = the default libcbessfm.so); prints ms/step per (lib, batch), twice.
batches=$1; shift
for rep in 1 2; do
  for lib in "$@"; do
    for b in $batches; do
      if [ -n "$lib" ]; then export CBESSFM_LIB=$PWD/paper_2409_14489_b200/$lib; else unset CBESSFM_LIB; fi
      ms=$(python bench.py --no-cpu-baseline --no-e2e --no-extras --batch $b ${BENCH_ARGS} 2>/dev/null | tail -1 | python -c "import json,sys; print(round(json.load(sys.stdin)['ms_per_step'],4))")
      echo "rep$rep ${lib:-default} batch=$b ms=$ms"
    done
  done
done
