# c128 cluster kernel: per-cluster timeline at batch 16 (2288 clusters): concurrency, gaps
export CBESSFM_LIB=paper_2409_14489_b200/libcbessfm_prof.so
python tools/timeline.py c128 16 > gpurun_out/tl_c128_b16.txt 2>&1
python tools/timeline.py c128 1 > gpurun_out/tl_c128_b1.txt 2>&1
unset CBESSFM_LIB
python - > gpurun_out/tl_occ.txt 2>&1 <<'PY'
import torch, paper_2409_14489_b200 as pb, bench
bench.WL = bench.WORKLOADS["cfg2"]
cfg, coeffs = bench.workload_cfg()
for dt in ("c128", "c64"):
    eng = pb.DbpEngine(cfg, coeffs, bench.RATE, dtype=dt)
    i = eng.plan.info(); print(dt, {f: getattr(i, f) for f, _ in i._fields_})
PY
tail -30 gpurun_out/tl_c128_b16.txt gpurun_out/tl_c128_b1.txt gpurun_out/tl_occ.txt
