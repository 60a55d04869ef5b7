# in-place-pass c128 kernel: parity first, then the bench A/B vs the cluster kernel
python -m pytest tests/test_gpu_parity.py -x -q -k "golden_parity and c128" > gpurun_out/r2_ip_golden.log 2>&1; echo "golden rc=$?"; tail -3 gpurun_out/r2_ip_golden.log
python -m pytest tests/test_gpu_configs.py -x -q -k "sweep or full" > gpurun_out/r2_ip_cfg.log 2>&1; echo "cfg rc=$?"; tail -3 gpurun_out/r2_ip_cfg.log
python bench.py --steps 5 --no-cpu-baseline --no-e2e --no-extras > gpurun_out/r2_ip_bench.json 2>&1; echo "bench rc=$?"
CBESSFM_KERNEL=cluster python bench.py --steps 5 --no-cpu-baseline --no-e2e --no-extras > gpurun_out/r2_ip_bench_cluster.json 2>&1
python bench.py --workload cfg2 --steps 20 --no-cpu-baseline --no-e2e --no-extras > gpurun_out/r2_ip_bench_cfg2.json 2>&1
for f in gpurun_out/r2_ip_bench*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['roofline']['frac'], d['kernel']['name'])"; done
