python bench.py --workload cfg2 --batch 8 --steps 10 --no-cpu-baseline --no-e2e --no-extras > gpurun_out/r2_ip2_b8.json 2>&1
CBESSFM_KERNEL=cluster python bench.py --workload cfg2 --batch 8 --steps 10 --no-cpu-baseline --no-e2e --no-extras > gpurun_out/r2_ip2_b8_cluster.json 2>&1
for f in gpurun_out/r2_ip2_b8*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['roofline']['frac'], d['kernel']['name'])"; done
ncu --set full --import-source on --clock-control none -k regex:cbessfm_ip_kernel -c 1 -o gpurun_out/ip_b8 python bench.py --workload cfg2 --batch 8 --steps 1 --warmup 1 --profile > gpurun_out/ncu_ip.log 2>&1
CBESSFM_KERNEL=cluster ncu --set full --import-source on --clock-control none -k regex:cbessfm_block_kernel -c 1 -o gpurun_out/cl_b8 python bench.py --workload cfg2 --batch 8 --steps 1 --warmup 1 --profile > gpurun_out/ncu_cl.log 2>&1
ls -la gpurun_out/*.ncu-rep
