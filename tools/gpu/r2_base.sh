set -x
nproc; free -g | head -2
python bench.py --workload cfg5 --dtype c128 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_base_cfg5_c128.json 2> gpurun_out/r2_base_cfg5_c128.err
python bench.py --workload cfg2 --dtype c128 --batch 8 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_base_cfg2_c128_b8.json 2>&1
CBESSFM_KERNEL=cluster python bench.py --workload cfg2 --dtype c64 --batch 8 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_base_cfg2_c64_b8_cluster.json 2>&1
