# ncu --set full of the in-place-pass c128 kernel on the same batched launch as the cluster capture
CBESSFM_KERNEL=ip python bench.py --workload cfg2 --batch 8 --steps 5 --no-cpu-baseline --no-e2e --no-extras > gpurun_out/ip_b8.json 2>&1; tail -1 gpurun_out/ip_b8.json | cut -c1-200
CBESSFM_KERNEL=ip ncu --set full --clock-control none --import-source on -k regex:cbessfm_ip_kernel -s 3 -c 1 -f -o gpurun_out/s2_ip_b8_full python bench.py --profile --workload cfg2 --batch 8 --steps 1 --warmup 3 --no-e2e > gpurun_out/s2_ncu_ip.log 2>&1; echo "ncu ip rc=$?"
CBESSFM_LIB=$PWD/paper_2409_14489_b200/libcbessfm_notm.so python bench.py --workload cfg2 --batch 8 --steps 3 --no-cpu-baseline --no-e2e --no-extras > gpurun_out/notm_b8.json 2>&1; tail -5 gpurun_out/notm_b8.json
