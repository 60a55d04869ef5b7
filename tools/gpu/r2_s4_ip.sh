mkdir -p gpurun_out
for rep in 1 2; do
for k in "" ip; do
  if [ -z "$k" ]; then unset CBESSFM_KERNEL; else export CBESSFM_KERNEL=$k; fi
  b=$(CBESSFM_PERSIST=0 python bench.py --workload cfg2 --batch 8 --steps 10 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],3), d['kernel']['name'])")
  echo "rep$rep kernel=${k:-cluster} persist=0 cfg2x8_c128 $b"
done; done
CBESSFM_KERNEL=ip ncu --set full --clock-control none --import-source on -k regex:cbessfm_ip_kernel -s 3 -c 1 -f -o gpurun_out/ip_c128_b8_full python bench.py --profile --workload cfg2 --batch 8 --steps 1 --warmup 3 --no-e2e > gpurun_out/ncu_ip.log 2>&1; echo "ncu ip rc=$?"
