# c128 evidence: launch list of the default bench (our kernels only), one ncu
# --set full capture of the c128 cluster kernel on a batched configs[1]
# launch, per-phase clocks of the c128 kernel under load
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:cbessfm -c 50 --csv --log-file gpurun_out/s2_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-extras > gpurun_out/s2_ncu_launch.log 2>&1; echo "launch rc=$?"
ncu --set full --clock-control none --import-source on -k regex:cbessfm_block_kernel -s 3 -c 1 -f -o gpurun_out/s2_c128_b8_full python bench.py --profile --workload cfg2 --batch 8 --steps 1 --warmup 3 --no-e2e > gpurun_out/s2_ncu_c128.log 2>&1; echo "ncu full rc=$?"
CBESSFM_LIB=paper_2409_14489_b200/libcbessfm_prof.so python tools/phase_profile.py c128 > gpurun_out/s2_phase_c128.txt 2>&1; echo "phase rc=$?"
cat gpurun_out/s2_phase_c128.txt | tail -30
