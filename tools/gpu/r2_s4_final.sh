# round-2 final evidence set at HEAD: GPU suite, smoke, default bench, reference arm, c64 line,
# launch list, one ncu --set full capture of the c128 cluster kernel, DRAM traffic per launch,
# determinism of the persistent launch
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/final_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/final_smoke.log
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err; echo "ref rc=$?"
python bench.py --dtype c64 --no-cpu-baseline > gpurun_out/final_bench_c64.json 2> gpurun_out/final_bench_c64.err; echo "c64 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:cbessfm -c 50 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-extras > gpurun_out/final_ncu_launch.log 2>&1; echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:cbessfm_block_kernel -s 3 -c 1 -f -o gpurun_out/final_c128_b8_full python bench.py --profile --workload cfg2 --batch 8 --steps 1 --warmup 3 --no-e2e > gpurun_out/final_ncu_c128.log 2>&1; echo "ncu full rc=$?"
for dt in c128 c64; do
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"cbessfm_(block|fat)_kernel" -s 3 -c 1 --csv --log-file gpurun_out/final_traffic_cfg5_$dt.csv python bench.py --profile --dtype $dt --steps 1 --warmup 3 > gpurun_out/final_traffic_$dt.log 2>&1; echo "$dt traffic rc=$?"
tail -3 gpurun_out/final_traffic_cfg5_$dt.csv
done
DIAG_REPS=16 python tools/gpu/diag_persist.py > gpurun_out/diag_persist.log 2>&1; echo "diag rc=$?"; grep -c "persistent.* 0 differing samples" gpurun_out/diag_persist.log
python tools/exp_copy2.py > gpurun_out/copy2.log 2>&1; tail -2 gpurun_out/copy2.log
