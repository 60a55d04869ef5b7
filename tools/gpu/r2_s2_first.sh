# round 2 (session 2) first box call: GPU suite, default bench, reference arm, launch list
nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/s2_gpu_tests.log 2>&1; echo "gpu tests rc=$?"
tail -5 gpurun_out/s2_gpu_tests.log
python bench.py > gpurun_out/s2_bench_default.json 2> gpurun_out/s2_bench_default.err; echo "bench rc=$?"
cat gpurun_out/s2_bench_default.json
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s2_bench_ref.json 2> gpurun_out/s2_bench_ref.err; echo "ref rc=$?"
cat gpurun_out/s2_bench_ref.json
python bench.py --dtype c64 --no-cpu-baseline > gpurun_out/s2_bench_c64.json 2> gpurun_out/s2_bench_c64.err; echo "c64 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/s2_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s2_ncu_launch.log 2>&1; echo "ncu rc=$?"
