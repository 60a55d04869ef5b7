# Round-end measurement set (run under gpurun): bench lines, the ncu launch
# list of the default bench command, and one `ncu --set full` capture per
# block-kernel regime. Summaries: tools/ncu_digest.py, tools/make_profile_summary.py.
set -x
python bench.py > gpurun_out/bench_c64.json 2> gpurun_out/bench_c64.err; tail -1 gpurun_out/bench_c64.json
python bench.py --dtype c128 --no-cpu-baseline > gpurun_out/bench_c128.json 2> gpurun_out/bench_c128.err; tail -1 gpurun_out/bench_c128.json
python bench.py --batch 8 --no-cpu-baseline --no-e2e > gpurun_out/bench_c64_b8.json 2>/dev/null; tail -1 gpurun_out/bench_c64_b8.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
K='regex:cbessfm_(fat|block)_kernel'
ncu --set full --clock-control none --import-source on -k $K -s 3 -c 1 -f -o gpurun_out/c64_full python bench.py --profile --steps 1 --warmup 3 --no-e2e > gpurun_out/ncu_c64.log 2>&1; echo c64=$?
ncu --set full --clock-control none --import-source on -k $K -s 3 -c 1 -f -o gpurun_out/c64_b8_full python bench.py --profile --batch 8 --steps 1 --warmup 3 --no-e2e > gpurun_out/ncu_c64b8.log 2>&1; echo c64b8=$?
ncu --set full --clock-control none --import-source on -k $K -s 3 -c 1 -f -o gpurun_out/c128_full python bench.py --profile --dtype c128 --steps 1 --warmup 3 --no-e2e > gpurun_out/ncu_c128.log 2>&1; echo c128=$?
ls -la gpurun_out
