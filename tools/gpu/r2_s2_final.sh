# round-2 evidence set: GPU suite, smoke, default bench, reference arm, c64 line, launch list
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/final_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/final_smoke.log
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err; echo "ref rc=$?"
python bench.py --dtype c64 --no-cpu-baseline > gpurun_out/final_bench_c64.json 2> gpurun_out/final_bench_c64.err; echo "c64 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:cbessfm -c 50 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-extras > gpurun_out/final_ncu_launch.log 2>&1; echo "launch list rc=$?"
