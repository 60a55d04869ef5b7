# round-2 harness check: new parity tests, bench contract, default bench line
nproc
python -m pytest tests/test_gpu_configs.py -x -q -k "full" > gpurun_out/r2_cfg_full.log 2>&1; echo "cfg_full rc=$?"
python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_contract.py -x -q > gpurun_out/r2_parity_bench.log 2>&1; echo "parity_bench rc=$?"
python bench.py > gpurun_out/r2_bench_default.json 2> gpurun_out/r2_bench_default.err; echo "bench rc=$?"
tail -3 gpurun_out/r2_cfg_full.log gpurun_out/r2_parity_bench.log
