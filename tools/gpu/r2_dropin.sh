python -m pytest tests/test_gpu_parity.py tests/test_reference_objects.py -x -q > gpurun_out/r2_dropin.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_dropin.log
python tools/time_run_dbp.py > gpurun_out/r2_run_dbp.txt 2>&1; cat gpurun_out/r2_run_dbp.txt | tail -8
