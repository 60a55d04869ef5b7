mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_checked.py tests/test_gpu_reference_suite.py -x -q -p no:cacheprovider > gpurun_out/p_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/p_tests.log
python tools/c64_errors.py > gpurun_out/errors_tab.txt 2>&1; tail -25 gpurun_out/errors_tab.txt
CBESSFM_LIB=$PWD/paper_2409_14489_b200/libcbessfm_notab.so python tools/c64_errors.py > gpurun_out/errors_notab.txt 2>&1; tail -25 gpurun_out/errors_notab.txt
VARIANT=notab bash tools/gpu/r2_s4_ab.sh
