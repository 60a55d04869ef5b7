mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/final_tests.log
