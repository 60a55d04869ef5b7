# full GPU suite + default bench line
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/full_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/full_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
