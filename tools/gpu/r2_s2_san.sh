# compute-sanitizer availability probe, then memcheck on the small kernel cases
mkdir -p gpurun_out/sanitize
which compute-sanitizer; compute-sanitizer --version 2>&1 | head -3
timeout 120 compute-sanitizer --tool memcheck ./tools/san_probe > gpurun_out/sanitize/probe_memcheck.log 2>&1; echo "probe rc=$?"; tail -5 gpurun_out/sanitize/probe_memcheck.log
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_cases.py fat > gpurun_out/sanitize/memcheck_fat.log 2>&1; echo "fat memcheck rc=$?"; tail -6 gpurun_out/sanitize/memcheck_fat.log
