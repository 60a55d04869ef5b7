export CBESSFM_LIB=paper_2409_14489_b200/libcbessfm_prof.so
python tools/timeline.py c128 16 > gpurun_out/tl_c128_ip.txt 2>&1
CBESSFM_KERNEL=cluster python tools/timeline.py c128 16 > gpurun_out/tl_c128_cl.txt 2>&1
tail -4 gpurun_out/tl_c128_ip.txt gpurun_out/tl_c128_cl.txt
