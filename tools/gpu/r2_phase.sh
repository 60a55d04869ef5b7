export CBESSFM_LIB=paper_2409_14489_b200/libcbessfm_prof.so
python tools/phase_profile.py c128 > gpurun_out/phase_c128_ip.txt 2>&1
CBESSFM_KERNEL=cluster python tools/phase_profile.py c128 > gpurun_out/phase_c128_cluster.txt 2>&1
cat gpurun_out/phase_c128_ip.txt gpurun_out/phase_c128_cluster.txt
