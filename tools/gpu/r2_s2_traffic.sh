# DRAM bytes per launch of the bench's dominant kernel (roofline.traffic), both dtypes
for dt in c128 c64; do
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"cbessfm_(block|fat)_kernel" -s 3 -c 1 --csv --log-file gpurun_out/traffic_cfg5_$dt.csv python bench.py --profile --dtype $dt --steps 1 --warmup 3 > gpurun_out/traffic_$dt.log 2>&1; echo "$dt rc=$?"
cat gpurun_out/traffic_cfg5_$dt.csv | tail -4
done
