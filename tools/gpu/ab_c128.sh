# c128 A/B: configs[4] (64 waveforms) and configs[1] batch 8, ip vs cluster kernel
python -m pytest tests/test_gpu_parity.py -x -q -k "golden_parity and c128" 2>&1 | tail -1
for k in ip cluster; do
  if [ $k = cluster ]; then export CBESSFM_KERNEL=cluster; else unset CBESSFM_KERNEL; fi
  python bench.py --steps 5 --no-cpu-baseline --no-e2e --no-extras > gpurun_out/ab_$k.json 2>&1
  python bench.py --workload cfg2 --batch 8 --steps 10 --no-cpu-baseline --no-e2e --no-extras > gpurun_out/ab_${k}_b8.json 2>&1
done
for f in gpurun_out/ab_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', '%.4g'%d['value'], '%.4f'%d['ms_per_step'], '%.4f'%d['roofline']['frac'], d['kernel']['name'])"; done
