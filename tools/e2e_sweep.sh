for inf in 2 3; do for ch in 4 8 16; do
BENCH_E2E_INFLIGHT=$inf BENCH_E2E_CHUNKS=$ch python bench.py --no-cpu-baseline --steps 200 > gpurun_out/b.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/b.json').read().splitlines()[-1]); print('inflight $inf chunks $ch', round(d['value']/1e9,3), round(d['e2e']['value']/1e9,3))"
done; done
CBESSFM_KERNEL=fat BENCH_E2E_CHUNKS=16 python bench.py --no-cpu-baseline --steps 200 > gpurun_out/b.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/b.json').read().splitlines()[-1]); print('fat chunks 16', round(d['value']/1e9,3), round(d['e2e']['value']/1e9,3))"
