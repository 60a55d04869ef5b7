# End-to-end rate (bench e2e leg) vs steps in flight, chunks and block kernel.
for k in ${KERNELS:-cluster fat}; do for inf in ${INFLIGHT:-2 3}; do for ch in ${CHUNKS:-1 2 8}; do
CBESSFM_KERNEL=$k BENCH_E2E_INFLIGHT=$inf BENCH_E2E_CHUNKS=$ch python bench.py --no-cpu-baseline --steps 200 > gpurun_out/b.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/b.json').read().splitlines()[-1]); print('$k inflight $inf chunks $ch', round(d['value']/1e9,3), round(d['e2e']['value']/1e9,3))"
done; done; done
