# sketch build: four loads in flight per lane (GS_SK_UNROLL=4) A/B, prep ms
for u in 1 4 1 4; do
  GS_SK_UNROLL=$u timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --python-ref-seconds 0 --no-e2e > /tmp/sk.json 2>/dev/null
  python -c "
import json; d=json.loads(open('/tmp/sk.json').read().strip().splitlines()[-1])
k={x['kernel'][:5]: x['ms'] for x in d['roofline']['kernels']}
print('unroll $u step', round(d['ms_per_step'],3), 'prep', k.get('prep:'), 'sketch decided', d['counts']['decided_by_sketch'])"
done
GS_SK_UNROLL=4 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --python-ref-seconds 0 --no-e2e --eps 0.2 > /tmp/sk2.json 2>/dev/null
python -c "
import json; d=json.loads(open('/tmp/sk2.json').read().strip().splitlines()[-1]); print('eps0.2 unroll4 step', round(d['ms_per_step'],2))"
GS_SK_UNROLL=4 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -1
