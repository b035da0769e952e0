timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
GS_WARP_MINB=4 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --python-ref-seconds 0 --no-e2e "$@" > gpurun_out/q.json 2> gpurun_out/q.err
python - <<PY
import json
d=json.load(open('gpurun_out/q.json'))
print(round(d['ms_per_step'],2), 'identify', round(d['phases_ms']['identify'],2), 'build', d['phases_ms']['build'])
for k in d['roofline']['kernels']: print('  ', k['kernel'][:40], k['ms'], round(k['bytes']/1e9,2), round(k['frac'] or 0,3))
PY
