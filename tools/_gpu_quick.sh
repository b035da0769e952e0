# quick bench: identify per-class times (tools/_gpu_quick.sh [extra bench args])
for v in 4 3; do
GS_WARP_MINB=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --python-ref-seconds 0 --no-e2e "$@" > gpurun_out/q_$v.json 2> gpurun_out/q_$v.err
python - <<PY
import json
d=json.load(open('gpurun_out/q_$v.json'))
print('MINB=$v', round(d['ms_per_step'],2), 'identify', round(d['phases_ms']['identify'],2), 'build', d['phases_ms']['build'])
for k in d['roofline']['kernels']: print('  ', k['kernel'][:40], k['ms'], round(k['bytes']/1e9,2), round(k['frac'] or 0,3))
PY
done
