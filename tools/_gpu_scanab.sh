# survivor-scan step size / speculation A/B (stage 2), eps 0.2 / 0.3 / 0.5
mkdir -p gpurun_out/sab
r() { tag=$1; shift; env "$@" timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --python-ref-seconds 0 $ARGS > gpurun_out/sab/$tag.json 2> gpurun_out/sab/$tag.err
  python - "$tag" <<'PY'
import json, sys
t = sys.argv[1]
try:
    d = json.loads(open(f'gpurun_out/sab/{t}.json').read().strip().splitlines()[-1])
except Exception as ex:
    print(t, 'FAILED', ex); print(open(f'gpurun_out/sab/{t}.err').read()[-1500:]); sys.exit()
k = {x['kernel'][:26]: x['ms'] for x in d['roofline']['kernels']}
print(t, 'step', round(d['ms_per_step'], 2), 'identify', round(d['phases_ms']['identify'], 2), 'cluster', round(d['phases_ms']['cluster'], 2), k)
PY
}
for e in 0.2 0.3 0.5; do
  ARGS="--eps $e --no-e2e"
  r e${e}_base GS_X=1
  r e${e}_u2 GS_SCAN_MINU=2
  r e${e}_spec GS_SCAN_SPEC=1
  r e${e}_u2spec GS_SCAN_MINU=2 GS_SCAN_SPEC=1
  r e${e}_u4 GS_SCAN_MINU=4
done
