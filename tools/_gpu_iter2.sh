# tests for the streamed sketch rows + core-list dense cluster passes; e2e and eps 0.2 A/B
mkdir -p gpurun_out/it2
timeout 1200 python -m pytest tests/test_gpu_build.py tests/test_gpu_parity.py tests/test_phases.py tests/test_gpu_variants.py -m gpu -x -q 2>&1 | tail -4
r() { tag=$1; shift; env "$@" timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --python-ref-seconds 0 $ARGS > gpurun_out/it2/$tag.json 2> gpurun_out/it2/$tag.err
  python - "$tag" <<'PY'
import json, sys
t = sys.argv[1]
try:
    d = json.loads(open(f'gpurun_out/it2/{t}.json').read().strip().splitlines()[-1])
except Exception as ex:
    print(t, 'FAILED', ex); print(open(f'gpurun_out/it2/{t}.err').read()[-1500:]); sys.exit()
e = d.get('e2e') or {}
print(t, 'step', round(d['ms_per_step'], 2), 'e2e', round(e.get('ms_per_step', 0), 2), {k: round(v, 2) for k, v in d['phases_ms'].items()})
PY
}
ARGS=""
r e2e_sk1 GS_SK_STREAM=1
r e2e_sk0 GS_SK_STREAM=0
r e2e_sk1b GS_SK_STREAM=1
ARGS="--eps 0.2 --no-e2e"
r e02_new GS_X=1
r e02_old GS_SPARSE_CLUSTER=0
r e02_new2 GS_X=1
ARGS="--eps 0.15 --mu 3 --no-e2e"
r e015_new GS_X=1
r e015_old GS_SPARSE_CLUSTER=0
