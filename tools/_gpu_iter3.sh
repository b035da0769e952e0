# b-list cluster passes: variants + parity tests; eps 0.2 / 0.15 A/B
mkdir -p gpurun_out/it3
timeout 1500 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_phases.py tests/test_gpu_build.py -m gpu -x -q 2>&1 | tail -4
r() { tag=$1; shift; env "$@" timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --python-ref-seconds 0 $ARGS > gpurun_out/it3/$tag.json 2> gpurun_out/it3/$tag.err
  python - "$tag" <<'PY'
import json, sys
t = sys.argv[1]
try:
    d = json.loads(open(f'gpurun_out/it3/{t}.json').read().strip().splitlines()[-1])
except Exception as ex:
    print(t, 'FAILED', ex); print(open(f'gpurun_out/it3/{t}.err').read()[-1500:]); sys.exit()
e = d.get('e2e') or {}
print(t, 'step', round(d['ms_per_step'], 2), 'e2e', round(e.get('ms_per_step', 0), 2), {k: round(v, 2) for k, v in d['phases_ms'].items()})
PY
}
ARGS="--eps 0.2 --no-e2e"
r e02_list GS_X=1
r e02_nolist GS_CLUSTER_LIST=0
r e02_list2 GS_X=1
ARGS="--eps 0.15 --mu 3 --no-e2e"
r e015_list GS_X=1
r e015_nolist GS_CLUSTER_LIST=0
ARGS="--eps 0.25 --mu 3 --no-e2e"
r e025_list GS_X=1
ARGS=""
r e05 GS_X=1
