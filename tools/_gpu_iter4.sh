# hub test pushed from the clustered side: tests; eps 0.2 / 0.15 / 0.25 with the listing gate at 2m/64, 2m/4, 2m
mkdir -p gpurun_out/it4
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_phases.py tests/test_gpu_variants.py -m gpu -x -q 2>&1 | tail -3
r() { tag=$1; shift; env "$@" timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --python-ref-seconds 0 $ARGS > gpurun_out/it4/$tag.json 2> gpurun_out/it4/$tag.err
  python - "$tag" <<'PY'
import json, sys
t = sys.argv[1]
try:
    d = json.loads(open(f'gpurun_out/it4/{t}.json').read().strip().splitlines()[-1])
except Exception as ex:
    print(t, 'FAILED', ex); print(open(f'gpurun_out/it4/{t}.err').read()[-1500:]); sys.exit()
print(t, 'step', round(d['ms_per_step'], 2), {k: round(v, 2) for k, v in d['phases_ms'].items()}, d['counts']['hubs'])
PY
}
for cfg in "0.2 5" "0.15 3" "0.25 3"; do
  set -- $cfg
  ARGS="--eps $1 --mu $2 --no-e2e"
  r e$1_div64 GS_LIST_DIV=64
  r e$1_div4 GS_LIST_DIV=4
  r e$1_div1 GS_LIST_DIV=1
done
