# iteration: GPU parity tests, quick bench at eps 0.5 / 0.2 (GS_WARP_MINB 4 and 3), optional ncu
# usage: bash tools/_gpu_iter.sh [ncu-kernel-regex] [ncu-count] [eps]
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_phases.py -m gpu -x -q 2>&1 | tail -2
q() {  # q <tag> <env...> -- bench args
  tag=$1; shift
  env "$@" timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --python-ref-seconds 0 --no-e2e ${EPSARG} > gpurun_out/q_$tag.json 2> gpurun_out/q_$tag.err
  python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
try:
    d = json.load(open(f'gpurun_out/q_{tag}.json'))
except Exception as ex:
    print(tag, 'FAILED', ex); print(open(f'gpurun_out/q_{tag}.err').read()[-2000:]); sys.exit()
print(tag, 'step', round(d['ms_per_step'], 2), 'identify', round(d['phases_ms']['identify'], 2), 'build', d['phases_ms']['build'], 'cluster', d['phases_ms']['cluster'], 'evals', d['counts']['sim_evals'])
for k in d['roofline']['kernels']: print('   ', k['kernel'][:44].ljust(44), k['ms'], round(k['bytes']/1e9, 2), round(k['frac'] or 0, 3))
PY
}
for e in 0.5 0.2; do
  EPSARG="--eps $e"
  q e${e}_minb4 GS_WARP_MINB=4
  q e${e}_minb3 GS_WARP_MINB=3
done
if [ -n "$1" ]; then
  GS_NO_WARMUP=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$1" -c ${2:-3} -o gpurun_out/iter_full python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --python-ref-seconds 0 --eps ${3:-0.5} > gpurun_out/iter_ncu.log 2>&1; tail -2 gpurun_out/iter_ncu.log
fi
