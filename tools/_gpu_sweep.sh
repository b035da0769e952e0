# bench sweep: each argument "tag|ENV=V ENV2=V|bench args" -> one quick bench line summary
mkdir -p gpurun_out
for spec in "$@"; do
  tag=$(echo "$spec" | cut -d'|' -f1); envs=$(echo "$spec" | cut -d'|' -f2); args=$(echo "$spec" | cut -d'|' -f3)
  env $envs timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --python-ref-seconds 0 --no-e2e $args > gpurun_out/s_$tag.json 2> gpurun_out/s_$tag.err
  python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
try:
    d = json.load(open(f'gpurun_out/s_{tag}.json'))
except Exception as ex:
    print(tag, 'FAILED', ex); print(open(f'gpurun_out/s_{tag}.err').read()[-1500:]); sys.exit()
print(tag, 'step', round(d['ms_per_step'], 2), 'identify', round(d['phases_ms']['identify'], 2), 'build', d['phases_ms']['build'], 'cluster', d['phases_ms']['cluster'], 'classify', d['phases_ms']['classify'], 'evals', d['counts']['sim_evals'], 'inters', d['counts']['intersections'], 'probes', d['counts']['adj_probes'])
for k in d['roofline']['kernels']: print('   ', k['kernel'][:44].ljust(44), k['ms'], round(k['bytes']/1e9, 2), round(k['frac'] or 0, 3))
PY
done
