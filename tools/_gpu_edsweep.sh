for rep in 1 2; do
for spec in "0|GS_EDGE_BUCKETS=0" "24pb|GS_EDGE_BSHIFT=24" "25pb|GS_EDGE_BSHIFT=25" "24sw|GS_EDGE_BSHIFT=24 GS_EDGE_PERBUCKET=0" "23pb|GS_EDGE_BSHIFT=23"; do
  tag=${spec%%|*}; ev=${spec#*|}
  env $ev timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --python-ref-seconds 0 --no-e2e > gpurun_out/eb_$tag.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/eb_$tag.json')); print('$tag', d['build_from_edges_ms'], d['ms_per_step'])"
done
done
