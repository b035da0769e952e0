# stage-1 variants at low eps (existing knob GS_P1_VARIANT): 0 default, 3 two 32-byte steps per check, 5/6 more CTAs
mkdir -p gpurun_out/p1v
for e in 0.2 0.3; do for v in 0 3 5 0 3; do
  GS_P1_VARIANT=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --python-ref-seconds 0 --no-e2e --eps $e > gpurun_out/p1v/e${e}_v$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/p1v/e${e}_v$v.json').read().strip().splitlines()[-1])
k={x['kernel'][:12]: x['ms'] for x in d['roofline']['kernels']}
print('eps $e variant $v step', round(d['ms_per_step'],2), 'filter', k.get('k_sk_filter '))"
done; done
