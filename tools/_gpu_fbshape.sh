# CTA shape of the fused build's CTA classes: build ms A/B
for s in "5 1" "6 1" "5 2" "6 2" "0 0" "5 1" "6 1" "5 2" "6 2"; do
  set -- $s
  GS_FB_SHAPE=$1 GS_FBD_SHAPE=$2 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --python-ref-seconds 0 --no-e2e > /tmp/fb.json 2>/dev/null
  python -c "
import json; d=json.loads(open('/tmp/fb.json').read().strip().splitlines()[-1])
print('shape $1 dyn $2 step', round(d['ms_per_step'],3), 'build', d['phases_ms']['build'])"
done
for s in "6 2" "5 1"; do set -- $s; GS_FB_SHAPE=$1 GS_FBD_SHAPE=$2 python -m pytest tests/test_gpu_build.py -m gpu -q -x -k "device_csr" 2>&1 | tail -1; done
