# sketch rows streamed with the host CSR: tests + e2e A/B
mkdir -p gpurun_out/sks
timeout 900 python -m pytest tests/test_gpu_build.py -m gpu -x -q 2>&1 | tail -3
for sk in 1 0 1 0; do
  GS_SK_STREAM=$sk timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --python-ref-seconds 0 > gpurun_out/sks/b_$sk.json 2> gpurun_out/sks/b_$sk.err
  python -c "
import json; d=json.loads(open('gpurun_out/sks/b_$sk.json').read().strip().splitlines()[-1])
print('sk_stream=$sk', 'step', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2), 'edges', round(d['e2e']['from_edge_array']['ms_per_step'],2))" || tail -5 gpurun_out/sks/b_$sk.err
done
