# Chung-Lu 1.24 B edges on the final tree: parity (three input paths) at eps 0.5 / 0.2 / 0.15 and the timing record
set -x
mkdir -p gpurun_out/cl
timeout 2400 python tools/parity_scale.py chunglu --logn 26 --samples 1300000000 --wmax 1e6 --cfg 0.5:5,0.2:5,0.15:3 > gpurun_out/cl/r02_parity_chunglu_1.24B.jsonl 2> gpurun_out/cl/r02_parity_chunglu_1.24B.err; echo rc=$?
timeout 900 python tools/chunglu_bench.py --steps 3 > gpurun_out/cl/chunglu.json 2> gpurun_out/cl/chunglu.err; echo rc=$?
grep -c '"identical": true' gpurun_out/cl/r02_parity_chunglu_1.24B.jsonl; grep -c '"identical": false' gpurun_out/cl/r02_parity_chunglu_1.24B.jsonl
tail -2 gpurun_out/cl/*.err
