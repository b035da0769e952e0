# parity on the final tree: s24 eps sweep (three paths), Chung-Lu 77.7M, out of core s24 under 2 GB
set -x
mkdir -p gpurun_out
timeout 1500 python tools/parity_scale.py rmat --scale 24 > gpurun_out/r02_parity_s24.jsonl 2>gpurun_out/r02_parity_s24.err; echo rc=$?
timeout 900 python tools/parity_scale.py chunglu > gpurun_out/r02_parity_chunglu.jsonl 2>gpurun_out/r02_parity_chunglu.err; echo rc=$?
timeout 1200 python tools/parity_scale.py ooc --scale 24 --oracle > gpurun_out/r02_parity_ooc_s24.jsonl 2>gpurun_out/r02_parity_ooc_s24.err; echo rc=$?
grep -c '"identical": true' gpurun_out/r02_parity_*.jsonl; grep -c '"identical": false' gpurun_out/r02_parity_*.jsonl
