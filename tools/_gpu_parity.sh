set -x
nproc; free -g | head -2
python tools/parity_scale.py rmat --scale 16 --cfg 0.2:5,0.5:5 2>&1 | tail -5
timeout 1500 python tools/parity_scale.py rmat --scale 24 > gpurun_out/r02_parity_s24.jsonl 2>gpurun_out/r02_parity_s24.err; echo rc=$?
timeout 900 python tools/parity_scale.py chunglu > gpurun_out/r02_parity_chunglu.jsonl 2>gpurun_out/r02_parity_chunglu.err; echo rc=$?
timeout 1200 python tools/parity_scale.py ooc --scale 24 --oracle > gpurun_out/r02_parity_ooc_s24.jsonl 2>gpurun_out/r02_parity_ooc_s24.err; echo rc=$?
cat gpurun_out/r02_parity_*.jsonl
