# parity on the current tree at BASELINE scale + the reference's own CPU path timed on this host
set -x
nproc; free -g | head -2
mkdir -p gpurun_out
timeout 1500 python tools/parity_scale.py rmat --scale 24 > gpurun_out/r02_parity_s24.jsonl 2>gpurun_out/r02_parity_s24.err; echo rc=$?
timeout 900 python tools/parity_scale.py chunglu > gpurun_out/r02_parity_chunglu.jsonl 2>gpurun_out/r02_parity_chunglu.err; echo rc=$?
timeout 900 python tools/reference_timing.py --scales 12 14 16 --extrapolate 20 > gpurun_out/r02_reference_timing.jsonl 2> gpurun_out/r02_reference_timing.err; echo rc=$?
cat gpurun_out/r02_parity_s24.jsonl gpurun_out/r02_parity_chunglu.jsonl gpurun_out/r02_reference_timing.jsonl
tail -3 gpurun_out/r02_reference_timing.err
