# BASELINE-scale parity on the current tree: s27 out of core under 2 GB (with core-producing eps) vs
# in-HBM and the oracle; Chung-Lu 1.24B edges vs the oracle; s28 out of core vs in-HBM
set -x
mkdir -p gpurun_out
timeout 2400 python tools/parity_scale.py ooc --scale 27 --oracle --cfg 0.5:5,0.2:5,0.15:3 > gpurun_out/r02_parity_ooc_s27.jsonl 2> gpurun_out/r02_parity_ooc_s27.err; echo rc=$?
timeout 1800 python tools/parity_scale.py chunglu --logn 26 --samples 1300000000 --wmax 1e6 --cfg 0.5:5,0.2:5,0.15:3 > gpurun_out/r02_parity_chunglu_1.24B.jsonl 2> gpurun_out/r02_parity_chunglu_1.24B.err; echo rc=$?
timeout 2400 python tools/parity_scale.py ooc --scale 28 --cap 8000000000 --cfg 0.5:5,0.2:5 > gpurun_out/r02_parity_ooc_s28.jsonl 2> gpurun_out/r02_parity_ooc_s28.err; echo rc=$?
cat gpurun_out/r02_parity_ooc_s27.jsonl gpurun_out/r02_parity_chunglu_1.24B.jsonl gpurun_out/r02_parity_ooc_s28.jsonl
tail -3 gpurun_out/*.err
