# parity on the final tree (after the cluster / classify / e2e-build changes): s24 eps sweep
# through three input paths, Chung-Lu 77.7M, out of core s24 under 2 GB; full GPU suite
set -x
mkdir -p gpurun_out/par
timeout 1500 python tools/parity_scale.py rmat --scale 24 > gpurun_out/par/r02b_parity_s24.jsonl 2>gpurun_out/par/r02b_parity_s24.err; echo rc=$?
timeout 900 python tools/parity_scale.py chunglu > gpurun_out/par/r02b_parity_chunglu.jsonl 2>gpurun_out/par/r02b_parity_chunglu.err; echo rc=$?
timeout 1200 python tools/parity_scale.py ooc --scale 24 --oracle > gpurun_out/par/r02b_parity_ooc_s24.jsonl 2>gpurun_out/par/r02b_parity_ooc_s24.err; echo rc=$?
grep -c '"identical": true' gpurun_out/par/r02b_parity_*.jsonl; grep -c '"identical": false' gpurun_out/par/r02b_parity_*.jsonl
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/par/pytest_gpu.log 2>&1; tail -3 gpurun_out/par/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
