# final records after the CTA-shape change + the GPU suite + s24 parity
set -x
bash tools/_gpu_final_records.sh
mkdir -p gpurun_out/par2
timeout 1500 python tools/parity_scale.py rmat --scale 24 > gpurun_out/par2/r02_parity_s24.jsonl 2>gpurun_out/par2/r02_parity_s24.err; echo rc=$?
grep -c '"identical": true' gpurun_out/par2/r02_parity_s24.jsonl; grep -c '"identical": false' gpurun_out/par2/r02_parity_s24.jsonl
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/par2/pytest_gpu.log 2>&1; tail -3 gpurun_out/par2/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
