# fresh-tree check: GPU tests, smoke, one bench line
mkdir -p gpurun_out/chk
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/chk/pytest_gpu.log 2>&1; tail -3 gpurun_out/chk/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/chk/bench.json 2> gpurun_out/chk/bench.err; cut -c1-600 gpurun_out/chk/bench.json
