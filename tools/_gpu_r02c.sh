# round 2 baseline on the current tree: smoke, GPU tests, bench, reference arm, launch list + traffic
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench1.json 2> gpurun_out/r02_bench1.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02_ref.json 2> gpurun_out/r02_ref.err
GS_NO_WARMUP=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --print-units base --csv --log-file gpurun_out/r02_s24_launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --python-ref-seconds 0 > /dev/null 2>&1
python tools/ncu_traffic.py gpurun_out/r02_s24_launches.csv --config "s24 eps=0.5 mu=5" --out gpurun_out/sim_traffic.json | tail -8
cp gpurun_out/sim_traffic.json profiles/sim_traffic.json
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --python-ref-seconds 0 > gpurun_out/r02_bench2.json 2> gpurun_out/r02_bench2.err
tail -c 3000 gpurun_out/r02_bench1.json; tail -3 gpurun_out/r02_bench1.err
