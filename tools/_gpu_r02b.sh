set -x
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench1.json 2> gpurun_out/r02_bench1.err
GS_NO_WARMUP=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --print-units base --csv --log-file gpurun_out/r02_s24_launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --python-ref-seconds 0 > /dev/null 2>&1
python tools/ncu_traffic.py gpurun_out/r02_s24_launches.csv --config "s24 eps=0.5 mu=5" --out gpurun_out/sim_traffic.json | tail -3
cp gpurun_out/sim_traffic.json profiles/sim_traffic.json
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --python-ref-seconds 0 > gpurun_out/r02_bench2.json 2> gpurun_out/r02_bench2.err
timeout 1500 python tools/parity_scale.py ooc --scale 27 --oracle --cfg 0.5:5,0.2:5,0.15:3 > gpurun_out/r02_parity_ooc_s27.jsonl 2> gpurun_out/r02_parity_ooc_s27.err; echo rc=$?
timeout 1200 python tools/parity_scale.py chunglu --logn 26 --samples 1300000000 --wmax 1e6 --cfg 0.5:5,0.2:5,0.15:3 > gpurun_out/r02_parity_chunglu_1.24B.jsonl 2> gpurun_out/r02_parity_chunglu_1.24B.err; echo rc=$?
timeout 1500 python tools/parity_scale.py ooc --scale 28 --cap 8000000000 --cfg 0.5:5,0.2:5 > gpurun_out/r02_parity_ooc_s28.jsonl 2> gpurun_out/r02_parity_ooc_s28.err; echo rc=$?
cat gpurun_out/r02_parity_ooc_s27.jsonl gpurun_out/r02_parity_chunglu_1.24B.jsonl gpurun_out/r02_parity_ooc_s28.jsonl
