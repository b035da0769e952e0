# final round-2 records on the frozen tree: launch list + stamped traffic, bench line,
# reference arm, eps sweep, ncu --set full of the dominant kernel
set -x
mkdir -p gpurun_out/fin
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
export B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --python-ref-seconds 0"
GS_NO_WARMUP=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --print-units base --csv --log-file gpurun_out/fin/launches_s24_eps0.5.csv $B > /dev/null 2>&1
python tools/ncu_traffic.py gpurun_out/fin/launches_s24_eps0.5.csv --config "s24 eps=0.5 mu=5" --out gpurun_out/fin/sim_traffic.json
cp gpurun_out/fin/sim_traffic.json profiles/sim_traffic.json
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/fin/bench_s24.json 2> gpurun_out/fin/bench_s24.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin/reference_s24.json 2> gpurun_out/fin/reference_s24.err
for e in 0.2 0.25 0.3 0.35 0.4 0.5 0.6 0.7 0.8; do timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --python-ref-seconds 0 --no-e2e --eps $e > gpurun_out/fin/eps_$e.json 2>/dev/null; done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --python-ref-seconds 0 --no-e2e --eps 0.25 --mu 3 > gpurun_out/fin/eps_0.25_mu3.json 2>/dev/null
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --python-ref-seconds 0 --no-e2e --eps 0.15 --mu 3 > gpurun_out/fin/eps_0.15_mu3.json 2>/dev/null
GS_NO_WARMUP=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sk_filter" -c 1 -o gpurun_out/fin/s24_eps0.5_filter $B > /dev/null 2>&1
GS_NO_WARMUP=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --print-units base --csv --log-file gpurun_out/fin/launches_s24_eps0.2.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --python-ref-seconds 0 --eps 0.2 > /dev/null 2>&1
ls -la gpurun_out/fin
