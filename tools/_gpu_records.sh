# round-2 records on the current tree: bench line, reference arm, launch list + traffic,
# eps sweep, ncu --set full of the dominant kernel, sharded phase path, Chung-Lu, s28
set -x
mkdir -p gpurun_out/rec
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
export B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --python-ref-seconds 0"
GS_NO_WARMUP=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --print-units base --csv --log-file gpurun_out/rec/launches_s24_eps0.5.csv $B > /dev/null 2>&1
python tools/ncu_traffic.py gpurun_out/rec/launches_s24_eps0.5.csv --config "s24 eps=0.5 mu=5" --out gpurun_out/rec/sim_traffic.json > /dev/null
cp gpurun_out/rec/sim_traffic.json profiles/sim_traffic.json
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/rec/bench_s24.json 2> gpurun_out/rec/bench_s24.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/rec/reference_s24.json 2> gpurun_out/rec/reference_s24.err
for e in 0.2 0.25 0.3 0.35 0.4 0.5 0.6 0.7 0.8; do timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --python-ref-seconds 0 --no-e2e --eps $e > gpurun_out/rec/eps_$e.json 2>/dev/null; done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --python-ref-seconds 0 --no-e2e --eps 0.25 --mu 3 > gpurun_out/rec/eps_0.25_mu3.json 2>/dev/null
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --python-ref-seconds 0 --no-e2e --eps 0.15 --mu 3 > gpurun_out/rec/eps_0.15_mu3.json 2>/dev/null
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --python-ref-seconds 0 --sharded > gpurun_out/rec/sharded_s24.json 2> gpurun_out/rec/sharded_s24.err
GS_NO_WARMUP=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sk_filter|k_fused_warp" -c 2 -o gpurun_out/rec/s24_eps0.5_full $B > /dev/null 2>&1
timeout 900 python tools/chunglu_bench.py --steps 3 > gpurun_out/rec/chunglu.json 2> gpurun_out/rec/chunglu.err
timeout 900 python bench.py --scale 28 --steps 2 --warmup 3 --no-cpu-baseline --python-ref-seconds 0 --no-e2e > gpurun_out/rec/s28.json 2> gpurun_out/rec/s28.err
ls -la gpurun_out/rec
