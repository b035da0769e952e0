# ncu: full capture of the dominant identify kernels (eps 0.5) + eps 0.2 launch list and full capture
set -x
mkdir -p gpurun_out
export GS_NO_WARMUP=1
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --python-ref-seconds 0"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_sim_hash<512|k_sim_warp' -c 2 -o gpurun_out/r02_s24_eps0.5_sim_full $B > gpurun_out/ncu1.log 2>&1; tail -3 gpurun_out/ncu1.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --print-units base --csv --log-file gpurun_out/r02_s24_eps0.2_launches.csv $B --eps 0.2 > gpurun_out/b02.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_sim_hash<512|k_sim_hash<1024|k_sim_warp' -c 4 -o gpurun_out/r02_s24_eps0.2_sim_full $B --eps 0.2 > gpurun_out/ncu2.log 2>&1; tail -3 gpurun_out/ncu2.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --python-ref-seconds 0 --no-e2e --eps 0.2 > gpurun_out/r02_bench_eps0.2.json 2>gpurun_out/r02_bench_eps0.2.err
timeout 900 python tools/reference_timing.py --scales 12 14 16 --extrapolate 18 > gpurun_out/r02_reference_timing.jsonl 2> gpurun_out/r02_reference_timing.err
cat gpurun_out/r02_reference_timing.jsonl
