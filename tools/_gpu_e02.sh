# launch list of one s24 eps 0.2 step (per-kernel time + DRAM bytes)
mkdir -p gpurun_out/e02
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --python-ref-seconds 0 --eps 0.2"
GS_NO_WARMUP=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --print-units base --csv --log-file gpurun_out/e02/launches.csv $B > gpurun_out/e02/ncu.log 2>&1
tail -2 gpurun_out/e02/ncu.log
