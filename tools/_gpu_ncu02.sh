# ncu --set full of the stage-1 filter at eps 0.2 (k = 8 rows)
mkdir -p gpurun_out/n02
GS_NO_WARMUP=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sk_filter" -c 1 -o gpurun_out/n02/filter_e02 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --python-ref-seconds 0 --eps 0.2 > gpurun_out/n02/ncu.log 2>&1
tail -2 gpurun_out/n02/ncu.log
