timeout 900 ncu --set full --import-source on --clock-control none -k regex:"poly_sample|root_filter_tma|tail_kernel" -c 3 -o gpurun_out/full python bench.py --profile --steps 1 --warmup 0 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
