set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"poly_sample|level_tma|finisher_all|planner" -c 8 -o gpurun_out/tail_full python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_tail.log 2>&1
ls -la gpurun_out
