# quick probe: launch list of one config-2 run + tail trace
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 12 --csv --log-file gpurun_out/launches.csv python bench.py --profile --steps 2 --warmup 1 > gpurun_out/ncu.log 2>&1
python tools/launches.py gpurun_out/launches.csv
VQHULL_TAIL_TRACE=1 timeout 300 python tools/cfg_time.py square 1e8 2 2>&1 | tail -7
