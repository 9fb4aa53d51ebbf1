# dev cycle: parity subset, tail trace, launch list
timeout 900 python -m pytest tests -q -x -m "gpu and not slow" 2>&1 | tail -3
VQHULL_TAIL_TRACE=1 timeout 300 python tools/cfg_time.py square 1e8 2 2>&1 | tail -8
timeout 100 python tools/cfg_time.py disk 1e3 1 2>&1 | tail -1
for c in "disk 1e6 1" "disk 1e8 5" "circle 1e7 3" "kuzmin 1e9 4"; do timeout 300 python tools/cfg_time.py $c 2>&1 | tail -1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 8 --csv --log-file gpurun_out/launches.csv python bench.py --profile --steps 2 --warmup 1 > gpurun_out/ncu.log 2>&1
python tools/launches.py gpurun_out/launches.csv
