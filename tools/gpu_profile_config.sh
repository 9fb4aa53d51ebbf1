#!/bin/bash
# Per-kernel picture of one config: bench family times, then the launch list
# of ONE hull (ncu gpu__time_duration, cold-cache serialised launches).
# usage: tools/gpu_profile_config.sh CONFIG TAG
c=${1:-3}; tag=${2:-cfg$c}
set -x
timeout 600 python bench.py --config $c --no-cpu --no-e2e --steps 5 --warmup 3 > gpurun_out/${tag}_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
   python tools/one_hull.py $c > gpurun_out/${tag}_ncu.log 2>&1
python tools/launches.py gpurun_out/${tag}_launches.csv > gpurun_out/${tag}_launches.txt 2>&1
