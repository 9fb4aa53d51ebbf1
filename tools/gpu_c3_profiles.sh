#!/bin/bash
# Config 3 (circle 1e7) profiles: launch list, then ncu --set full of one wide
# level, one segment-per-CTA level and the finisher launches.
# usage: tools/gpu_c3_profiles.sh TAG
tag=${1:-c3}
set -x
timeout 600 python tools/one_hull.py 3 2 > gpurun_out/${tag}_plain.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
   python tools/one_hull.py 3 > gpurun_out/${tag}_ncu.log 2>&1
python tools/launches.py gpurun_out/${tag}_launches.csv > gpurun_out/${tag}_launches.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:level_tma --launch-skip 6 -c 1 \
   -o gpurun_out/${tag}_level_wide -f python tools/one_hull.py 3 > gpurun_out/${tag}_lw.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:level_tma --launch-skip 13 -c 1 \
   -o gpurun_out/${tag}_level_segcta -f python tools/one_hull.py 3 > gpurun_out/${tag}_ls.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:finisher --launch-skip 12 -c 6 \
   -o gpurun_out/${tag}_finisher -f python tools/one_hull.py 3 > gpurun_out/${tag}_fin.log 2>&1
ls -la gpurun_out/*.ncu-rep
