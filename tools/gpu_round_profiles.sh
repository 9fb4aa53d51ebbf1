#!/bin/bash
# Round-end profiles: config 2 launch list + ncu --set full of its kernels,
# config 3's wide level, segment-per-CTA level and finisher.  Reports in
# gpurun_out/ (read here with tools/ncu_summary2.py / tools/ncu_lines.py).
set -x
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
   --log-file gpurun_out/r02_c2_launches.csv python bench.py --profile --steps 2 --warmup 1 > gpurun_out/r02_c2_ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none \
   -k regex:"poly_sample|root_filter_tma|cluster_tail" -c 3 -o gpurun_out/r02_c2_full \
   python bench.py --profile --steps 1 --warmup 0 > gpurun_out/r02_c2_full.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:level_tma --launch-skip 3 -c 1 \
   -o gpurun_out/r02_c3_level_wide python tools/one_hull.py 3 > gpurun_out/r02_c3_lw.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:level_tma --launch-skip 13 -c 1 \
   -o gpurun_out/r02_c3_level_segcta python tools/one_hull.py 3 > gpurun_out/r02_c3_ls.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:finisher_all --launch-skip 14 -c 1 \
   -o gpurun_out/r02_c3_finisher python tools/one_hull.py 3 > gpurun_out/r02_c3_fin.log 2>&1
ls -la gpurun_out/*.ncu-rep
