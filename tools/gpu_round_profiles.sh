#!/bin/bash
# Round-end profiles (reports in gpurun_out/, read here with tools/ncu_summary2.py,
# tools/ncu_lines.py, tools/ncu_rep_metrics.py and summarised under profiles/):
#  * config 2: launch list of bench.py (the command the bench line comes from)
#    + ncu --set full of its three kernels;
#  * config 3: launch list of one hull + ncu --set full of one wide level, one
#    segment-per-CTA level and the finisher launches;
#  * disk 1e8: ncu --set full of the filter pass.
# usage: tools/gpu_round_profiles.sh TAG
tag=${1:-r02}
set -x
timeout 600 python bench.py --profile --steps 2 --warmup 1 > gpurun_out/${tag}_c2_plain.log 2>&1 || exit 1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/${tag}_c2_launches.csv python bench.py --profile --steps 2 --warmup 1 > gpurun_out/${tag}_c2_ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none \
   -k regex:"poly_sample|root_filter_tma|cluster_tail" -c 3 -o gpurun_out/${tag}_c2_full -f \
   python bench.py --profile --steps 1 --warmup 0 > gpurun_out/${tag}_c2_full.log 2>&1
timeout 600 python tools/one_hull.py 3 2 > gpurun_out/${tag}_c3_plain.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_c3_launches.csv \
   python tools/one_hull.py 3 > gpurun_out/${tag}_c3_ncu.log 2>&1
python tools/launches.py gpurun_out/${tag}_c3_launches.csv > gpurun_out/${tag}_c3_launches.txt 2>&1
python tools/launches.py gpurun_out/${tag}_c2_launches.csv > gpurun_out/${tag}_c2_launches.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:level_tma --launch-skip 6 -c 1 \
   -o gpurun_out/${tag}_c3_level_wide -f python tools/one_hull.py 3 > gpurun_out/${tag}_c3_lw.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:level_tma --launch-skip 13 -c 1 \
   -o gpurun_out/${tag}_c3_level_segcta -f python tools/one_hull.py 3 > gpurun_out/${tag}_c3_ls.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:finisher_batch --launch-skip 14 -c 2 \
   -o gpurun_out/${tag}_c3_finisher -f python tools/one_hull.py 3 > gpurun_out/${tag}_c3_fin.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:root_filter_tma --launch-skip 3 -c 1 \
   -o gpurun_out/${tag}_kf_disk -f python tools/cfg_time.py disk 1e8 5 > gpurun_out/${tag}_kf_disk.log 2>&1
ls -la gpurun_out/${tag}_*.ncu-rep
