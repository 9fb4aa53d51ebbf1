# K_F on disk 1e8: family times + one ncu --set full capture of root_filter_tma
python tools/cfg_time.py disk 1e8 5 2>&1 | tail -1
python tools/cfg_time.py square 1e8 2 2>&1 | tail -1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"root_filter_tma" -s 3 -c 1 -o gpurun_out/kf_disk python tools/cfg_time.py disk 1e8 5 > gpurun_out/kf_disk.log 2>&1; echo ncu rc=$?
