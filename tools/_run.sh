set -x
timeout 900 python -m pytest tests/test_sharded_gpu.py -x -q > gpurun_out/fb2_sharded.log 2>&1; tail -n 3 gpurun_out/fb2_sharded.log
L=paper_2510_09417_b200/lib
bash tools/variants.sh "circle:1e7:3 disk:1e8:7" $L/libvqhull_b200.so $L/libvqhull_b200_fb4.so > gpurun_out/fb2_variants.txt 2>&1
cat gpurun_out/fb2_variants.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:finisher_batch --launch-skip 12 -c 6 \
   -o gpurun_out/fb2_finisher -f python tools/one_hull.py 3 > gpurun_out/fb2_fin.log 2>&1
