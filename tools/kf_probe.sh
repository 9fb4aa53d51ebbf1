g++ -std=c++17 -O2 -I include -I /usr/local/cuda/include tools/cbench/hull_loop.cpp -L paper_2510_09417_b200/lib -lvqhull_b200 -Wl,-rpath,$PWD/paper_2510_09417_b200/lib -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,/usr/local/cuda/lib64 -o /tmp/hull_loop
for k in "3 1e8 2 30" "2 1e8 5 10" "0 1e9 4 5"; do timeout 60 /tmp/hull_loop $k; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:root_filter -c 3 python bench.py --profile --steps 2 --warmup 1 2>&1 | grep -E "duration|grid" | head -6
