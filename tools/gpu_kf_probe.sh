# K_F change probe: C++ loop on disk/square, family times, all GPU tests
g++ -std=c++17 -O2 -I include -I /usr/local/cuda/include tools/cbench/hull_loop.cpp -L paper_2510_09417_b200/lib -lvqhull_b200 -Wl,-rpath,$PWD/paper_2510_09417_b200/lib -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,/usr/local/cuda/lib64 -o /tmp/hull_loop
for k in "2 1e8 5 10" "3 1e8 2 30" "2 1e6 1 100" "1 1e7 3 5"; do timeout 120 /tmp/hull_loop $k; done
for c in "disk 1e8 5" "kuzmin 1e9 4"; do timeout 300 python tools/cfg_time.py $c 2>&1 | tail -1; done
timeout 1500 python -m pytest tests -q -x -m "gpu" 2>&1 | tail -3
