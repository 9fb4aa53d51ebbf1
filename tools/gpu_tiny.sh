g++ -std=c++17 -O2 -I include -I /usr/local/cuda/include tools/cbench/hull_loop.cpp -L paper_2510_09417_b200/lib -lvqhull_b200 -Wl,-rpath,$PWD/paper_2510_09417_b200/lib -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,/usr/local/cuda/lib64 -o /tmp/hull_loop
for k in "2 300 1 200" "2 700 1 200" "2 1e3 1 200" "3 1e8 2 30" "2 1e6 1 100"; do timeout 60 /tmp/hull_loop $k; done
VQHULL_TINY=0 timeout 60 /tmp/hull_loop 2 700 1 200
timeout 900 python -m pytest tests -q -x -m "gpu and not slow" 2>&1 | tail -2
