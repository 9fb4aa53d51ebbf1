g++ -std=c++17 -O2 -I include -I /usr/local/cuda/include tools/cbench/hull_loop.cpp -L paper_2510_09417_b200/lib -lvqhull_b200 -Wl,-rpath,$PWD/paper_2510_09417_b200/lib -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,/usr/local/cuda/lib64 -o /tmp/hull_loop
VQHULL_SAMPLE_TRACE=1 timeout 60 /tmp/hull_loop 3 1e8 2 5 2>&1 | tail -2
for k in "3 1e8 2 30" "2 1e8 5 10" "0 1e9 4 5" "2 1e6 1 100"; do timeout 60 /tmp/hull_loop $k; done
timeout 900 python -m pytest tests -q -x -m "gpu and not slow" 2>&1 | tail -2
