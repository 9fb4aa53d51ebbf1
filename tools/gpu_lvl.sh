g++ -std=c++17 -O2 -I include -I /usr/local/cuda/include tools/cbench/hull_loop.cpp -L paper_2510_09417_b200/lib -lvqhull_b200 -Wl,-rpath,$PWD/paper_2510_09417_b200/lib -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,/usr/local/cuda/lib64 -o /tmp/hull_loop
timeout 60 /tmp/hull_loop 2 1e5 1 3 || { echo "small case failed/hung"; exit 1; }
for v in 2 1; do echo "level v$v"; for k in "1 1e7 3 5" "2 1e8 5 10" "3 1e8 2 20"; do if [ $v = 1 ]; then VQHULL_LEVEL_V1=1 timeout 120 /tmp/hull_loop $k; else timeout 120 /tmp/hull_loop $k; fi; done; done
timeout 900 python -m pytest tests -q -x -m "gpu" 2>&1 | tail -2
