g++ -std=c++17 -O2 -I include -I /usr/local/cuda/include tools/cbench/hull_loop.cpp -L paper_2510_09417_b200/lib -lvqhull_b200 -Wl,-rpath,$PWD/paper_2510_09417_b200/lib -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,/usr/local/cuda/lib64 -o /tmp/hull_loop
for k in "1 1e7 3 5" "2 1e8 5 10" "3 1e8 2 30" "2 1e6 1 200"; do timeout 60 /tmp/hull_loop $k; done
for c in 1 3 4 5; do timeout 900 python bench.py --config $c --no-cpu --no-e2e --steps 5 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['ms_per_step'])"; done
timeout 1500 python -m pytest tests -q -x -m gpu 2>&1 | tail -2
