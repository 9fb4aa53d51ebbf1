g++ -std=c++17 -O2 -I include -I /usr/local/cuda/include tools/cbench/hull_loop.cpp -L paper_2510_09417_b200/lib -lvqhull_b200 -Wl,-rpath,$PWD/paper_2510_09417_b200/lib -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,/usr/local/cuda/lib64 -o /tmp/hull_loop
for o in 2 1 2 1; do echo "occ $o"; for k in "3 1e8 2 30" "2 1e6 1 100" "2 1e3 1 200"; do VQHULL_TAIL_OCC=$o /tmp/hull_loop $k; done; done
