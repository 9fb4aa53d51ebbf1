g++ -std=c++17 -O2 -I include -I /usr/local/cuda/include tools/cbench/hull_loop.cpp -L paper_2510_09417_b200/lib -lvqhull_b200 -Wl,-rpath,$PWD/paper_2510_09417_b200/lib -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,/usr/local/cuda/lib64 -o /tmp/hull_loop
for n in 2.5e7 5e7 1e8 2e8 4e8; do VQHULL_SAMPLE_TRACE=1 timeout 120 /tmp/hull_loop 3 $n 2 5 2>&1 | tail -2; done
