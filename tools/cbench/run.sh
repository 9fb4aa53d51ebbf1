g++ -std=c++17 -O2 -I include -I /usr/local/cuda/include tools/cbench/hull_loop.cpp -L paper_2510_09417_b200/lib -lvqhull_b200 -Wl,-rpath,$PWD/paper_2510_09417_b200/lib -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,/usr/local/cuda/lib64 -o /tmp/hull_loop || exit 1
/tmp/hull_loop 3 1e8 2 30
/tmp/hull_loop 2 1e3 1 200
/tmp/hull_loop 2 1e6 1 100
