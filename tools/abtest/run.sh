# A/B of prebuilt library variants with the C++ loop (LD_LIBRARY_PATH swap)
g++ -std=c++17 -O2 -I include -I /usr/local/cuda/include tools/cbench/hull_loop.cpp -L paper_2510_09417_b200/lib -lvqhull_b200 -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,/usr/local/cuda/lib64 -o /tmp/hull_loop
for v in ${VARIANTS:-libA libB}; do mkdir -p /tmp/$v; cp tools/abtest/$v.so /tmp/$v/libvqhull_b200.so; echo "== $v"
  LD_LIBRARY_PATH=/tmp/$v timeout 60 /tmp/hull_loop 2 1e8 5 10; LD_LIBRARY_PATH=/tmp/$v timeout 60 /tmp/hull_loop 3 1e8 2 30; LD_LIBRARY_PATH=/tmp/$v timeout 60 /tmp/hull_loop 2 1e6 1 200; done
