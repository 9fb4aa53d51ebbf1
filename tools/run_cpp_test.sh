set -e
g++ -std=c++17 -O1 -I include -I /usr/local/cuda/include tests/cpp/test_cpp_api.cpp -L paper_2510_09417_b200/lib -lvqhull_b200 -Wl,-rpath,$PWD/paper_2510_09417_b200/lib -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,/usr/local/cuda/lib64 -o /tmp/test_cpp_api
timeout 60 /tmp/test_cpp_api; echo "rc=$?"
