for n in 20000 50000 100000 200000 400000; do timeout 120 python tools/repro_config.py circle $n 3 2 2>&1 | grep -E "rep 1|ERR" | cut -c1-120; done
echo "--- no prefetch"
for n in 200000 1000000; do VQHULL_LIB=paper_2510_09417_b200/lib/libvqhull_b200_nopf.so timeout 120 python tools/repro_config.py circle $n 3 3 2>&1 | grep -E "rep|ERR" | cut -c1-120; done
