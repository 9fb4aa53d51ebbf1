for c in "square 1e8 2" "disk 1e6 1" "disk 1e8 5" "kuzmin 1e8 4"; do
VQHULL_TAIL_TRACE=1 python tools/cfg_time.py $c 2>&1 | tail -14
done
