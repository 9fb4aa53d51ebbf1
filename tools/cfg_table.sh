# per-config device time table (development aid)
for c in "disk 1e6 1" "square 1e8 2" "circle 1e7 3" "kuzmin 1e9 4" "disk 1e8 5"; do
  timeout 300 python tools/cfg_time.py $c
  VQHULL_ROOT=octagon timeout 300 python tools/cfg_time.py $c | sed 's/^/[octagon] /'
done
timeout 1500 python -m pytest tests -m slow -q -rs 2>&1 | tail -5
