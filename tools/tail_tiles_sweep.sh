# VQHULL_TAIL_MAXTILES sweep (largest level the persistent tail kernel takes over)
for t in 148 296 592 1184; do
  for c in "--config 2" "--config 5 --n 100000000" "--config 3" "--config 1"; do
    r=$(VQHULL_TAIL_MAXTILES=$t timeout 300 python bench.py $c --steps 20 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.readline());print(round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['roofline']['families_ms_per_step'].items() if v})")
    echo "maxtiles=$t $c $r" >> gpurun_out/tail_tiles_sweep.log
  done
done
