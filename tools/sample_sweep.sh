# VQHULL_SAMPLE_MIN sweep (poly_sample_kernel sample size) on config 2, disk 1e8, disk 1e6
for s in 375000 750000 1500000 3000000; do
  for c in "--config 2" "--config 5 --n 100000000" "--config 1"; do
    r=$(VQHULL_SAMPLE_MIN=$s timeout 300 python bench.py $c --steps 20 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.readline());print(round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['roofline']['families_ms_per_step'].items() if v})")
    echo "smin=$s $c $r" >> gpurun_out/sample_sweep.log
  done
done
