# K_S CTAs per SM vs the K_S -> K_F launch gap (config 2)
for o in 1 2 4 8; do
  VQHULL_POLY_OCC=$o VQHULL_SAMPLE_TRACE=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e 2> gpurun_out/pocc$o.err > /dev/null
  r=$(VQHULL_POLY_OCC=$o timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.readline());print(round(d['ms_per_step'],4))")
  echo "occ=$o ms=$r $(grep '\[sample\]' gpurun_out/pocc$o.err | tail -1)" >> gpurun_out/poly_occ.log
done
