# EXPERIMENT (round 1): needs a lib/libvqhull_b200_exp.so built with upload_root_consts limited to the first calls; compares the K_S->K_F gap
for lib in libvqhull_b200.so libvqhull_b200_exp.so; do
  VQHULL_LIB=paper_2510_09417_b200/lib/$lib VQHULL_GRAPH=0 VQHULL_SAMPLE_TRACE=1 timeout 300 python bench.py --steps 5 --warmup 4 --no-cpu --no-e2e 2> gpurun_out/exp_$lib.err > /dev/null
  r=$(VQHULL_LIB=paper_2510_09417_b200/lib/$lib VQHULL_GRAPH=0 timeout 300 python bench.py --steps 20 --warmup 4 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.readline());print(round(d['ms_per_step'],4), d['config']['hull_vertices'])")
  echo "$lib ms,h=$r $(grep '\[sample\]' gpurun_out/exp_$lib.err | tail -1)" >> gpurun_out/exp_const.log
done
