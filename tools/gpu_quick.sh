#!/bin/bash
# Quick GPU round trip: full GPU suite (stop at first failure), then the
# device-resident bench line of the configs given.  usage: tools/gpu_quick.sh TAG "3 1 2"
tag=${1:-q}; cfgs=${2:-"3"}
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/${tag}_gpu_all.log 2>&1
tail -n 5 gpurun_out/${tag}_gpu_all.log
for c in $cfgs; do
  timeout 900 python bench.py --config $c --no-cpu --no-e2e --steps 5 --warmup 3 2>/dev/null | tail -1 >> gpurun_out/${tag}_configs.jsonl
done
python - <<PY
import json
for l in open("gpurun_out/${tag}_configs.jsonl"):
    d = json.loads(l)
    r = d.get("roofline", {})
    print(d["config"]["workload"][:40], f"{d['ms_per_step']:.3f} ms", r.get("families_ms_per_step"))
PY
