#!/bin/bash
# Bench lines of every BASELINE config (device-resident, no CPU/e2e legs).
# usage: tools/gpu_configs.sh TAG
tag=${1:-cfg}
for c in 1 2 3 4 5; do
  timeout 900 python bench.py --config $c --no-cpu --no-e2e --steps 5 --warmup 3 2>/dev/null | tail -1 >> gpurun_out/${tag}_configs.jsonl
done
python - <<PY
import json
for l in open("gpurun_out/${tag}_configs.jsonl"):
    d = json.loads(l)
    r = d.get("roofline", {})
    print(d["config"]["workload"][:60], f"{d['ms_per_step']:.3f} ms", f"{d['value']:.3g} pts/s",
          r.get("kernel", "")[:30], f"{r.get('frac', 0):.3f}", r.get("families_ms_per_step"))
PY
