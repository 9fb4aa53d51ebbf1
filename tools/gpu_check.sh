#!/bin/bash
# One GPU round trip: box facts, the sharded-path GPU tests, the full GPU
# suite, the default bench line and the reference arm.  Logs in gpurun_out/.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/box.txt 2>&1
(free -g; nproc; lscpu | grep -i "model name") >> gpurun_out/box.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests/test_sharded_gpu.py -x -q > gpurun_out/sharded.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_all.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
tail -n 3 gpurun_out/sharded.log; tail -n 3 gpurun_out/gpu_all.log; cat gpurun_out/bench.log gpurun_out/bench_ref.log
