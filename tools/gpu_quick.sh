# quick GPU cycle: parity tests (not slow), bench line, launch list
set -x
timeout 1200 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench.log 2>gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --profile --steps 2 --warmup 1 > gpurun_out/ncu.log 2>&1
tail -5 gpurun_out/gpu_tests.log; cat gpurun_out/bench.log; tail -3 gpurun_out/bench.err
