# round profile: full bench line, launch list, ncu --set full of the three kernels of config 2
set -x
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 12 --csv --log-file gpurun_out/launches.csv python bench.py --profile --steps 2 --warmup 1 > gpurun_out/ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"poly_sample|root_filter_tma|tail_kernel" -c 3 -o gpurun_out/full python bench.py --profile --steps 1 --warmup 0 > gpurun_out/ncu_full.log 2>&1
for c in 1 3 4 5; do timeout 900 python bench.py --config $c --no-cpu --no-e2e --steps 5 >> gpurun_out/bench_configs.log 2>&1; done
cat gpurun_out/bench.log; tail -2 gpurun_out/bench_ref.log
