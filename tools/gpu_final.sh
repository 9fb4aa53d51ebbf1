# round-end evidence: tests (all), smoke, bench lines, launch list, ncu capture
set -x
timeout 1800 python -m pytest tests -m gpu -q -rs > gpurun_out/gpu_tests_all.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
bash tools/gpu_profile.sh
tail -3 gpurun_out/gpu_tests_all.log; cat gpurun_out/smoke.log
