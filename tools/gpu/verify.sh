set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r06_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/r06_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r06_smoke.log 2>&1; echo "smoke rc=$?"; cat gpurun_out/r06_smoke.log | tail -3
timeout 600 python bench.py > gpurun_out/r06_bench.json 2> gpurun_out/r06_bench.err; echo "bench rc=$?"; cat gpurun_out/r06_bench.json
