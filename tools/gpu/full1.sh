mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shared_factors.py -q -x > gpurun_out/shared.log 2>&1; echo "shared rc=$?"; grep -E "passed|failed|^E  " gpurun_out/shared.log | head -12
timeout 2700 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-extra > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; head -c 1500 gpurun_out/bench.json
