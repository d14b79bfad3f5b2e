mkdir -p gpurun_out
timeout 600 python tools/kernel_times.py --config 3 > gpurun_out/kt.log 2>&1; echo "kt rc=$?"; tail -7 gpurun_out/kt.log
timeout 2700 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
