mkdir -p gpurun_out
TMG_SETUP_PROFILE=1 timeout 900 python tools/setup_sweep.py --config 3 --settings "0:0" > gpurun_out/setup3.log 2>&1; echo "setup rc=$?"; grep -E "setup\]|setup_ms" gpurun_out/setup3.log | tail -10
timeout 2700 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
