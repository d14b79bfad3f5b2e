mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_generic.py -q --timeout 600 > gpurun_out/generic.log 2>&1; echo "generic rc=$?"
grep -E "passed|failed|Error|^E  " gpurun_out/generic.log | head -30
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x > gpurun_out/parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/parity.log
