# generic brick shapes (row A20): bash tools/gpu/generic_check.sh
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_generic.py -q --timeout 600 > gpurun_out/generic.log 2>&1; echo "generic rc=$?"
grep -E "passed|failed|Error|^E  " gpurun_out/generic.log | head -30

