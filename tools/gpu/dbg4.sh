mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_generic.py -q --timeout 600 > gpurun_out/generic.log 2>&1; echo "generic rc=$?"
grep -E "passed|failed|Error|^E  " gpurun_out/generic.log | head -30
TMG_SETUP_PROFILE=1 timeout 900 python tools/setup_sweep.py --config 3 --settings "0:0" > gpurun_out/setup3.log 2>&1; echo "setup rc=$?"; grep -E "setup\]|setup_ms" gpurun_out/setup3.log | tail -10
