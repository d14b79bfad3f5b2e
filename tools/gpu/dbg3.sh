mkdir -p gpurun_out
timeout 300 python tools/generic_debug2.py > gpurun_out/eigdbg2.log 2>&1; echo "dbg rc=$?"; cat gpurun_out/eigdbg2.log | tail -14
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/generic_debug2.py > gpurun_out/eigdbg3.log 2>&1; echo "dbg blocking rc=$?"; cat gpurun_out/eigdbg3.log | tail -14
