mkdir -p gpurun_out
timeout 300 python tools/generic_debug.py > gpurun_out/eigdbg_normal.log 2>&1; echo "dbg rc=$?"; cat gpurun_out/eigdbg_normal.log | tail -6
timeout 1500 python -m pytest tests/test_gpu_generic.py -q --timeout 600 > gpurun_out/generic.log 2>&1; echo "generic rc=$?"
grep -E "passed|failed|Error|^E  " gpurun_out/generic.log | head -30
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_thomas_factor" --launch-count 1 \
  -o gpurun_out/thomas_prof python tools/prof_case.py --n 128 --ncc 8 --sd 2 --solves 1 > gpurun_out/thomas_prof.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/thomas_prof.ncu-rep
