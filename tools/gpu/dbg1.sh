mkdir -p gpurun_out
TMG_LIB=build_var/eigdbg/libtopmg_b200.so timeout 300 python tools/generic_debug.py > gpurun_out/eigdbg.log 2>&1; echo "dbg rc=$?"
grep -v "^\[eig" gpurun_out/eigdbg.log | tail -8; grep "^\[eig" gpurun_out/eigdbg.log | head -40
bash tools/gpu/setup_prof.sh setup_r2
