# Session-5 step 7: batched loads in k_restrict_bnd
mkdir -p gpurun_out
bash tools/gpu/ab_c3.sh prev base > gpurun_out/s5g_ab_c3.txt 2>&1; cat gpurun_out/s5g_ab_c3.txt
for v in prev base; do
  if [ "$v" = base ]; then lib=paper_2410_06850_b200/libtopmg_b200.so; else lib=build_var/$v/libtopmg_b200.so; fi
  echo "== $v"; TMG_LIB=$lib timeout 300 python tools/kernel_times.py --config 3 2>&1 | tail -8
done > gpurun_out/s5g_kernel_times.txt 2>&1; cat gpurun_out/s5g_kernel_times.txt
timeout 2400 python -m pytest tests/test_gpu_shared_factors.py tests/test_gpu_parity.py tests/test_gpu_slabs.py -x -q > gpurun_out/s5g_pytest.txt 2>&1; tail -3 gpurun_out/s5g_pytest.txt
