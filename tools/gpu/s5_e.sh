# Session-5 step 5: deferred grid sums of k_update / k_post_bnd (k_reduce_fin)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_shared_factors.py tests/test_gpu_parity.py tests/test_gpu_slabs.py tests/test_gpu_configs.py -x -q > gpurun_out/s5e_pytest.txt 2>&1; tail -3 gpurun_out/s5e_pytest.txt
bash tools/gpu/ab_c3.sh nofdefer base > gpurun_out/s5e_ab_c3.txt 2>&1; cat gpurun_out/s5e_ab_c3.txt
for v in base; do
  lib=paper_2410_06850_b200/libtopmg_b200.so
  echo "== $v"; TMG_LIB=$lib timeout 300 python tools/kernel_times.py --config 3 2>&1 | tail -8
  echo "== $v configs[1]"; TMG_LIB=$lib timeout 300 python tools/kernel_times.py --config 1 2>&1 | tail -8
done > gpurun_out/s5e_kernel_times.txt 2>&1; cat gpurun_out/s5e_kernel_times.txt
