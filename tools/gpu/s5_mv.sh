# Session-5 A/B: rows per mat-vec thread of the block solve (TMG_MV_ROWS 1/2/4).
# main lib = R 2, build_var/mv1 = R 1 (the round-2b layout), build_var/mv4 = R 4.
mkdir -p gpurun_out
for r in 1 2 4; do echo "== microbench R=$r"; timeout 120 tools/gpu/bin/thomas_bench_r$r; done > gpurun_out/s5_microbench.txt 2>&1
cat gpurun_out/s5_microbench.txt | grep -E "==|real |L2 |copy "
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shared_factors.py -x -q > gpurun_out/s5_pytest_mv2.txt 2>&1; tail -2 gpurun_out/s5_pytest_mv2.txt
TMG_LIB=build_var/mv4/libtopmg_b200.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shared_factors.py -x -q > gpurun_out/s5_pytest_mv4.txt 2>&1; tail -2 gpurun_out/s5_pytest_mv4.txt
bash tools/gpu/ab_c3.sh mv1 base mv4 > gpurun_out/s5_ab_c3.txt 2>&1; cat gpurun_out/s5_ab_c3.txt
for v in mv1 base mv4; do
  if [ "$v" = base ]; then lib=paper_2410_06850_b200/libtopmg_b200.so; else lib=build_var/$v/libtopmg_b200.so; fi
  echo "== $v"; TMG_LIB=$lib timeout 300 python tools/kernel_times.py --config 3 2>&1 | tail -8
done > gpurun_out/s5_kernel_times.txt 2>&1; cat gpurun_out/s5_kernel_times.txt
