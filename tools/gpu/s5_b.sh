# Session-5 step 2: L2 look-ahead / hints with two rows per thread (microbench),
# correctness and configs[3] A/B of the current library (R 2, register-line
# fast diagonalisation, k_search without the stored diagonal) against mv1.
mkdir -p gpurun_out
for v in r2 r2_a1 r2_a2 r2_a4 r2_nohint; do echo "== microbench $v"; timeout 120 tools/gpu/bin/thomas_bench_$v | head -4; done > gpurun_out/s5b_microbench.txt 2>&1
cat gpurun_out/s5b_microbench.txt
timeout 1500 python -m pytest tests/test_gpu_shared_factors.py tests/test_gpu_parity.py -x -q > gpurun_out/s5b_pytest.txt 2>&1; tail -3 gpurun_out/s5b_pytest.txt
bash tools/gpu/ab_c3.sh mv1 base > gpurun_out/s5b_ab_c3.txt 2>&1; cat gpurun_out/s5b_ab_c3.txt
for v in base; do
  lib=paper_2410_06850_b200/libtopmg_b200.so
  echo "== $v"; TMG_LIB=$lib timeout 300 python tools/kernel_times.py --config 3 2>&1 | tail -8
  echo "== $v configs[1]"; TMG_LIB=$lib timeout 300 python tools/kernel_times.py --config 1 2>&1 | tail -8
done > gpurun_out/s5b_kernel_times.txt 2>&1; cat gpurun_out/s5b_kernel_times.txt
