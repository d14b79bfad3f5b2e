# Session-5 step 4: packed diagonal blocks + deferred p.q reduction: microbench,
# correctness, configs[3] A/B against the variants without each change.
mkdir -p gpurun_out
for v in r2 r2pack; do echo "== microbench $v nb=32768"; timeout 200 tools/gpu/bin/thomas_persist_$v 32768 | head -4; done > gpurun_out/s5d_microbench.txt 2>&1
cat gpurun_out/s5d_microbench.txt
timeout 1500 python -m pytest tests/test_gpu_shared_factors.py tests/test_gpu_parity.py -x -q > gpurun_out/s5d_pytest.txt 2>&1; tail -3 gpurun_out/s5d_pytest.txt
bash tools/gpu/ab_c3.sh nopack base nodefer nohint > gpurun_out/s5d_ab_c3.txt 2>&1; cat gpurun_out/s5d_ab_c3.txt
for v in base; do
  lib=paper_2410_06850_b200/libtopmg_b200.so
  echo "== $v"; TMG_LIB=$lib timeout 300 python tools/kernel_times.py --config 3 2>&1 | tail -8
  echo "== $v configs[1]"; TMG_LIB=$lib timeout 300 python tools/kernel_times.py --config 1 2>&1 | tail -8
done > gpurun_out/s5d_kernel_times.txt 2>&1; cat gpurun_out/s5d_kernel_times.txt
