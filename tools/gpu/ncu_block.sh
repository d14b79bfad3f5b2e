# ncu captures of the fine block solve: the microbenchmark and the live k_update / k_post
set -x
mkdir -p gpurun_out
./tools/gpu/bin/thomas_bench > gpurun_out/tb.log 2>&1; cat gpurun_out/tb.log
ncu --set full --clock-control none --import-source on -k regex:k_bench -c 3 -o gpurun_out/tb ./tools/gpu/bin/thomas_bench > gpurun_out/tb_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_update|k_post|k_search" --launch-skip 30 -c 3 -o gpurun_out/solve python bench.py --steps 3 --warmup 3 --no-side-by-side --no-cpu-baseline > gpurun_out/solve_ncu.log 2>&1
tail -3 gpurun_out/solve_ncu.log
