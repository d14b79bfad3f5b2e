# ncu --set full of selected solve kernels: bash tools/gpu/ncu_kernels.sh <tag> <regex>
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$2" \
  --launch-skip 40 --launch-count 4 -o gpurun_out/$1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-side-by-side \
  > gpurun_out/$1.log 2>&1; echo "ncu rc=$?"
