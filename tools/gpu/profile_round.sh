# Round evidence: bench line, launch list, one ncu --set full capture of the solve kernels.
#   bash tools/gpu/profile_round.sh <tag>
T=$1
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
cat gpurun_out/${T}_bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-side-by-side > gpurun_out/${T}_ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_update|k_post_bnd|k_search|k_restrict_bnd|k_coarse_fused" \
  --launch-skip 40 --launch-count 5 -o gpurun_out/${T}_solve python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-side-by-side \
  > gpurun_out/${T}_ncu_full.log 2>&1; echo "ncu full rc=$?"
