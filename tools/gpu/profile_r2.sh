# Round-2 evidence at the headline config (configs[3], 512^3): launch list +
# one ncu --set full capture of the solve kernels. Run after the plain bench
# exited 0.   bash tools/gpu/profile_r2.sh <tag>
T=$1
mkdir -p gpurun_out
CMD="python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --no-extra"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
  $CMD > gpurun_out/${T}_ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 2400 ncu --set full --clock-control none --import-source on \
  -k regex:"k_update|k_post_bnd|k_search|k_restrict_bnd|k_coarse|k_symv|k_gemv|k_acc" \
  --launch-skip 300 --launch-count 12 -o gpurun_out/${T}_solve $CMD > gpurun_out/${T}_ncu_full.log 2>&1
echo "ncu full rc=$?"
