# Round-2 evidence: default bench line (configs[3]), launch list, ncu --set full
# of the solve kernels, reference arm.  bash tools/gpu/final_r2.sh <tag>
T=$1
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_bench_reference.json 2> gpurun_out/${T}_bench_reference.err; echo "reference rc=$?"
CMD="python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --no-extra"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
  $CMD > gpurun_out/${T}_ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 2400 ncu --set full --clock-control none --import-source on \
  -k regex:"k_update|k_post_bnd|k_search|k_restrict_bnd" \
  --launch-skip 20 --launch-count 4 -o gpurun_out/${T}_solve $CMD > gpurun_out/${T}_ncu_full.log 2>&1
echo "ncu full rc=$?"
