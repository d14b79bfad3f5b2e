timeout 2400 python -m pytest tests -m gpu -q --maxfail=5 -p no:cacheprovider 2>&1 | tail -12
CMD="python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --no-extra"
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"k_update|k_post_bnd|k_search|k_restrict_bnd|k_coarse_smooth" \
  --launch-skip 20 --launch-count 5 -o gpurun_out/r2b_solve $CMD > gpurun_out/r2b_ncu_full.log 2>&1
echo "ncu full rc=$?"
timeout 1200 python tools/config4_proxy.py --out gpurun_out/r2_config4_proxy.json 2>&1 | tail -2
TMG_SETUP_PROFILE=1 timeout 900 python tools/setup_sweep.py --config 3 --settings "1e-11:32,1e-9:32,1e-8:32,1e-9:24,1e-9:16" > gpurun_out/r2_setup_sweep.json 2> gpurun_out/r2_setup_sweep.err
echo "sweep rc=$?"; cat gpurun_out/r2_setup_sweep.json
