timeout 2400 python -m pytest tests -m gpu -q --maxfail=10 -p no:cacheprovider 2>&1 | tail -15
timeout 900 python tools/config4_proxy.py --out gpurun_out/r2_config4_proxy.json 2>&1 | tail -3
bash tools/gpu/profile_r2.sh r2a 2>&1 | tail -3
bash tools/gpu/sanitize.sh memcheck 2>&1 | tail -12
