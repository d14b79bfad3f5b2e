timeout 600 python -m pytest tests/test_gpu_gen.py -q -k tree 2>&1 | tail -2
timeout 1800 python tools/config4_proxy.py --out gpurun_out/r2_config4_proxy.json 2>&1 | tail -2
