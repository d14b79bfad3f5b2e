bash tools/gpu/ab_c3.sh base
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -x -q -p no:cacheprovider 2>&1 | tail -3
TMG_SETUP_PROFILE=1 timeout 600 python tools/setup_sweep.py --config 3 --settings "0:0" 2>&1 | grep -E "setup\]|setup_ms" | tail -9
