grep -o -w "avx512f\|avx2\|amx_tile" /proc/cpuinfo | sort | uniq -c
timeout 2400 python -m pytest tests/test_gpu_configs.py -x -q -s --durations=0 2>&1 | tail -30
