python tools/true_residual_probe.py --n 128 --restarts 1 2>&1 | tail -3
timeout 1500 python -m pytest tests/test_gpu_configs.py -x -q -s 2>&1 | grep -E "configs|passed|failed|Error|assert" | head -30
timeout 1800 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_configs.py 2>&1 | tail -5
