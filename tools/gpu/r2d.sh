timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s -k "cc_blocks_32 or adapter or limits" 2>&1 | tail -15
timeout 900 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc=$?"; tail -3 gpurun_out/r2_bench.err
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
