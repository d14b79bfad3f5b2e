timeout 1800 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "num_local_basis or smoother_sweeps or mmg_pcg or local_bases or coarse_operator or vcycle or golden" 2>&1 | tail -4
bash tools/gpu/ab_c3.sh base
