python tools/eig_probe.py --n 256
timeout 900 ncu --set full --clock-control none -k regex:"k_local_basis|k_thomas_factor|k_cc_subspace|k_batched_gj" --launch-count 4 -o gpurun_out/r2c_setup python tools/config3.py --n 256 --solves 1 > gpurun_out/r2c_ncu.log 2>&1; echo "ncu rc=$?"
