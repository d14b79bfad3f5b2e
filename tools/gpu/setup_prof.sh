# ncu --set full of the set-up kernels on configs[3]'s hierarchy at 128^3
#   bash tools/gpu/setup_prof.sh <tag>
T=${1:-setup}
mkdir -p gpurun_out
(compute-sanitizer --version; echo rc=$?) > gpurun_out/sanitizer_version.txt 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"k_thomas_factor|k_local_basis|k_cc_subspace|k_batched_gj|k_coarse_blocks" --launch-count 5 \
  -o gpurun_out/${T}_prof python tools/prof_case.py --n 128 --ncc 4 --sd 4 --lcc 12 --solves 1 \
  > gpurun_out/${T}_prof.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/${T}_prof.ncu-rep > gpurun_out/${T}_prof_summary.txt 2>&1
cat gpurun_out/${T}_prof_summary.txt
