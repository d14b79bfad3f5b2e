# Round-2e evidence: default bench line (configs[3]), reference arm, launch list,
# ncu --set full of the solve kernels, configs[4] slab proxy, configs[2] loops,
# the GPU test suite and smoke().  bash tools/gpu/final_r2e.sh <tag>
T=$1
bash tools/gpu/final_r2.sh $T
timeout 900 python tools/config4_proxy.py --out gpurun_out/${T}_config4_proxy.json > gpurun_out/${T}_config4_proxy.log 2>&1; echo "config4 proxy rc=$?"
timeout 600 python tools/simp_bench.py --out gpurun_out/${T}_simp.json > gpurun_out/${T}_simp.log 2>&1; echo "simp rc=$?"
timeout 600 python tools/optim_bench.py --out gpurun_out/${T}_optim.json > gpurun_out/${T}_optim.log 2>&1; echo "optim rc=$?"
python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest_gpu.txt 2>&1; tail -3 gpurun_out/${T}_pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1; tail -1 gpurun_out/${T}_smoke.txt
