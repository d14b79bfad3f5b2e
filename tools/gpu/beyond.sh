# configs[3] (512^3, one GPU), configs[2] SIMP loop, reference MMA loop
mkdir -p gpurun_out
timeout 900 python tools/config3.py --out gpurun_out/r06_config3_512_lcc12.json > gpurun_out/r06_config3.log 2>&1; echo "config3 rc=$?"; tail -3 gpurun_out/r06_config3.log
timeout 600 python tools/simp_bench.py --out gpurun_out/r06_simp.json > gpurun_out/r06_simp.log 2>&1; echo "simp rc=$?"; tail -1 gpurun_out/r06_simp.log | cut -c1-400
timeout 600 python tools/optim_bench.py --out gpurun_out/r06_optim.json > gpurun_out/r06_optim.log 2>&1; echo "optim rc=$?"; tail -1 gpurun_out/r06_optim.log | cut -c1-400
