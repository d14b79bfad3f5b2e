mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shared_factors.py tests/test_gpu_parity.py -q -x -k "shared or local or basis or warm or vcycle" > gpurun_out/shared.log 2>&1; echo "shared rc=$?"; grep -E "passed|failed|^E  " gpurun_out/shared.log | head -12
for ks in 16 24; do
TMG_CC_KS=$ks TMG_SETUP_PROFILE=1 timeout 900 python tools/setup_sweep.py --config 3 --settings "0:0" > gpurun_out/setup3_ks$ks.log 2>&1; echo "setup ks=$ks rc=$?"; grep -E "setup\]|setup_ms" gpurun_out/setup3_ks$ks.log | tail -10
done
