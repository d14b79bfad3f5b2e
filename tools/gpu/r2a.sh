set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep -i "model name"; free -g | head -2
for n in 256 512; do
python tools/config3.py --n $n --solves 1 --out gpurun_out/c3_bnd_$n.json 2>&1 | tail -2
TMG_LIB=build_var/literal/libtopmg_b200.so python tools/config3.py --n $n --solves 1 --out gpurun_out/c3_lit_$n.json 2>&1 | tail -2
done
