# configs[2] SIMP loop and configs[1] bench with the dense A_cc inverse vs the plane block Thomas
mkdir -p gpurun_out
for P in 0 1; do
  TMG_ACC_PLANES=$P timeout 600 python tools/simp_bench.py --out gpurun_out/simp_planes$P.json > gpurun_out/simp_planes$P.log 2>&1; echo "simp planes=$P rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/simp_planes$P.json')); print('planes=$P', {k: d[k] for k in ('seconds_per_design_iteration','setup_s','ls1_s','ls2_s')}, d['ls1_iterations'])"
  TMG_ACC_PLANES=$P timeout 600 python bench.py --no-side-by-side --no-cpu-baseline > gpurun_out/bench_planes$P.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_planes$P.json')); print('planes=$P', round(d['value']), d['config']['iterations'], round(d['ms_per_step'],3), d['config']['kernel_ms_per_launch'], round(d['config']['setup_ms'],1), round(d['config']['time_to_solution_ms'],1))"
done
