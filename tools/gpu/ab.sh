# A/B: in-tree library vs tools/gpu/bin/libtopmg_<v>.so for each argument v
mkdir -p gpurun_out
for V in "$@"; do
[ -n "$AB_TESTS" ] && TMG_LIB=$PWD/tools/gpu/bin/libtopmg_$V.so timeout 900 python -m pytest tests -m gpu -x -q -k "not block_jacobi_vs_oracle" > gpurun_out/ab_pytest_$V.log 2>&1; echo "pytest $V rc=$?"; tail -1 gpurun_out/ab_pytest_$V.log
done
for lib in base "$@"; do
  if [ $lib = base ]; then unset TMG_LIB; else export TMG_LIB=$PWD/tools/gpu/bin/libtopmg_$lib.so; fi
  timeout 600 python bench.py --no-side-by-side --no-cpu-baseline > gpurun_out/ab_bench_$lib.json 2> gpurun_out/ab_bench_$lib.err; echo "bench $lib rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/ab_bench_$lib.json'))
print('$lib', round(d['value']), d['config']['iterations'], round(d['ms_per_step'],3), d['config']['kernel_ms_per_launch'], round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], round(d['config']['setup_ms'],1))"
done
