# quick GPU check: parity subset + bench (no side-by-side rows, no CPU baseline)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not block_jacobi_vs_oracle" > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/q_pytest.log
timeout 600 python bench.py --no-side-by-side --no-cpu-baseline > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/q_bench.json'))
print(d['value'], d['ms_per_step'], d['config']['kernel_ms_per_launch'], d['roofline']['frac'], d['clocks'])"
