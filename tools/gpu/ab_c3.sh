# A/B of library variants at configs[3] (512^3): ms per PCG iteration,
# interleaved rounds.  bash tools/gpu/ab_c3.sh base l2a2 l2a4 ...
mkdir -p gpurun_out
for round in 1 2; do
  for v in "$@"; do
    if [ "$v" = base ]; then lib=paper_2410_06850_b200/libtopmg_b200.so; else lib=build_var/$v/libtopmg_b200.so; fi
    r=$(TMG_LIB=$lib timeout 300 python tools/config3.py --solves 3 2>/dev/null | tail -1)
    echo "$round $v $(echo $r | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["iterations"], round(d["ms_per_iteration"],3), round(d["mdof_iter_per_s"]))')"
  done
done
