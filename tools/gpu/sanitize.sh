# compute-sanitizer over every kernel family (tools/sanitize_cases.py).
#   bash tools/gpu/sanitize.sh [tools...]   -> gpurun_out/sanitize/<tool>_<case>.log
mkdir -p gpurun_out/sanitize
TOOLS=${@:-memcheck racecheck synccheck}
CASES="mmg_cell mmg_cc16 mmg_cc32 mmg_large_q two_grid block_jacobi jacobi acc_planes slabs gen_optim simp"
for t in $TOOLS; do
  for c in $CASES; do
    extra=""
    [ "$t" = "memcheck" ] && extra="--leak-check no"
    [ "$t" = "racecheck" ] && extra="--racecheck-report all"
    timeout 900 compute-sanitizer --tool $t $extra --target-processes all --print-limit 20 \
      python tools/sanitize_cases.py $c > gpurun_out/sanitize/${t}_${c}.log 2>&1
    echo "$t $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize/${t}_${c}.log | tail -1)"
  done
done
