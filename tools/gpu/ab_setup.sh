# A/B of library variants: set-up phases at configs[3]   bash tools/gpu/ab_setup.sh base v1 v2
for v in "$@"; do
  if [ "$v" = base ]; then lib=paper_2410_06850_b200/libtopmg_b200.so; else lib=build_var/$v/libtopmg_b200.so; fi
  echo "=== $v"
  TMG_LIB=$lib TMG_SETUP_PROFILE=1 timeout 600 python tools/setup_sweep.py --config 3 --settings "0:0" 2>&1 | grep -E "local_basis|thomas|cc_basis|setup_ms" | tail -4
done
