# cc-basis subspace-iteration knobs at configs[3]: set-up phases + iterations
for ks in 16 24; do for tol in 1e-12 1e-10; do
  echo "=== KS $ks tol $tol"
  TMG_CC_KS=$ks TMG_CC_TOL=$tol TMG_SETUP_PROFILE=1 timeout 600 python tools/setup_sweep.py --config 3 --settings "1e-9:32" 2>&1 | grep -E "cc |cc_basis|iterations|local_basis" | tail -4
done; done
