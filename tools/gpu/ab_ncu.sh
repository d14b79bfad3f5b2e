# quick_ab plus DRAM bytes of the solve kernels for base and each variant
bash tools/gpu/quick_ab.sh "$@"
for lib in base "$@"; do
  if [ $lib = base ]; then unset TMG_LIB; else export TMG_LIB=$PWD/tools/gpu/bin/libtopmg_$lib.so; fi
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_update|k_post|k_search" \
    --launch-skip 40 --launch-count 4 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-side-by-side 2>/dev/null \
    | grep -E "k_update|k_post" | awk -F'","' -v L=$lib '{print L, substr($5,1,40), $(NF-2), $NF}' | tr -d '"'
done
