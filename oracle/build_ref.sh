#!/usr/bin/env bash
# ORACLE — test infrastructure only.
# Compiles the reference's own proj/core sources, unmodified and where they lie
# under /root/reference, together with the Eigen-API subset shim
# (oracle/eigen_shim) and the C harness (oracle/ref_harness.cpp) into
# oracle/_ref/libtopmg_ref.so. No reference source is copied into the repo and
# the reference's own CMake build is not used. The output is git-ignored but
# travels to the GPU box with the working tree.
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
REF="${TOPMG_REFERENCE:-/root/reference}/proj/core"
OUT="$HERE/_ref"
if [ ! -d "$REF/src" ]; then
  echo "build_ref.sh: reference sources not found at $REF" >&2
  exit 1
fi
mkdir -p "$OUT/obj"
CXX=/usr/bin/g++
CC=/usr/bin/gcc
# x86-64-v2: portable to the GPU box host; no FMA contraction (matches the
# oracle restatement's rounding of dot products).
FLAGS="-O2 -march=x86-64-v2 -fPIC -pthread"
SRCS="grid material fvm sparse solver coarse_space parallel rng optim io"
pids=()
for s in $SRCS; do
  $CXX -std=c++20 $FLAGS -I"$REF/include" -I"$HERE/eigen_shim" -c "$REF/src/$s.cpp" -o "$OUT/obj/$s.o" &
  pids+=($!)
done
$CXX -std=c++20 $FLAGS -I"$REF/include" -I"$HERE/eigen_shim" -c "$HERE/ref_harness.cpp" -o "$OUT/obj/ref_harness.o" &
pids+=($!)
$CC -std=c11 $FLAGS -c "$HERE/dense_la.c" -o "$OUT/obj/dense_la.o" &
pids+=($!)
$CC -std=c11 $FLAGS -c "$HERE/lapack_glue.c" -o "$OUT/obj/lapack_glue.o" &
pids+=($!)
for p in "${pids[@]}"; do wait "$p"; done
$CXX -shared -pthread -o "$OUT/libtopmg_ref.so" "$OUT"/obj/*.o -lm -ldl
echo "built $OUT/libtopmg_ref.so"
# Timing variant for bench.py's CPU arm (-O3 -march=native).
# Built here for this container's CPU; bench.py probes it in a child process
# on the GPU box and falls back to the portable build if the ISA is missing.
NFLAGS="-O3 -march=native -fPIC -pthread"
mkdir -p "$OUT/obj_native"
pids=()
for s in $SRCS; do
  $CXX -std=c++20 $NFLAGS -I"$REF/include" -I"$HERE/eigen_shim" -c "$REF/src/$s.cpp" -o "$OUT/obj_native/$s.o" &
  pids+=($!)
done
$CXX -std=c++20 $NFLAGS -I"$REF/include" -I"$HERE/eigen_shim" -c "$HERE/ref_harness.cpp" -o "$OUT/obj_native/ref_harness.o" &
pids+=($!)
$CC -std=c11 $NFLAGS -c "$HERE/dense_la.c" -o "$OUT/obj_native/dense_la.o" &
pids+=($!)
$CC -std=c11 $NFLAGS -c "$HERE/lapack_glue.c" -o "$OUT/obj_native/lapack_glue.o" &
pids+=($!)
for p in "${pids[@]}"; do wait "$p"; done
$CXX -shared -pthread -o "$OUT/libtopmg_ref_native.so" "$OUT"/obj_native/*.o -lm -ldl
$CXX -march=native -Q --help=target 2>/dev/null | awk '$1 == "-march=" {print "march=" $2}' \
  > "$OUT/libtopmg_ref_native.so.march"
echo "built $OUT/libtopmg_ref_native.so ($(cat "$OUT/libtopmg_ref_native.so.march"))"
# integration demo of include/topmg_b200.hpp inside the reference code base
if [ -f "$HERE/../paper_2410_06850_b200/libtopmg_b200.so" ]; then
  $CXX -std=c++20 $FLAGS -I"$REF/include" -I"$HERE/../include" "$HERE/adapter_demo.cpp" \
    "$OUT"/obj/{grid,material,fvm,sparse,solver,coarse_space,parallel,rng,dense_la,lapack_glue}.o \
    -L"$HERE/../paper_2410_06850_b200" -ltopmg_b200 -Wl,-rpath,'$ORIGIN/../../paper_2410_06850_b200' \
    -ldl -o "$OUT/adapter_demo"
  echo "built $OUT/adapter_demo"
fi
