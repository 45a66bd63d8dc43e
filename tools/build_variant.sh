#!/bin/bash
# Build libchr.so with extra nvcc defines into build/variants/<name>.so
# (select at run time with CHR_LIB_PATH):  tools/build_variant.sh NAME -DCHR_KBT=512 ...
set -e
name=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=$ROOT/paper_2408_05462_b200/csrc
OUT=$ROOT/build/variants/$name
mkdir -p $OUT
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC --expt-relaxed-constexpr"
rm -f $OUT/*.o
pids=()
for f in $SRC/*.cu; do
  nvcc $FLAGS "$@" -c $f -o $OUT/$(basename $f .cu).o &
  pids+=($!)
done
g++ -O2 -fPIC -std=c++17 -ffp-contract=off -c $SRC/plan.cpp -o $OUT/plan.o
for p in "${pids[@]}"; do wait $p || { echo "variant $name: compile failed" >&2; exit 1; }; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/build/variants/$name.so $OUT/*.o -lcudart
echo built $ROOT/build/variants/$name.so
