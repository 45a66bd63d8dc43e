#!/bin/bash
# Diagnostic: k_band per-tile phase timestamps (decode.cu CHR_BAND_TRACE build)
# for one c3 step; writes gpurun_out/band_trace.bin (8 u64 per tile).
set -e
D=paper_2408_05462_b200/csrc
O=/tmp/trlib; mkdir -p $O
for f in $D/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC \
       --expt-relaxed-constexpr -DCHR_BAND_TRACE -c $f -o $O/$(basename $f .cu).o &
done
for f in $D/*.cpp; do g++ -O2 -fPIC -std=c++17 -ffp-contract=off -c $f -o $O/$(basename $f .cpp).o & done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $O/libchr.so $O/*.o -lcudart
CHR_LIB_PATH=$O/libchr.so CHR_BAND_TRACE_FILE=gpurun_out/band_trace.bin python tools/one_step.py c3
