#!/bin/bash
# ncu --set full of selected kernels in one bench step: tools/ncu_kern.sh TAG REGEX [COUNT]
tag=$1; rx=$2; cnt=${3:-2}
ncu --set full --import-source on --clock-control none -k regex:"$rx" -c $cnt -o gpurun_out/$tag \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_$tag.log 2>&1
echo ncu_rc=$? >> gpurun_out/ncu_$tag.log
