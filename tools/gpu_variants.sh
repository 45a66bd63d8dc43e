#!/bin/bash
# One bench line per library variant (build/variants/<name>.so; "base" = the in-tree build)
tag=$1; shift
for v in "$@"; do
    if [ "$v" = base ]; then lp=""; else lp="CHR_LIB_PATH=$PWD/build/variants/$v.so"; fi
    env $lp python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-api-e2e \
        > gpurun_out/v_${tag}_$v.json 2> gpurun_out/v_${tag}_$v.err
done
