#!/bin/bash
# Quick GPU check: parity subset, then one bench line per environment variant.
#   tools/gpu_ab.sh TAG "VAR=a" "VAR=b" ...   (use "X=0" for the default build)
tag=$1; shift
python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_configs.py tests/test_gpu_reference_behaviour.py tests/test_gpu_multi.py \
    tests/test_blocking_api.py tests/test_gpu_determinism.py -m gpu -q -x > gpurun_out/t_$tag.log 2>&1
echo rc=$? >> gpurun_out/t_$tag.log
i=0
for v in "$@"; do
    env $v python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-api-e2e \
        > gpurun_out/b_${tag}_$i.json 2> gpurun_out/b_${tag}_$i.err
    i=$((i + 1))
done
