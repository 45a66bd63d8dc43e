#!/bin/bash
# Parity subset on the in-tree build, the decoder error/malformed-stream tests,
# then one bench line per library variant (tools/gpu_variants.sh) -- tag = $1
tag=$1; shift
python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_configs.py tests/test_gpu_reference_behaviour.py \
    tests/test_blocking_api.py tests/test_gpu_determinism.py tests/test_gpu_reference_suite.py -m gpu -q -x > gpurun_out/t_$tag.log 2>&1
echo rc=$? >> gpurun_out/t_$tag.log
bash tools/gpu_variants.sh $tag "$@"
