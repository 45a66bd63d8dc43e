#!/bin/bash
# quick GPU check: parity subset + a short bench (tag = $1)
tag=${1:-q}
python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_configs.py tests/test_gpu_reference_behaviour.py tests/test_blocking_api.py -m gpu -q -x > gpurun_out/t_$tag.log 2>&1
echo rc=$? >> gpurun_out/t_$tag.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_$tag.json 2> gpurun_out/b_$tag.err
