#!/bin/bash
# Full GPU test suite (as the driver runs it) -> gpurun_out/gputest_$1.log
tag=${1:-t}
timeout 3000 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/gputest_$tag.log 2>&1
echo rc=$? >> gpurun_out/gputest_$tag.log
