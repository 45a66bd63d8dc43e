#!/bin/bash
# compute-sanitizer over tools/sanitize_case.py: memcheck, racecheck (shared
# memory hazards), synccheck (barriers), initcheck.  Logs -> gpurun_out/.
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 $CS --tool $tool --print-limit 50 --error-exitcode 9 python tools/sanitize_case.py \
      > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
done
