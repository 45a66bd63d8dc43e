#!/bin/bash
# Round-2 GPU evidence run: smoke, bench (ours + reference arm), full gpu tests, ncu launch list + full capture.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err; echo bench=$?
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
timeout 2400 python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/gputest.log 2>&1; echo tests=$?
bash tools/prof_r02.sh r02a
