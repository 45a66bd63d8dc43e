#!/bin/bash
# Round-2 GPU evidence run (tag $1): smoke, bench as the driver runs it (ours + reference arm), c4/c5 lines,
# full gpu tests, ncu launch list + --set full of the top kernels (tools/prof_r02.sh).
tag=${1:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$tag.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo smoke=$?
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo bench=$?
python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-api-e2e > gpurun_out/bench_c4_$tag.json 2> gpurun_out/bench_c4_$tag.err; echo c4=$?
python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-api-e2e > gpurun_out/bench_c5_$tag.json 2> gpurun_out/bench_c5_$tag.err; echo c5=$?
python bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err; echo ref=$?
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/gputest_$tag.log 2>&1; echo tests=$? | tee -a gpurun_out/gputest_$tag.log
bash tools/prof_r02.sh $tag
