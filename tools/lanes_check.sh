for l in 1 2 3; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-api-e2e --lanes $l > gpurun_out/lanes_$l.json 2> gpurun_out/lanes_$l.err; done
python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-api-e2e > gpurun_out/lanes_c4.json 2> gpurun_out/lanes_c4.err
python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-api-e2e > gpurun_out/lanes_c5.json 2> gpurun_out/lanes_c5.err
python -m pytest tests/test_gpu_reference_suite.py -q -m gpu > gpurun_out/refsuite.log 2>&1; echo rc=$? >> gpurun_out/refsuite.log
