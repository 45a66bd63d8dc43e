CHR_TRACE_HOST=1 python tools/one_step.py c3 > gpurun_out/trace_host.txt 2>&1
