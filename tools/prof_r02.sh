#!/bin/bash
# Round-2 profile set (c3, one pipeline step between cudaProfilerStart/Stop):
#   launch list with per-kernel DRAM bytes, then --set full of the top kernels.
# tools/prof_r02.sh TAG
tag=${1:-r02}
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/launches_$tag.csv python tools/one_step.py c3 \
    > gpurun_out/ncu_launch_$tag.log 2>&1
echo rc1=$?
ncu --set full --import-source on --clock-control none --profile-from-start off \
    -k regex:"k_band|k_mc_emit4|k_mc_count4|k_emit_q2|k_quant_band|k_stats_rows|k_crc_segments|k_tok_fast|k_seg_locate|k_summarize2" \
    -c 12 -o gpurun_out/top_$tag python tools/one_step.py c3 > gpurun_out/ncu_top_$tag.log 2>&1
echo rc2=$?
