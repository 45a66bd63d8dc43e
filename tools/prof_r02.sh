set -x
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_r02b.csv python tools/one_step.py c3 > gpurun_out/ncu_launch_r02b.log 2>&1
echo rc1=$?
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_band|k_mc_emit3|k_emit_q2|k_quant_band|k_stats_rows|k_crc_segments" -c 7 -o gpurun_out/top_r02b python tools/one_step.py c3 > gpurun_out/ncu_top_r02b.log 2>&1
echo rc2=$?
