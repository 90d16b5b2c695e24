mkdir -p gpurun_out
L=$PWD/paper_2209_03883_b200
python -m pytest tests -m gpu -x -q -k "cfg4 or cfg1 or fused or tile" > gpurun_out/t10.log 2>&1
python tools/fused_rate.py >> gpurun_out/t10.log 2>&1
OFDMR_LIB=$L/libofdmr_b200_tmapf.so python tools/fused_rate.py >> gpurun_out/t10.log 2>&1
python tools/fused_rate.py >> gpurun_out/t10.log 2>&1
OFDMR_LIB=$L/libofdmr_b200_tmapf.so python tools/fused_rate.py >> gpurun_out/t10.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fused_ce -c 2 --csv --log-file gpurun_out/t10_traffic.csv python tools/ce_only.py 8192 2 > /dev/null 2>&1
OFDMR_LIB=$L/libofdmr_b200_tmapf.so ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fused_ce -c 2 --csv --log-file gpurun_out/t10_traffic_pf.csv python tools/ce_only.py 8192 2 > /dev/null 2>&1
cat gpurun_out/t10.log; grep -h fused_ce gpurun_out/t10_traffic.csv gpurun_out/t10_traffic_pf.csv | cut -d, -f13-
