mkdir -p gpurun_out
L=$PWD/paper_2209_03883_b200
OFDMR_LIB=$L/libofdmr_b200_tt0.so python tools/phase_timing.py 4096 > gpurun_out/t12.log 2>&1
OFDMR_LIB=$L/libofdmr_b200_tt2.so python tools/phase_timing.py 4096 >> gpurun_out/t12.log 2>&1
cat gpurun_out/t12.log
