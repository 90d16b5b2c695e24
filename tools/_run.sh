set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "cfg2 or zp or colpass2048 or detect" > gpurun_out/t2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t2_pytest.log
python tools/cfg_rate.py cfg2 256 8 > gpurun_out/t2_cfg2_16.log 2>&1
OFDMR_LIB=$PWD/paper_2209_03883_b200/libofdmr_b200_zp12.so python tools/cfg_rate.py cfg2 256 8 > gpurun_out/t2_cfg2_12.log 2>&1
tail -3 gpurun_out/t2_pytest.log; cat gpurun_out/t2_cfg2_16.log gpurun_out/t2_cfg2_12.log
