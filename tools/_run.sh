mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "cfg2 or zp or colpass2048" > gpurun_out/t14.log 2>&1
tail -3 gpurun_out/t14.log
