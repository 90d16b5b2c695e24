cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_sft_general.py tests/test_gpu_parity.py tests/test_sft_pipeline.py -x -q -m gpu -k "sft or general or fig8" 2>&1 | tail -25
python tools/sft_rate.py 2>&1 | tail -2
