cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_estimators.py tests/test_montecarlo.py tests/test_gpu_parity.py -x -q -m gpu -k "estimators or partial or small_map or rmse or generator" 2>&1 | tail -15
python -c "
from paper_2209_03883_b200 import configs
from paper_2209_03883_b200.estimators import bench_estimators
B=configs.CFG0.replace(n=2048, n_prime=2048, m=256, m_prime=256, qam=16, window=1)
for r in bench_estimators(B, [256,512,1024,2048], 5, 5, 13, snr_db=40.0, batch=256, bandwidth_hz=60e6): print(r)
"
