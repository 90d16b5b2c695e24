"""GPU bench_estimators (metrics.cpp:145-253, paper_2209_03883_b200/estimators.py) against the
reference's own harness (oracle/_ref): same scenes (targets from Rng(derive_seed(seed, N))), same
frames, both detectors agree on the support (the harness raises otherwise), the recovered support
is the scene's on-bin targets, and FPS-SFT's samples_used equals the reference's.  fig6 numerology
(B = 60 MHz, 16-QAM, Hamming, SNR 40 dB, K = 5, seed 13) with M = 256 (the GPU path takes powers of
two)."""
import pytest

import oracle as O
from paper_2209_03883_b200 import configs
from paper_2209_03883_b200.estimators import _targets, _with_df, bench_estimators

pytestmark = pytest.mark.gpu
SIZES = [256, 512, 1024, 2048]
BASE = configs.CFG0.replace(n=2048, n_prime=2048, m=256, m_prime=256, qam=16, window=1)
B = 60e6


def test_bench_estimators_matches_reference_harness(cuda):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    rows = bench_estimators(BASE, SIZES, 5, 3, 13, snr_db=40.0, batch=64, bandwidth_hz=B)
    ref = O.ref_bench_estimators(2048, 256, B / 2048, 77e9, 16, 1, BASE.pfa, 40.0, SIZES, 5, 1, 13)
    for r, (n, _, _, _, su) in zip(rows, ref):
        assert r.n == n
        assert r.samples_used == su, (n, r.samples_used, su)
        cfg = BASE.replace(n=n, n_prime=n, n_cp=n // 4)
        _, _, truth = _targets(_with_df(cfg, B / n), 5, 13)
        assert r.support == sorted(truth), (n, r.support, truth)
        assert r.periodogram_ms > 0 and r.sft_ms > 0
