"""Grids whose sizes are not powers of two: the reference's default
WaveformConfig / table1 numerology 2048 x 560 (waveform.hpp:21-28, config.cpp:194-207), fig6's
M = 200, the desk numerology 512 x 140 and small odd sizes run on the mixed-radix kernels
(csrc/mixed_kernels.cu: radix 8/4/2/3/5/7/11/13 Stockham passes).  Checked against the oracle on
the same c64 inputs (maps <= 1e-4 of the frame maximum, DFT-CE <= 1e-5 of the peak, detections
bit-exact) and, on the paper's Fig. 8 scene at table1 numerology, against the reference's own
run_pipeline (oracle/_ref)."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2209_03883_b200 import gen
from paper_2209_03883_b200.receiver import ConfigError, Receiver

pytestmark = pytest.mark.gpu


def _noise(n, m, seed):
    return gen.noise_grid(n, m, 1.0, seed).astype(np.complex64)


@pytest.mark.parametrize("n,m,np_,mp,window", [(2048, 560, 2048, 560, 1), (512, 140, 1024, 280, 0),
                                               (200, 96, 256, 200, 1), (105, 49, 105, 49, 0), (64, 48, 64, 48, 1),
                                               (48, 70, 96, 140, 0)])
def test_mixed_periodogram_matches_oracle(cuda, n, m, np_, mp, window):
    F = 3
    h = np.stack([_noise(n, m, 100 + f) for f in range(F)])
    h[1, 5 % n, 7 % m] += 40.0  # a strong cell
    with Receiver(n, m, np_, mp, window=window) as rx:
        p = rx.periodogram(h).cpu().numpy()
    for f in range(F):
        ref = O.periodogram(h[f].astype(np.complex128), window, np_, mp)
        assert np.abs(p[f] - ref).max() <= 1e-4 * ref.max(), (n, m, np_, mp, f)


@pytest.mark.parametrize("n,m,L", [(560, 32, 140), (2048, 560, 512), (105, 20, 26)])
def test_mixed_dft_ce_matches_oracle(cuda, n, m, L):
    h = np.stack([_noise(n, m, 7 + f) for f in range(2)])
    with Receiver(n, m, estimator="dft-ce", n_cp=L) as rx:
        g = rx.dft_ce(h).cpu().numpy()
    for f in range(2):
        ref = O.dft_ce(h[f].astype(np.complex128), L)
        assert np.abs(g[f] - ref).max() <= 1e-5 * np.abs(ref).max()


def test_mixed_detect_on_shared_map_is_exact(cuda):
    # extract_peaks on the same fp32 map (odd M'): selection identical to the oracle's
    rng = np.random.default_rng(3)
    maps = [rng.exponential(1.0, (200, 147)).astype(np.float32) for _ in range(3)]
    with Receiver(200, 147, 200, 147, window="rectangular", max_targets=10) as rx:
        d = rx.extract_peaks(np.stack(maps), np.array([3.0, 4.0, 5.0]))
    for f, pm in enumerate(maps):
        ref = O.extract_peaks(pm.astype(np.float64), [3.0, 4.0, 5.0][f], 10)
        assert [(a, b) for a, b, _ in d.frame(f)] == [(a, b) for a, b, _ in ref]


FIG8_DELAY = [328, 394, 442, 485, 508]
FIG8_DOPP = [45, -37, 7, 25, -22]


def _fig8_targets(n=2048, m=560, df=240e3, ncp=512):
    ts = (1.0 + ncp / n) / df
    return ([3.0e8 * d / (2.0 * n * df) for d in FIG8_DELAY], [3.0e8 * b / (2.0 * 77e9 * m * ts) for b in FIG8_DOPP])


@pytest.mark.parametrize("estimator", [0, 1], ids=["ls", "dft-ce"])
def test_table1_fig8_pipeline_matches_oracle_and_reference(cuda, estimator):
    """config.cpp:358-370 fig8 scene (5 on-bin targets, SNR 20 dB) at the reference's default
    table1 numerology (2048 x 560, 16-QAM, Hamming, N_cp 512, P_fa 1e-2) with the periodogram
    detector: GPU detections equal the oracle's on the same c64 frames and the reference's own
    run_pipeline on its complex<double> frames."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    n, m, df, ncp = 2048, 560, 240e3, 512
    r, v = _fig8_targets()
    F = 4
    frames = [O.ref_make_frame_pair(n, m, df, 77e9, ncp, 16, r, v, 20.0, 19 + f) for f in range(F)]
    y = np.stack([a.astype(np.complex64) for a, _, _ in frames])
    x = np.stack([b.astype(np.complex64) for _, b, _ in frames])
    s2 = np.array([s for _, _, s in frames])
    with Receiver(n, m, n, m, window="hamming", estimator=estimator, n_cp=ncp, max_targets=5) as rx:
        dets, pm = rx.pipeline(y, x, s2, want_map=True)
        pm = pm.cpu().numpy()
        s2h = dets.sigma2_h.cpu().numpy()
    rc = O.rx_config(n, m, n, m, estimator, ncp, 1, 1e-2)
    scn = (n, m, n, m, df, 77e9, ncp, 1, 1e-2, estimator, np.array(r), np.array(v))
    for f in range(F):
        ref, ref_s2h, _, ref_map = O.receive_frame(rc, y[f], x[f], float(s2[f]), 5, want_map=True)
        assert abs(s2h[f] - ref_s2h) <= 1e-6 * ref_s2h
        assert np.abs(pm[f] - ref_map).max() <= 1e-4 * ref_map.max()
        got = [(a, b) for a, b, _ in dets.frame(f)]
        assert got == [(a, b) for a, b, _ in ref], (f, got, ref)
        rd, rv, _, _ = O.ref_run_pipeline_qam(scn, 16, 20.0, 19 + f) if hasattr(O, "ref_run_pipeline_qam") else (
            None, None, None, None)
        if rd is not None:
            assert got == list(zip(rd.tolist(), rv.tolist())), (f, got, rd, rv)
        assert sorted(got) == sorted(zip(FIG8_DELAY, FIG8_DOPP))


def test_mixed_limits_are_config_errors(cuda):
    with pytest.raises(ConfigError):
        Receiver(17 * 19, 32)  # prime factors outside 2, 3, 5, 7, 11, 13
    with Receiver(560, 32, n_cp=16) as rx:
        with pytest.raises(ConfigError):  # N above 4096 on the FPS-SFT path
            rx.sft(torch.zeros(4100, 2, dtype=torch.complex64), [1], [0.1])
        with pytest.raises(ConfigError):  # Q = lcm(N, M) = 4093 x 4091 above 2^20
            rx.sft(torch.zeros(4093, 4091, dtype=torch.complex64), [1], [0.1])
