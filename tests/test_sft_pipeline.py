"""FPS-SFT receiver branch on the GPU: detections_from_spectrum
(sft.cpp:461-490), sft_detect (sft.cpp:492-500) and run_pipeline's FPS-SFT branch
(pipeline.cpp:97-113) through the C-ABI entry points ofdmr_sft_detections / ofdmr_sft_detect /
ofdmr_pipeline_sft, against
  * the oracle chain on the same c64 inputs (bins and order exact, powers 1e-4, sigma2_used 1e-6),
  * the reference's own run_pipeline (oracle/_ref) on the frames it generates (bins exact).
Scene: fig8-like (config.cpp:358-370: 5 on-grid targets, 16-QAM, SNR 20 dB, FPS-SFT, K = 5) on a
power-of-two grid (1024 x 256, delta-f 240 kHz, N_cp 256) with Doppler bins inside the model's
velocity bound.
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2209_03883_b200 import configs, gen
from paper_2209_03883_b200.receiver import Receiver, SparseSpectrum, detections_from_spectrum, sft_detect

pytestmark = pytest.mark.gpu
C0 = 3.0e8
N, M, DF, FC, NCP, QAM = 1024, 256, 240e3, 77e9, 256, 16
DELAY = [100, 150, 180, 210, 240]
DOPP = [25, -20, 7, 15, -12]
K, PFA, IMAX = 5, 1e-2, 10


def _targets():
    ts = (1.0 + NCP / N) / DF  # WaveformConfig::symbol_time (waveform.hpp:31-35)
    r = [C0 * d / (2.0 * N * DF) for d in DELAY]
    v = [C0 * b / (2.0 * FC * M * ts) for b in DOPP]
    return r, v


def _frames(F, snr=20.0, seed0=19):
    r, v = _targets()
    ys, xs, s2 = [], [], []
    for f in range(F):
        y, x, s = O.ref_make_frame_pair(N, M, DF, FC, NCP, QAM, r, v, snr, seed0 + f)
        ys.append(y)
        xs.append(x)
        s2.append(s)
    return np.stack(ys), np.stack(xs), np.array(s2)


@pytest.fixture(scope="module")
def frames():
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    return _frames(12)


@pytest.mark.parametrize("estimator,noise", [(0, False), (0, True), (1, False)], ids=["ls", "ls-noise", "dftce"])
def test_pipeline_sft_matches_oracle_chain(cuda, frames, estimator, noise):
    y, x, s2 = frames
    F = y.shape[0]
    y64, x64 = y.astype(np.complex64), x.astype(np.complex64)
    seeds = [19 + f for f in range(F)]
    sft_seeds = [gen.derive_seed(s, 0x736674) for s in seeds]
    noise_seeds = [gen.derive_seed(s, 0x6e6573) for s in seeds] if noise else None
    with Receiver(N, M, window="rectangular", estimator=estimator, n_cp=NCP, max_targets=K, pfa=PFA) as rx:
        d = rx.pipeline_sft(y64, x64, s2, sft_seeds, noise_seeds, i_max=IMAX)
        s2u = d.sigma2_h.cpu().numpy()
        assert int(rx.last_status.abs().sum()) == 0
    for f in range(F):
        ref, ref_s2, _ = O.sft_pipeline_frame(y64[f], x64[f], float(s2[f]), estimator, NCP, sft_seeds[f],
                                              noise_seeds[f] if noise else None, IMAX, PFA, K)
        # division noise: fp64 sums (tree vs sequential order); slice estimate: the median |S|^2 of
        # the fp32 channel estimate's slice spectrum (the oracle's H is fp64)
        assert abs(s2u[f] - ref_s2) <= (1e-5 if noise else 1e-9) * ref_s2, (f, s2u[f], ref_s2)
        got = d.frame(f)
        assert [(a, b) for a, b, _ in got] == [(a, b) for a, b, _ in ref], (f, got, ref)
        for (_, _, pg), (_, _, pr) in zip(got, ref):
            assert abs(pg - pr) <= 1e-4 * pr


@pytest.mark.parametrize("noise", [False, True])
def test_pipeline_sft_matches_reference_run_pipeline(cuda, frames, noise):
    # the reference's own run_pipeline(FpsSft) on its complex<double> frames; the GPU reads them as c64
    y, x, s2 = frames
    F = y.shape[0]
    r, v = _targets()
    seeds = [19 + f for f in range(F)]
    with Receiver(N, M, window="rectangular", estimator="ls", n_cp=NCP, max_targets=K, pfa=PFA) as rx:
        d = rx.pipeline_sft(y.astype(np.complex64), x.astype(np.complex64), s2,
                            [gen.derive_seed(s, 0x736674) for s in seeds],
                            [gen.derive_seed(s, 0x6e6573) for s in seeds] if noise else None, i_max=IMAX)
        s2u = d.sigma2_h.cpu().numpy()
    found = 0
    for f in range(F):
        ref, ref_s2u = O.ref_run_pipeline_sft(N, M, DF, FC, NCP, QAM, 0, r, v, 20.0, seeds[f], noise, IMAX, K)
        assert abs(s2u[f] - ref_s2u) <= 1e-5 * ref_s2u, (f, s2u[f], ref_s2u)
        got = d.frame(f)
        assert [(a, b) for a, b, _ in got] == [(a, b) for a, b, _ in ref], (f, got, ref)
        found += sorted((a, b) for a, b, _ in got) == sorted(zip(DELAY, DOPP))
    assert found >= F // 2  # the scene's targets are recovered (sanity of the scene, not parity)


def test_sft_detect_and_detections_from_spectrum(cuda):
    c3 = configs.CFG3
    F = 16
    h, s2, _, _ = gen.sparse_frames(c3.n, c3.m, c3.targets, c3.snr_db, c3.base_seed, 0, F)
    seeds = [gen.derive_seed(c3.base_seed + f, 0x736674) for f in range(F)]
    with Receiver(16, 16, max_targets=c3.max_targets) as rx:
        d = rx.sft_detect(h, seeds, s2, pfa=c3.pfa, i_max=c3.i_max)
        out = rx.sft(h, seeds, s2, i_max=c3.i_max, pfa=c3.pfa, stream_ordered=True)
        assert int(out["status"].abs().sum()) == 0
        d2 = rx.sft_detections(out, c3.n, c3.m, s2, c3.pfa, k_per_frame=np.full(F, 4, np.int32))
    for f in range(F):
        ref = O.sft_iterate(h[f].astype(np.complex128), seeds[f], float(s2[f]), i_max=c3.i_max, pfa=c3.pfa)
        od = O.detections_from_spectrum(ref["entries"], c3.n, c3.m, float(s2[f]), c3.pfa, c3.max_targets)
        assert [(a, b) for a, b, _ in d.frame(f)] == [(a, b) for a, b, _ in od]
        assert [(a, b) for a, b, _ in d2.frame(f)] == [(a, b) for a, b, _ in od[:4]]
        # module-level reference-named functions (single grid)
        if f < 2:
            spec = SparseSpectrum(ref["entries"])
            md = detections_from_spectrum(spec, c3.n, c3.m, float(s2[f]), c3.pfa, c3.max_targets)
            assert [(x.delay_bin, x.doppler_bin, x.peak_power) for x in md] == od
            sd = sft_detect(h[f], seeds[f], float(s2[f]), c3.pfa, c3.max_targets, i_max=c3.i_max)
            assert [(x.delay_bin, x.doppler_bin) for x in sd] == [(a, b) for a, b, _ in od]
