"""FPS-SFT on grids whose Q = lcm(N, M) is not a power of two <= 2048: the
slice FFT runs Bluestein in the oracle's exact operation order (bit-identical spectra) on
per-frame work arrays in global memory.  Same bar as the power-of-two path: (k, l) lists,
iterations, samples_used and convergence equal to the oracle's, amplitudes <= 1e-4; the
estimate-noise slice median bit-exact; and the paper's Fig. 8 FPS-SFT scene at the reference's
default table1 numerology (2048 x 560, Q = 71680) equal to the reference's own run_pipeline."""
import numpy as np
import pytest

import oracle as O
from paper_2209_03883_b200 import gen
from paper_2209_03883_b200.receiver import Receiver

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,m,k", [(64, 48, 5), (48, 70, 4), (100, 36, 6), (2048, 560, 5)])
def test_sft_general_sizes_match_oracle(cuda, n, m, k):
    F = 6 if n * m < 1e6 else 2
    h, s2, _, _ = gen.sparse_frames(n, m, k, 20.0, 1234, 0, F)
    seeds = [gen.derive_seed(1234 + f, 0x736674) for f in range(F)]
    with Receiver(16, 16) as rx:
        out = rx.sft(h, seeds, s2, i_max=8)
        nz = rx.estimate_noise_from_slice(h, seeds).cpu().numpy()
    kk, ll = out["k"].cpu().numpy(), out["l"].cpu().numpy()
    amp, ne = out["amp"].cpu().numpy(), out["n_entries"].cpu().numpy()
    for f in range(F):
        ref = O.sft_iterate(h[f].astype(np.complex128), seeds[f], float(s2[f]), i_max=8)
        assert int(ne[f]) == ref["n_entries"], (n, m, f)
        got = [(int(kk[f, i]), int(ll[f, i])) for i in range(int(ne[f]))]
        assert got == [(a, b) for a, b, _ in ref["entries"]], (n, m, f)
        ga = amp[f, : int(ne[f]), 0] + 1j * amp[f, : int(ne[f]), 1]
        ra = np.array([a for _, _, a in ref["entries"]])
        assert np.abs(ga - ra).max(initial=0) <= 1e-4 * np.abs(ra).max(initial=1)
        assert int(out["iterations"][f]) == ref["iterations"]
        assert int(out["samples_used"][f]) == ref["samples_used"]
        assert bool(out["converged"][f]) == ref["converged"]
        assert nz[f] == O.estimate_noise_from_slice(h[f].astype(np.complex128), seeds[f])


FIG8_DELAY = [328, 394, 442, 485, 508]
FIG8_DOPP = [45, -37, 7, 25, -22]


@pytest.mark.parametrize("noise", [False, True])
def test_fig8_fps_sft_pipeline_matches_reference(cuda, noise):
    """config.cpp:358-370: table1 numerology, 5 on-bin targets, SNR 20 dB, FPS-SFT detector."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    n, m, df, ncp = 2048, 560, 240e3, 512
    ts = (1.0 + ncp / n) / df
    r = [3.0e8 * d / (2.0 * n * df) for d in FIG8_DELAY]
    v = [3.0e8 * b / (2.0 * 77e9 * m * ts) for b in FIG8_DOPP]
    F = 2
    seeds = [19 + f for f in range(F)]
    frames = [O.ref_make_frame_pair(n, m, df, 77e9, ncp, 16, r, v, 20.0, s) for s in seeds]
    y = np.stack([a.astype(np.complex64) for a, _, _ in frames])
    x = np.stack([b.astype(np.complex64) for _, b, _ in frames])
    s2 = np.array([s for _, _, s in frames])
    with Receiver(n, m, window="hamming", estimator="ls", n_cp=ncp, max_targets=5) as rx:
        d = rx.pipeline_sft(y, x, s2, [gen.derive_seed(s, 0x736674) for s in seeds],
                            [gen.derive_seed(s, 0x6e6573) for s in seeds] if noise else None, i_max=10)
    for f in range(F):
        ref, _ = O.ref_run_pipeline_sft(n, m, df, 77e9, ncp, 16, 0, r, v, 20.0, seeds[f], noise, 10, 5)
        got = [(a, b) for a, b, _ in d.frame(f)]
        assert got == [(a, b) for a, b, _ in ref], (f, got, ref)
        assert sorted(got) == sorted(zip(FIG8_DELAY, FIG8_DOPP))
