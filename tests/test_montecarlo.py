"""§8(f) item 2, Monte-Carlo callers: the host-side reduction of paper_2209_03883_b200.montecarlo
(bins_to_physics, resolutions, match_detections, the RMSE rows) pinned against the reference's
own rmse_sweep (metrics.cpp:92-120, oracle/_ref) on detections produced by the reference's own
run_pipeline — CPU only, small grid."""
import numpy as np
import pytest

import oracle as O
from paper_2209_03883_b200 import configs, gen
from paper_2209_03883_b200 import montecarlo as mc

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def _small_cfg():
    return configs.CFG1.replace(n=64, m=32, n_prime=64, m_prime=32, n_cp=16, max_targets=3)


def _scenario(cfg, ranges, vels):
    return (cfg.n, cfg.m, cfg.n_prime, cfg.m_prime, cfg.df_hz, 77e9, cfg.n_cp, cfg.window, cfg.pfa, cfg.estimator,
            ranges, vels)


def test_rmse_reduction_matches_reference_rmse_sweep():
    cfg = _small_cfg()
    ranges = np.array([1.0, 2.2, 3.7])
    vels = np.array([-900.0, 300.0, 1200.0])  # within the model's ICI bound (0.1 c df / 2 fc)
    scn = _scenario(cfg, ranges, vels)
    grid = [-5.0, 5.0, 20.0]
    trials, seed = 6, 424242
    ref_rows = O.ref_rmse_sweep(scn, grid, trials, seed)
    res = mc.resolutions(cfg)
    truths = list(zip(ranges.tolist(), vels.tolist()))
    for si, snr in enumerate(grid):
        stats = mc.MatchStats()
        for t in range(trials):
            d, v, r, vel = O.ref_run_pipeline(scn, snr, gen.derive_seed(seed, t))
            phys = [mc.bins_to_physics(int(a), int(b), cfg) for a, b in zip(d, v)]
            # our fp64 physics is the reference's, bit for bit
            assert [p[0] for p in phys] == list(r) and [p[1] for p in phys] == list(vel)
            mc.match_detections(phys, truths, res, stats)
        row = mc.finish_row(snr, "dft-ce", stats, trials)
        assert (row.range_rmse_m, row.velocity_rmse_mps, row.miss_rate) == tuple(ref_rows[si]), (row, ref_rows[si])


def test_match_detections_penalties():
    cfg = _small_cfg()
    res = mc.resolutions(cfg)
    st = mc.MatchStats()
    mc.match_detections([], [(1.0, 0.0), (2.0, 0.0)], res, st)
    pen_r, pen_v = res["cp_range_limit_m"], res["unambiguous_velocity_mps"] / 2.0
    assert st.misses == 2 and st.truths == 2
    assert st.sum_sq_range == 2 * pen_r * pen_r and st.sum_sq_velocity == 2 * pen_v * pen_v


@pytest.mark.gpu
def test_gpu_rmse_sweep_matches_reference(cuda):
    """GPU generator + fused pipeline + host reduction against the reference's rmse_sweep on
    the cfg1 numerology (1024 x 256, DFT-CE L = 128, Hamming), targets inside the CP range."""
    cfg = configs.CFG1
    ranges = np.array([8.0, 17.5, 31.0])
    vels = np.array([-35.0, 12.0, 60.0])
    grid = [-15.0, -5.0, 5.0]
    trials, seed = 24, 777
    rows = mc.rmse_sweep(cfg, ranges, vels, grid, trials, seed)
    ref_rows = O.ref_rmse_sweep(_scenario(cfg, ranges, vels), grid, trials, seed)
    for row, ref in zip(rows, ref_rows):
        got = np.array([row.range_rmse_m, row.velocity_rmse_mps, row.miss_rate])
        # frames are c64 and the receiver fp32 on the GPU path: identical detections give
        # identical rows; a near-tie flip in one of the 72 truths moves a row by < 1 / 72
        assert np.allclose(got, ref, rtol=1e-9, atol=0), (row, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("estimator", [0, 1], ids=["ls", "dft-ce"])
def test_gpu_mse_sweep_matches_reference(cuda, estimator):
    """mse_sweep (metrics.cpp:122-143): GPU generator true channel (c128) vs GPU estimate_channel
    (fp32 on c64 frames) against the reference's fp64 sweep.  The fp32 estimate error
    (~1e-7 of |H|) is far below the estimation noise being measured: rtol 1e-4."""
    cfg = configs.CFG1.replace(estimator=estimator)
    ranges = np.array([8.0, 17.5, 31.0])
    vels = np.array([-35.0, 12.0, 60.0])
    grid = [-10.0, 0.0, 20.0]
    trials, seed = 6, 99
    rows = mc.mse_sweep(cfg, ranges, vels, grid, trials, seed)
    ref = O.ref_mse_sweep(_scenario(cfg, ranges, vels), grid, trials, seed)
    got = np.array([r.channel_mse for r in rows])
    assert np.allclose(got, ref, rtol=1e-4, atol=0), (got, ref)


@pytest.mark.gpu
def test_gpu_rmse_sweep_partial_batches_match_reference(cuda):
    """Several batches per SNR point, the last one partial (batch 5, 24 trials): the cross-SNR
    two-slot pipelining of rmse_sweep (the host matches batch j - 1 while the GPU generates and
    receives batch j, across SNR boundaries) gives the reference's rows."""
    cfg = configs.CFG1
    ranges = np.array([8.0, 17.5, 31.0])
    vels = np.array([-35.0, 12.0, 60.0])
    grid = [-15.0, 5.0]
    trials, seed = 24, 777
    rows = mc.rmse_sweep(cfg, ranges, vels, grid, trials, seed, batch=5)
    ref_rows = O.ref_rmse_sweep(_scenario(cfg, ranges, vels), grid, trials, seed)
    for row, ref in zip(rows, ref_rows):
        got = np.array([row.range_rmse_m, row.velocity_rmse_mps, row.miss_rate])
        assert np.allclose(got, ref, rtol=1e-9, atol=0), (row, ref)
