"""GPU parity tests: the CUDA path (through the C-ABI) against the CPU oracle on the
same seeded c64 inputs.  Bars (BASELINE north_star / SURVEY.md §8d):
  * detection bins + order bit-exact (fp32-unresolvable oracle near-ties counted apart),
  * peak powers within 1e-4 relative, whole maps within 1e-4 of the frame maximum,
  * FPS-SFT (k, l) sets bit-exact, amplitudes within 1e-4, iterations / convergence equal.
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2209_03883_b200 import configs, gen
from paper_2209_03883_b200.receiver import ConfigError, Receiver
from tests.parity import classify, powers_close

pytestmark = pytest.mark.gpu
TWO_PI = 6.283185307179586476925286766559
MAP_TOL = 1e-4


def _rc(cfg):
    return O.rx_config(cfg.n, cfg.m, cfg.n_prime, cfg.m_prime, cfg.estimator, cfg.n_cp, cfg.window, cfg.pfa)


def _pipeline_parity(cfg, frames, first=0, check_map=False):
    fb = gen.frames(cfg, first, frames)
    kf = fb.n_targets if cfg.per_frame_k else None
    with Receiver.from_config(cfg) as rx:
        dets, pmap = rx.pipeline(fb.y, fb.x, fb.sigma2, k_per_frame=kf, want_map=True)
        torch.cuda.synchronize()
        pmap = pmap.cpu().numpy()
        s2h = dets.sigma2_h.cpu().numpy()
        # production path (no map requested): the fused single-launch kernel where eligible
        l0 = rx.launch_count
        fdets, _ = rx.pipeline(fb.y, fb.x, fb.sigma2, k_per_frame=kf)
        torch.cuda.synchronize()
        if _fused_eligible(cfg):
            assert rx.launch_count - l0 == 1, "fused kernel expected"
    rc = _rc(cfg)
    stats = {"ok": 0, "tie": 0, "fail": 0}
    for f in range(frames):
        k = int(kf[f]) if kf is not None else cfg.max_targets
        ref, ref_s2h, eta, ref_map = O.receive_frame(rc, fb.y[f], fb.x[f], float(fb.sigma2[f]), k, want_map=True)
        assert abs(s2h[f] - ref_s2h) <= 1e-6 * ref_s2h
        err = np.abs(pmap[f] - ref_map).max() / ref_map.max()
        assert err <= MAP_TOL, (cfg.name, f, err)
        for dd in (dets, fdets):
            got = dd.frame(f)
            verdict = classify(got, ref, ref_map, eta, k)
            stats[verdict] += 1
            assert verdict != "fail", (cfg.name, f, got, ref)
            assert powers_close(got, ref), (got, ref)
    assert stats["tie"] <= max(2, frames // 50), stats
    return stats


def _fused_eligible(cfg):
    return (cfg.n, cfg.m, cfg.n_prime, cfg.m_prime) == (1024, 256, 1024, 256) and cfg.estimator == 1 and 0 < cfg.n_cp <= 128


def test_spectral_division_and_zero_cell(cuda):
    cfg = configs.CFG0
    fb = gen.frames(cfg, 0, 2)
    with Receiver.from_config(cfg) as rx:
        h = rx.spectral_division(fb.y, fb.x).cpu().numpy()
        for f in range(2):
            ref = O.spectral_division(fb.y[f], fb.x[f])
            assert np.abs(h[f] - ref).max() <= 1e-6 * np.abs(ref).max()
        x = fb.x.copy()
        x[1, 5, 7] = 0
        with pytest.raises(ConfigError):
            rx.spectral_division(fb.y, x)


@pytest.mark.parametrize("n,m,L", [(1024, 256, 128), (2048, 512, 256), (64, 16, 16), (256, 64, 0), (128, 32, 128)])
def test_dft_ce_matches_oracle(cuda, n, m, L):
    rng = np.random.default_rng(n + L)
    h = (rng.normal(size=(3, n, m)) + 1j * rng.normal(size=(3, n, m))).astype(np.complex64)
    with Receiver(n, m, estimator="dft-ce", n_cp=L) as rx:
        out = rx.dft_ce(h).cpu().numpy()
    for f in range(3):
        ref = O.dft_ce(h[f].astype(np.complex128), L)
        scale = max(np.abs(ref).max(), 1e-30)
        assert np.abs(out[f] - ref).max() <= 1e-5 * scale if L else np.abs(out[f]).max() == 0


@pytest.mark.parametrize("n,m,np_,mp,window", [
    (1024, 256, 1024, 256, 0), (1024, 256, 1024, 256, 1), (64, 32, 128, 64, 1), (16, 16, 64, 16, 0),
    (128, 64, 512, 128, 1), (2048, 512, 4096, 2048, 1), (1024, 1024, 1024, 1024, 0), (256, 4096, 256, 4096, 0),
])
def test_periodogram_matches_oracle(cuda, n, m, np_, mp, window):
    F = 2
    h = np.stack([gen.noise_grid(n, m, 1.0, 77 + f) for f in range(F)]).astype(np.complex64)
    h[0] += 3.0 * np.exp(1j * TWO_PI * (-np.arange(n)[:, None] * 5 / n + np.arange(m)[None, :] * 3 / m))
    with Receiver(n, m, np_, mp, window=window) as rx:
        p = rx.periodogram(h).cpu().numpy()
    for f in range(F):
        ref = O.periodogram(h[f].astype(np.complex128), window, np_, mp)
        assert np.abs(p[f] - ref).max() / ref.max() <= MAP_TOL


def test_reference_unit_analogues(cuda):
    # DC peak (test_periodogram.cpp:58-67), analytic target (:90-104), two targets (:152-178)
    with Receiver(16, 16, 16, 16, window=0, max_targets=8) as rx:
        p = rx.periodogram(np.ones((16, 16), np.complex64)).cpu().numpy()
        r, c = np.unravel_index(np.argmax(p), p.shape)
        assert r == 0 and c - 8 == 0
    n, m = 64, 32
    k = np.arange(n)[:, None]
    l = np.arange(m)[None, :]
    t1 = np.exp(1j * TWO_PI * (-k * 10 / n + l * 5 / m))
    t2 = np.exp(1j * TWO_PI * (-k * 30 / n + l * (-8) / m))
    with Receiver(n, m, window=0, max_targets=8) as rx:
        p = rx.periodogram((t1 + 0.7 * t2).astype(np.complex64))
        d = rx.extract_peaks(p, 1.0).frame(0)
        assert [(a, b) for a, b, _ in d] == [(10, 5), (30, -8)]
        p1 = rx.periodogram(np.exp(1j * TWO_PI * (-k * 21 / n + l * 9 / m)).astype(np.complex64)).cpu().numpy()
        r, c = np.unravel_index(np.argmax(p1), p1.shape)
        assert r == 21 and c - m // 2 == 9


def test_extract_peaks_small_map_rejected(cuda):
    from paper_2209_03883_b200.receiver import extract_peaks

    with pytest.raises(ConfigError):
        extract_peaks(np.ones((8, 32), np.float32), 0.5, 3)
    got = extract_peaks(np.pad(np.ones((1, 1), np.float32), ((5, 10), (7, 8))), 0.5, 3)
    assert [(d.delay_bin, d.doppler_bin) for d in got] == [(5, 7 - 8)]


def test_detect_on_shared_map_is_exact(cuda):
    # extract_peaks on the SAME fp32 map: GPU selection must equal the oracle's exactly
    cfg = configs.CFG1
    fb = gen.frames(cfg, 0, 4)
    rc = _rc(cfg)
    maps, etas, refs = [], [], []
    for f in range(4):
        _, s2h, eta, pm = O.receive_frame(rc, fb.y[f], fb.x[f], float(fb.sigma2[f]), 3, want_map=True)
        pm32 = pm.astype(np.float32)
        maps.append(pm32)
        etas.append(eta)
        refs.append(O.extract_peaks(pm32.astype(np.float64), eta, 16))
    with Receiver.from_config(cfg.replace(max_targets=16)) as rx:
        d = rx.extract_peaks(np.stack(maps), np.array(etas))
        for f in range(4):
            got = d.frame(f)
            assert [(a, b) for a, b, _ in got] == [(a, b) for a, b, _ in refs[f]]
            assert all(float(np.float32(w)) == pytest.approx(wr, rel=1e-7) for (_, _, w), (_, _, wr) in zip(got, refs[f]))


def test_pipeline_cfg0(cuda):
    _pipeline_parity(configs.CFG0, 1)


def test_pipeline_cfg1(cuda):
    _pipeline_parity(configs.CFG1, 16)


def test_pipeline_cfg1_rect_shortcut(cuda):
    # rectangular window + N' = N takes the exact DFT-CE collapse (G has only L rows)
    _pipeline_parity(configs.CFG1.replace(window=0), 8)


def test_pipeline_cfg4_subset(cuda):
    _pipeline_parity(configs.CFG4, 64, first=1000)


def test_pipeline_cfg2_zc_precoded(cuda):
    _pipeline_parity(configs.CFG2, 2)


def test_pipeline_host_equals_device_and_deterministic(cuda):
    cfg = configs.CFG4
    fb = gen.frames(cfg, 0, 40)
    with Receiver.from_config(cfg, chunk_frames=16) as rx:
        d1, _ = rx.pipeline(fb.y, fb.x, fb.sigma2, k_per_frame=fb.n_targets)
        d2, _ = rx.pipeline(fb.y, fb.x, fb.sigma2, k_per_frame=fb.n_targets)
        hd, hv, hp, hc = rx.pipeline_host(fb.y, fb.x, fb.sigma2, fb.n_targets)
    for a, b in ((d1.delay_bin, d2.delay_bin), (d1.doppler_bin, d2.doppler_bin), (d1.peak_power, d2.peak_power)):
        assert torch.equal(a, b)
    assert (d1.delay_bin.cpu().numpy() == hd).all() and (d1.doppler_bin.cpu().numpy() == hv).all()
    assert (d1.peak_power.cpu().numpy() == hp).all() and (d1.counts.cpu().numpy() == hc).all()


def test_pipeline_zero_cell_raises(cuda):
    cfg = configs.CFG0
    fb = gen.frames(cfg, 0, 1)
    x = fb.x.copy()
    x[0, 100, 3] = 0
    with Receiver.from_config(cfg) as rx:
        with pytest.raises(ConfigError):
            rx.pipeline(fb.y, x, fb.sigma2)
        with pytest.raises(ConfigError):
            rx.pipeline_host(fb.y, x, fb.sigma2)


def test_pipeline_zero_cell_raises_on_fused_path(cuda):
    # the fused DFT-CE kernel flags abnormal |x|^2 for exact recompute (status bit 1); the exact
    # path then raises the zero-cell ConfigError (estimation.cpp:17)
    cfg = configs.CFG4
    fb = gen.frames(cfg, 0, 3)
    x = fb.x.copy()
    x[1, 700, 200] = 0
    with Receiver.from_config(cfg) as rx:
        with pytest.raises(ConfigError):
            rx.pipeline(fb.y, x, fb.sigma2, k_per_frame=fb.n_targets)
        with pytest.raises(ConfigError):
            rx.pipeline_host(fb.y, x, fb.sigma2, fb.n_targets)


@pytest.mark.parametrize("cfg", [configs.CFG4, configs.CFG0], ids=["fused", "ls"])
def test_denormal_and_huge_x_cells_are_divided_not_rejected(cuda, cfg):
    # estimation.cpp:17 rejects only an exactly zero x cell; a denormal x (|x|^2 underflows fp32)
    # or a huge one (|x|^2 overflows fp32) is divided like the reference's complex<double>
    fb = gen.frames(cfg, 0, 2)
    y, x = fb.y.copy(), fb.x.copy()
    x[0, 100, 3] = np.complex64(1e-39 + 0.5e-39j)   # fp32 denormals
    y[0, 100, 3] = x[0, 100, 3] * np.complex64(0.5 - 0.25j)
    x[1, 5, 7] = np.complex64(3e19 - 1e19j)           # |x|^2 ~ 1e39 > FLT_MAX
    y[1, 5, 7] = x[1, 5, 7] * np.complex64(0.3 + 0.1j)
    kf = fb.n_targets if cfg.per_frame_k else None
    rc = _rc(cfg)
    with Receiver.from_config(cfg) as rx:
        dets, _ = rx.pipeline(y, x, fb.sigma2, k_per_frame=kf)  # no ConfigError
        s2h = dets.sigma2_h.cpu().numpy()
        hd, hv, hp, hc = rx.pipeline_host(y, x, fb.sigma2, kf)
        h = rx.spectral_division(y, x).cpu().numpy()
    assert h[0, 100, 3] == pytest.approx(0.5 - 0.25j, rel=1e-6)
    assert h[1, 5, 7] == pytest.approx(0.3 + 0.1j, rel=1e-6)
    for f in range(2):
        k = int(kf[f]) if kf is not None else cfg.max_targets
        ref, ref_s2h, _, _ = O.receive_frame(rc, y[f], x[f], float(fb.sigma2[f]), k)
        assert abs(s2h[f] - ref_s2h) <= 1e-6 * ref_s2h, (f, s2h[f], ref_s2h)
        assert [(a, b) for a, b, _ in dets.frame(f)] == [(a, b) for a, b, _ in ref]
        assert [(int(hd[f, i]), int(hv[f, i])) for i in range(int(hc[f]))] == [(a, b) for a, b, _ in ref]


@pytest.mark.parametrize("f0,F", [(0, 8), (100, 64)])
def test_sft_cfg3_subset_matches_oracle(cuda, f0, F):
    # 64 more frames (512 slope draws): the lattice decode's shortcut over long solution
    # progressions (even slopes with a large power of two) is taken many times
    c3 = configs.CFG3
    h, s2, tk, tl = gen.sparse_frames(c3.n, c3.m, c3.targets, c3.snr_db, c3.base_seed, f0, F)
    seeds = np.array([gen.derive_seed(c3.base_seed + f0 + f, 0x736674) for f in range(F)], np.uint64)
    with Receiver(16, 16) as rx:
        out = rx.sft(h, seeds, s2, i_max=c3.i_max, pfa=c3.pfa, decimation=c3.decimation)
        torch.cuda.synchronize()
    k = out["k"].cpu().numpy()
    l = out["l"].cpu().numpy()
    amp = out["amp"].cpu().numpy()
    ne = out["n_entries"].cpu().numpy()
    for f in range(F):
        ref = O.sft_iterate(h[f].astype(np.complex128), int(seeds[f]), float(s2[f]), i_max=c3.i_max,
                            pfa=c3.pfa, decimation=c3.decimation)
        assert int(ne[f]) == ref["n_entries"]
        got = [(int(k[f, i]), int(l[f, i])) for i in range(int(ne[f]))]
        assert got == [(a, b) for a, b, _ in ref["entries"]]
        ga = amp[f, : int(ne[f]), 0] + 1j * amp[f, : int(ne[f]), 1]
        ra = np.array([a for _, _, a in ref["entries"]])
        assert np.abs(ga - ra).max(initial=0) <= 1e-4 * np.abs(ra).max(initial=1)
        assert int(out["iterations"][f]) == ref["iterations"]
        assert int(out["samples_used"][f]) == ref["samples_used"]
        assert bool(out["converged"][f]) == ref["converged"]


def test_sft_small_grids_match_oracle(cuda):
    rng = np.random.default_rng(5)
    F, n, m = 16, 64, 32
    hs = []
    for f in range(F):
        a = np.arange(n)[:, None]
        b = np.arange(m)[None, :]
        h = sum((0.5 + rng.random()) * np.exp(1j * TWO_PI * (a * rng.integers(n) / n + b * rng.integers(m) / m + rng.random()))
                for _ in range(4))
        h = h + 0.05 * (rng.normal(size=(n, m)) + 1j * rng.normal(size=(n, m)))
        hs.append(h)
    h = np.stack(hs).astype(np.complex64)
    seeds = np.arange(F, dtype=np.uint64) + 11
    s2 = np.full(F, 0.005)
    with Receiver(16, 16) as rx:
        out = rx.sft(h, seeds, s2, i_max=10)
    for f in range(F):
        ref = O.sft_iterate(h[f].astype(np.complex128), int(seeds[f]), 0.005, i_max=10)
        ne = int(out["n_entries"][f])
        assert ne == ref["n_entries"]
        got = [(int(out["k"][f, i]), int(out["l"][f, i])) for i in range(ne)]
        assert got == [(a, b) for a, b, _ in ref["entries"]]


def test_cpp_shim_against_reference_sources(cuda):
    """examples/shim_vs_reference: a reference C++ caller switched to ofdmradar::b200::
    (include/ofdmradar_b200.hpp) reproduces the reference's own receiver functions."""
    import subprocess
    from pathlib import Path

    exe = Path(__file__).resolve().parents[1] / "examples" / "_bin" / "shim_vs_reference"
    if not exe.exists():
        pytest.skip("integration example not built (needs the reference tree at build time)")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


def test_fused_candidate_overflow_recomputed_exactly(cuda):
    """sigma2 far below the noise floor puts eta near 0, so almost every strict local
    maximum is a candidate (> 1024 per half-frame): the fused kernel flags status bit 1 and
    the wrapper recomputes on the general path; results must still match the oracle."""
    cfg = configs.CFG1.replace(max_targets=8)
    fb = gen.frames(cfg, 0, 3)
    s2 = np.full(3, 1e-12)
    with Receiver.from_config(cfg) as rx:
        dets, _ = rx.pipeline(fb.y, fb.x, s2)
        torch.cuda.synchronize()
        hd, hv, hp, hc = rx.pipeline_host(fb.y, fb.x, s2)
    rc = _rc(cfg)
    for f in range(3):
        ref, _, eta, ref_map = O.receive_frame(rc, fb.y[f], fb.x[f], 1e-12, 8, want_map=True)
        got = dets.frame(f)
        assert classify(got, ref, ref_map, eta, 8) != "fail", (got, ref)
        assert [(int(a), int(b)) for a, b in zip(hd[f][: hc[f]], hv[f][: hc[f]])] == [(a, b) for a, b, _ in got]


@pytest.mark.parametrize("window", [1, 0])
def test_fused_tile_boundary_peaks(cuda, window):
    """Targets whose periodogram peaks sit on the fused kernel's tile and CTA boundaries
    (Doppler columns = 0, 7, 8, 15 mod 16, i.e. the columns whose 3x3 test needs the partner
    CTA's edge columns, incl. the wrap 255 <-> 0), in adjacent pairs of near-equal power
    one column apart, and rows shifted by -1/0/+1 so the deciding neighbour is in every
    position of the partner column.  Fused (no map) detections must match the oracle."""
    # K below the number of planted targets: every reported peak is a target peak (weak
    # sidelobe/noise maxima far below the frame maximum are not resolvable to 1e-4 in fp32)
    cfg = configs.CFG1.replace(window=window, max_targets=8, per_frame_k=False)
    n, m = cfg.n, cfg.m
    rng = np.random.default_rng(7)
    frames = 12
    x = np.exp(1j * (np.pi / 2) * rng.integers(0, 4, (frames, n, m)) + 1j * np.pi / 4).astype(np.complex64)
    nn = np.arange(n)[:, None]
    mm = np.arange(m)[None, :]
    y = np.empty_like(x)
    for f in range(frames):
        h = np.zeros((n, m), np.complex128)
        for j in range(10):
            c = int(rng.choice([7, 15])) + 16 * int(rng.integers(0, 16))  # left column of the pair
            d = int(rng.integers(2, 120))
            for side, cc in enumerate((c, (c + 1) % m)):
                dd = d + (int(rng.integers(-1, 2)) if side else 0)
                amp = 1.0 + 0.02 * rng.standard_normal()
                h += amp * np.exp(-2j * np.pi * nn * dd / n) * np.exp(2j * np.pi * mm * (cc - m // 2) / m)
        noise = 0.05 * (rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m))) / np.sqrt(2)
        y[f] = (x[f] * h + noise).astype(np.complex64)
    s2 = np.full(frames, 0.05 ** 2)
    rc = _rc(cfg)
    with Receiver.from_config(cfg) as rx:
        l0 = rx.launch_count
        dets, _ = rx.pipeline(y, x, s2)
        torch.cuda.synchronize()
        assert rx.launch_count - l0 == 1
    hits = 0
    for f in range(frames):
        ref, _, eta, ref_map = O.receive_frame(rc, y[f], x[f], float(s2[f]), cfg.max_targets, want_map=True)
        got = dets.frame(f)
        assert classify(got, ref, ref_map, eta, cfg.max_targets) != "fail", (f, got, ref)
        assert powers_close(got, ref)
        hits += sum(1 for _, b, _ in ref if (b + m // 2) % 16 in (0, 7, 8, 15))
    assert hits >= frames * 3  # the boundary columns really were exercised


@pytest.mark.parametrize("window", [0, 1])
def test_fused_periodogram_many_frames_per_cluster(cuda, window, monkeypatch):
    """More frames than co-resident clusters (each cluster loops over several frames, G
    reused): every frame of the fused single-launch periodogram must match the ticketed
    persistent kernel, and sampled frames the oracle."""
    n, m, F = 1024, 256, 96
    rng = np.random.default_rng(11)
    h = (rng.standard_normal((F, n, m)) + 1j * rng.standard_normal((F, n, m))).astype(np.complex64)
    with Receiver(n, m, window=window) as rx:
        l0 = rx.launch_count
        p = rx.periodogram(h).cpu().numpy()
        assert rx.launch_count - l0 == 1
        monkeypatch.setenv("OFDMR_PG_PERSIST", "1")
        q = rx.periodogram(h).cpu().numpy()
    for f in range(F):
        assert np.abs(p[f] - q[f]).max() / q[f].max() <= MAP_TOL, f
    for f in (0, 41, F - 1):
        ref = O.periodogram(h[f].astype(np.complex128), window, n, m)
        assert np.abs(p[f] - ref).max() / ref.max() <= MAP_TOL


def test_fused_full_batch_position_independent(cuda):
    """cfg4 at the bench's full size: 256 distinct frames tiled to 8192 (every cluster runs
    ~55 software-pipelined rounds).  Size-independent property: every copy of a frame gets
    bit-identical detections wherever it sits in the batch; sampled frames match the oracle."""
    cfg = configs.CFG4
    pool, F = 256, 8192
    fb = gen.frames(cfg, 0, pool)
    reps = F // pool
    y = torch.from_numpy(fb.y).cuda().repeat(reps, 1, 1)
    x = torch.from_numpy(fb.x).cuda().repeat(reps, 1, 1)
    s2 = torch.from_numpy(np.tile(fb.sigma2, reps)).cuda()
    kf = torch.from_numpy(np.tile(fb.n_targets, reps).astype(np.int32)).cuda()
    with Receiver.from_config(cfg) as rx:
        l0 = rx.launch_count
        dets, _ = rx.pipeline(y, x, s2, k_per_frame=kf)
        torch.cuda.synchronize()
        assert rx.launch_count - l0 == 1
    d = dets.delay_bin.cpu().numpy().reshape(reps, pool, -1)
    v = dets.doppler_bin.cpu().numpy().reshape(reps, pool, -1)
    p = dets.peak_power.cpu().numpy().reshape(reps, pool, -1)
    c = dets.counts.cpu().numpy().reshape(reps, pool)
    for arr in (d, v, p, c):
        assert (arr == arr[0:1]).all()
    rc = _rc(cfg)
    for f in range(0, pool, 8):
        k = int(fb.n_targets[f])
        ref, _, eta, ref_map = O.receive_frame(rc, fb.y[f], fb.x[f], float(fb.sigma2[f]), k, want_map=True)
        got = dets.frame(f)
        assert classify(got, ref, ref_map, eta, k) != "fail", (f, got, ref)
        assert powers_close(got, ref)


def _ulp_dist(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    ia = a.view(np.int32).astype(np.int64)
    ib = b.view(np.int32).astype(np.int64)
    ia = np.where(ia < 0, np.int64(-(2**31)) - ia, ia)
    ib = np.where(ib < 0, np.int64(-(2**31)) - ib, ib)
    return np.abs(ia - ib)


@pytest.mark.parametrize("cfg", [configs.CFG4, configs.CFG0, configs.CFG4.replace(qam=16, snr_lo_db=0.0, snr_hi_db=0.0)],
                         ids=["cfg4", "cfg0", "cfg4_16qam"])
def test_gpu_generator_matches_cpu_generator(cuda, cfg):
    """§8(f) item 1: the device generator reproduces the CPU generator (which is bit-exact with
    the reference's make_random_frame / apply_channel, tests/test_oracle_pins.py): symbols,
    scene and σ² exactly; y to at most 1 ulp of c64 in rare cells (fp64 sin/cos/log differ
    between the GPU and glibc in the last bit)."""
    F, first = 12, 5
    ref = gen.frames(cfg, first, F)
    d = gen.frames_device(cfg, first, F)
    assert d["regenerated_on_cpu"] == 0
    torch.cuda.synchronize()
    x = d["x"].cpu().numpy()
    y = d["y"].cpu().numpy()
    assert np.array_equal(x, ref.x)
    assert np.array_equal(d["n_targets"].cpu().numpy(), ref.n_targets)
    assert np.array_equal(d["ranges"].cpu().numpy(), ref.ranges)
    assert np.array_equal(d["vels"].cpu().numpy(), ref.vels)
    assert np.array_equal(d["snr_db"].cpu().numpy(), ref.snr_db)
    s2 = d["sigma2"].cpu().numpy()
    assert np.all(np.abs(s2 - ref.sigma2) <= 4e-16 * ref.sigma2), (s2, ref.sigma2)
    u = _ulp_dist(y.view(np.float32), ref.y.view(np.float32))
    assert u.max() <= 2, u.max()
    assert (u > 0).mean() <= 1e-3, (u > 0).mean()


@pytest.mark.parametrize("window,F", [(0, 5), (1, 300)])
def test_fused_periodogram_matches_two_pass_kernel(cuda, window, F, monkeypatch):
    """The split-exchange periodogram (fused_pg3, default at 1024 x 256) against the previous
    warp-specialised kernel (fused_pg2, OFDMR_PG2) on every frame: fewer frames than frame
    groups, and many frames per group (double-buffered G reused ~16 times)."""
    n, m = 1024, 256
    rng = np.random.default_rng(5 + F)
    base = (rng.standard_normal((min(F, 37), n, m)) + 1j * rng.standard_normal((min(F, 37), n, m))).astype(np.complex64)
    h = np.concatenate([base] * (-(-F // len(base))))[:F] * np.linspace(0.5, 2.0, F, dtype=np.float32)[:, None, None]
    with Receiver(n, m, window=window) as rx:
        p = rx.periodogram(h).cpu().numpy()
        monkeypatch.setenv("OFDMR_PG2", "1")
        q = rx.periodogram(h).cpu().numpy()
    for f in range(F):
        assert np.abs(p[f] - q[f]).max() / q[f].max() <= MAP_TOL, f
    ref = O.periodogram(h[F - 1].astype(np.complex128), window, n, m)
    assert np.abs(p[F - 1] - ref).max() / ref.max() <= MAP_TOL


@pytest.mark.parametrize("n,m,np_,mp,window", [(1024, 256, 1024, 256, 1), (64, 32, 128, 64, 0), (2048, 512, 4096, 2048, 1),
                                               (16, 16, 16, 16, 0)])
def test_estimate_noise_power(cuda, n, m, np_, mp, window):
    """estimate_noise_power (periodogram.cpp:146-152): the radix select returns exactly the
    nth_element order statistic P[count/2] of the device map (bit-exact sigma2 from it), and
    matches the oracle's fp64 estimate on its own map."""
    F = 2 if np_ * mp > 2**20 else 5
    h = np.stack([gen.noise_grid(n, m, 0.3 + f, 300 + f) for f in range(F)]).astype(np.complex64)
    pf = O.power_factor(window, n, m)
    with Receiver(n, m, np_, mp, window=window) as rx:
        p = rx.periodogram(h)
        s2 = rx.estimate_noise_power(p).cpu().numpy()
        pz = torch.zeros_like(p[:1])
        assert rx.estimate_noise_power(pz).cpu().numpy()[0] == 0.0
        pc = torch.full_like(p[:1], 0.25)  # all ties
        assert rx.estimate_noise_power(pc).cpu().numpy()[0] == 0.25 / 0.6931471805599453 / pf
    p = p.cpu().numpy()
    mid = np_ * mp // 2
    for f in range(F):
        v = float(np.partition(p[f].ravel(), mid)[mid])
        assert s2[f] == v / 0.6931471805599453 / pf, f
        ref = O.estimate_noise_power(O.periodogram(h[f].astype(np.complex128), window, np_, mp), pf)
        assert abs(s2[f] - ref) <= 1e-4 * ref, (f, s2[f], ref)


def test_pipeline_estimate_noise_mode(cuda):
    """run_pipeline with detector.estimate_noise (pipeline.cpp:86-87) on LS frames (cfg0 and a
    Hamming variant): the threshold from the estimated noise; detections equal the oracle
    composition on the same frames (periodogram -> estimate_noise_power -> threshold ->
    extract_peaks).  (With DFT-CE the median cell is an algebraic zero, so the estimate is
    fp roundoff in both implementations and is not compared.)"""
    _estimate_noise_parity(configs.CFG0)
    _estimate_noise_parity(configs.CFG0.replace(window=1, snr_lo_db=0.0, snr_hi_db=0.0))


def _estimate_noise_parity(cfg):
    fb = gen.frames(cfg, 0, 8)
    with Receiver.from_config(cfg) as rx:
        dets, pm = rx.pipeline(fb.y, fb.x, fb.sigma2, want_map=True, estimate_noise=True)
        s2e = dets.sigma2_h.cpu().numpy()
    pfac = O.power_factor(cfg.window, cfg.n, cfg.m)
    for f in range(8):
        h = O.spectral_division(fb.y[f].astype(np.complex128), fb.x[f].astype(np.complex128))
        ref_map = O.periodogram(h, cfg.window, cfg.n_prime, cfg.m_prime)
        ref_s2 = O.estimate_noise_power(ref_map, pfac)
        assert abs(s2e[f] - ref_s2) <= 1e-4 * ref_s2
        eta = O.detection_threshold(ref_s2, cfg.pfa, pfac)
        ref = O.extract_peaks(ref_map, eta, cfg.max_targets)
        got = dets.frame(f)
        assert classify(got, ref, ref_map, eta, cfg.max_targets) != "fail", (f, got, ref)
        assert powers_close(got, ref)


@pytest.mark.parametrize("n,m,ncp", [(1024, 256, 128), (2048, 16, 256), (4096, 16, 1024), (16, 16, 0), (64, 16, 64),
                                     (256, 32, 7), (560, 28, 140), (2048, 20, 512), (200, 16, 50)])
def test_ofdm_front_end_matches_oracle(cuda, n, m, ncp):
    """§8(f) item 3, the OFDM time-domain front end (waveform.cpp:133-166): GPU ofdm_modulate
    and ofdm_demodulate against the oracle restatement on identical c64 inputs (fp32 FFT:
    1e-5 of the frame's peak magnitude), the modulate -> demodulate round trip, batching."""
    F = 3
    rng = np.random.default_rng(n + m + ncp)
    x = (rng.standard_normal((F, n, m)) + 1j * rng.standard_normal((F, n, m))).astype(np.complex64)
    noise = (0.05 * (rng.standard_normal((F, m, n + ncp)) + 1j * rng.standard_normal((F, m, n + ncp))))
    with Receiver(n, m, n_cp=ncp, window="rectangular") as rx:
        st = rx.ofdm_modulate(x)
        assert tuple(st.shape) == (F, m, n + ncp)
        st_np = st.cpu().numpy()
        noisy = (st_np + noise).astype(np.complex64)
        gr = rx.ofdm_demodulate(noisy).cpu().numpy()
        rt = rx.ofdm_demodulate(st).cpu().numpy()
        single = rx.ofdm_demodulate(noisy[1].reshape(-1)).cpu().numpy()
        with pytest.raises(ConfigError):
            rx.ofdm_demodulate(noisy[:, :, 1:])
        with pytest.raises(ConfigError):
            rx.ofdm_modulate(x[:, :, 1:])
    for f in range(F):
        ref_st = O.ofdm_modulate(x[f].astype(np.complex128), ncp)
        assert np.abs(st_np[f] - ref_st).max() <= 1e-5 * np.abs(ref_st).max()
        ref_gr = O.ofdm_demodulate(noisy[f].astype(np.complex128), n, m, ncp)
        assert np.abs(gr[f] - ref_gr).max() <= 1e-5 * np.abs(ref_gr).max()
        assert np.abs(rt[f] - x[f]).max() <= 1e-5 * np.abs(x[f]).max()
    assert np.array_equal(single, gr[1])


def test_ofdm_cp_longer_than_symbol_rejected(cuda):
    with Receiver(64, 16, n_cp=65, window="rectangular") as rx:
        with pytest.raises(ConfigError):
            rx.ofdm_modulate(np.zeros((64, 16), np.complex64))


def test_map_to_pgm_matches_reference_writer(cuda, tmp_path):
    """§8(f) item 4: write_map_pgm pixels (io.cpp:94-110) computed on the GPU for a batch of
    device maps equal the host restatement byte for byte, and (where the reference's writer
    library was built) the reference's own file for the same map."""
    from paper_2209_03883_b200 import io as W
    n, m = 1024, 256
    h = np.stack([gen.noise_grid(n, m, 1.0, 900 + f) for f in range(3)]).astype(np.complex64)
    h[1] += 4.0 * np.exp(1j * TWO_PI * (-np.arange(n)[:, None] * 9 / n + np.arange(m)[None, :] * 5 / m))
    with Receiver(n, m, window=1) as rx:
        p = rx.periodogram(h)
        p[2] = 0.0  # degenerate map: peak 0 -> 1 (io.cpp:99)
        px = rx.map_to_pgm(p).cpu().numpy()
    pn = p.cpu().numpy()
    for f in range(3):
        assert np.array_equal(px[f], W.pgm_pixels(pn[f])), f
    W.write_pgm_bytes(tmp_path / "g.pgm", px[1])
    if O.REF_IO_SO.exists():
        pd = np.ascontiguousarray(pn[1], np.float64)
        assert O.ref_io().ref_write_map_pgm(pd.ctypes.data, n, m, str(tmp_path / "r.pgm").encode()) == 0
        assert (tmp_path / "g.pgm").read_bytes() == (tmp_path / "r.pgm").read_bytes()


@pytest.mark.parametrize("cfg,F", [(configs.CFG2.replace(n=256, m=64, n_prime=512, m_prime=128, n_cp=32), 6),
                                   (configs.CFG2, 1)], ids=["zc256x64", "cfg2"])
def test_gpu_generator_zc_precoded(cuda, cfg, F):
    """§8(f) item 1, ZC precode (zadoffchu.cpp:58-87,133-136, D = N): the device generator's
    fp64 x -> Z x -> channel path against the CPU generator.  The ZC matrix uses the GPU's
    sincos, so precoded cells may differ in the last c64 bit; symbols' scene, counts exact."""
    ref = gen.frames(cfg, 3, F)
    d = gen.frames_device(cfg, 3, F)
    assert d["regenerated_on_cpu"] == 0
    torch.cuda.synchronize()
    assert np.array_equal(d["n_targets"].cpu().numpy(), ref.n_targets)
    assert np.array_equal(d["snr_db"].cpu().numpy(), ref.snr_db)
    s2 = d["sigma2"].cpu().numpy()
    assert np.all(np.abs(s2 - ref.sigma2) <= 1e-12 * ref.sigma2), (s2, ref.sigma2)
    for name, got, want in (("x", d["x"].cpu().numpy(), ref.x), ("y", d["y"].cpu().numpy(), ref.y)):
        u = _ulp_dist(got.view(np.float32), want.view(np.float32))
        assert u.max() <= 4, (name, u.max())
        assert (u > 0).mean() <= 0.05, (name, (u > 0).mean())


@pytest.mark.parametrize("n,m", [(64, 32), (1024, 1024), (256, 16), (16, 2048)])
def test_sft_estimate_noise_from_slice(cuda, n, m):
    """estimate_noise_from_slice (pipeline.cpp:26-43): same host slope draws, the oracle's
    radix-2 FFT schedule in fp64 and an exact median, so the GPU value equals the oracle's
    bit for bit on identical c64 grids (the oracle itself is pinned to the reference's
    run_pipeline sigma2_used, tests/golden/sft_noise_*.npz)."""
    F = 4
    h = np.stack([gen.noise_grid(n, m, 0.5 + f, 40 + f) for f in range(F)]).astype(np.complex64)
    seeds = np.array([O.derive_seed(7 + f, 0x6E6573) for f in range(F)], np.uint64)
    with Receiver(16, 16) as rx:
        got = rx.estimate_noise_from_slice(h, seeds).cpu().numpy()
    for f in range(F):
        ref = O.estimate_noise_from_slice(h[f].astype(np.complex128), int(seeds[f]))
        assert got[f] == ref, (f, got[f], ref)


@pytest.mark.parametrize("variant", ["dft_ce_L201", "ls_rect"])
def test_pipeline_cfg2_column_variants(cuda, variant):
    """cfg2's register-FFT column pass (colpass2048.cu) off its default: an odd tap count L = 201
    (part of the last tap block masked) and the plain LS estimator with a rectangular window."""
    if variant == "dft_ce_L201":
        cfg = configs.CFG2.replace(n_cp=201)
    else:
        cfg = configs.CFG2.replace(estimator=configs.EST_LS, window=configs.WINDOW_RECT)
    _pipeline_parity(cfg, 2)


def test_colpass2048_matches_generic_column_pass(cuda, monkeypatch):
    """The cfg2 column pass (warp FFT_1024 chain) against the generic shared-memory Stockham
    column pass (OFDMR_COL2048=0) on the same 6 ZC-precoded frames: maps, sigma_h^2, detections."""
    cfg = configs.CFG2
    fb = gen.frames(cfg, 20, 6)
    with Receiver.from_config(cfg) as rx:
        d1, p1 = rx.pipeline(fb.y, fb.x, fb.sigma2, want_map=True)
        monkeypatch.setenv("OFDMR_COL2048", "0")
        d0, p0 = rx.pipeline(fb.y, fb.x, fb.sigma2, want_map=True)
        torch.cuda.synchronize()
    p0, p1 = p0.cpu().numpy(), p1.cpu().numpy()
    for f in range(6):
        assert np.abs(p1[f] - p0[f]).max() <= 2e-5 * p0[f].max(), f
        assert [(a, b) for a, b, _ in d1.frame(f)] == [(a, b) for a, b, _ in d0.frame(f)], f
    s1, s0 = d1.sigma2_h.cpu().numpy(), d0.sigma2_h.cpu().numpy()
    # colpass2048 forms 1/|x|^2 with rcp.approx and sums runs of 16 terms in fp32 (as the fused
    # kernels do); the generic pass divides in IEEE fp32 and sums in fp64
    assert np.abs(s1 - s0).max() <= 1e-7 * s0.max()


def test_pipeline_cfg2_zero_cell_raises(cuda):
    cfg = configs.CFG2
    fb = gen.frames(cfg, 0, 2)
    x = fb.x.copy()
    x[1, 1500, 300] = 0
    with Receiver.from_config(cfg) as rx:
        with pytest.raises(ConfigError):
            rx.pipeline(fb.y, x, fb.sigma2)


def test_rowpass_zp_matches_generic_rowpass(cuda):
    # cfg2's zero-padded row pass (rowpass_zp.cu: 4 x FFT_512 per row, K <= 8) against the generic
    # shared-memory row pass (taken for K > 8) on the same 12 ZC-precoded frames
    cfg = configs.CFG2
    fb = gen.frames(cfg, 0, 12)
    with Receiver.from_config(cfg) as rx:
        d8, _ = rx.pipeline(fb.y, fb.x, fb.sigma2)
    with Receiver.from_config(cfg.replace(max_targets=9)) as rx:
        d9, _ = rx.pipeline(fb.y, fb.x, fb.sigma2)
    for f in range(12):
        a, b = d8.frame(f), d9.frame(f)[:8]
        assert [(x, y) for x, y, _ in a] == [(x, y) for x, y, _ in b]
        assert all(abs(p - q) <= 1e-4 * q for (_, _, p), (_, _, q) in zip(a, b))


@pytest.mark.parametrize("n,np_,window,L", [(64, 64, configs.WINDOW_RECT, 16), (128, 256, configs.WINDOW_HAMMING, 32)])
def test_rowpass_zp_other_delay_sizes(cuda, n, np_, window, L):
    # rowpass_zp (M = 512 -> M' = 2048, K <= 8) behind the generic column pass: the DFT-CE shortcut's
    # all-zero rows (rect, N' = N), a last row block shorter than 14 rows, and a 1/(N M) that is not
    # an even power of two (scale kept out of the twiddles)
    cfg = configs.CFG1.replace(name="zp-small", n=n, m=512, n_prime=np_, m_prime=2048, n_cp=L, window=window,
                               max_targets=4, snr_lo_db=5.0, snr_hi_db=5.0)
    _pipeline_parity(cfg, 2)


def test_rowpass_zp_full_scan_fallback(cuda):
    # a threshold far below the noise floor puts more cells above eta than the tile's candidate
    # list holds: rowpass_zp falls back to its full scan; same frames through the generic row pass
    cfg = configs.CFG2
    fb = gen.frames(cfg, 0, 3)
    s2 = fb.sigma2 * 1e-3
    with Receiver.from_config(cfg) as rx:
        d8, _ = rx.pipeline(fb.y, fb.x, s2)
    with Receiver.from_config(cfg.replace(max_targets=9)) as rx:
        d9, _ = rx.pipeline(fb.y, fb.x, s2)
    for f in range(3):
        a, b = d8.frame(f), d9.frame(f)[:8]
        assert len(a) == 8
        assert [(x, y) for x, y, _ in a] == [(x, y) for x, y, _ in b]
        assert all(abs(p - q) <= 1e-4 * q for (_, _, p), (_, _, q) in zip(a, b))


@pytest.mark.parametrize("window", [0, 1])
def test_fused_periodogram_many_frames_on_device(cuda, window, monkeypatch):
    """1000 frames (~55 per 8-CTA frame group: each double-buffered G buffer reused ~27 times,
    the discard -> release ordering exercised on every frame) against the previous kernel,
    compared on the device."""
    import torch
    n, m, F = 1024, 256, 1000
    g = torch.Generator(device="cuda").manual_seed(11 + window)
    h = torch.randn(F, n, m, dtype=torch.complex64, device="cuda", generator=g)
    h *= torch.linspace(0.5, 2.0, F, device="cuda")[:, None, None]
    with Receiver(n, m, window=window) as rx:
        p = rx.periodogram(h)
        monkeypatch.setenv("OFDMR_PG2", "1")
        q = rx.periodogram(h)
    err = ((p - q).abs().amax(dim=(1, 2)) / q.amax(dim=(1, 2))).max().item()
    assert err <= MAP_TOL, err


def test_sft_concurrent_host_threads(cuda):
    """Two host threads, one receiver each, run FPS-SFT at the same time (the per-frame draws
    share one persistent host worker pool): results equal the sequential ones."""
    import threading
    c3 = configs.CFG3
    F = 32
    h, s2, _, _ = gen.sparse_frames(c3.n, c3.m, c3.targets, c3.snr_db, c3.base_seed, 0, F)
    seeds = np.array([gen.derive_seed(c3.base_seed + f, 0x736674) for f in range(F)], np.uint64)

    def run(out, idx):
        with Receiver(16, 16) as rx:
            o = rx.sft(h, seeds, s2, i_max=c3.i_max, pfa=c3.pfa, decimation=c3.decimation)
            torch.cuda.synchronize()
            out[idx] = (o["k"].cpu().numpy(), o["l"].cpu().numpy(), o["n_entries"].cpu().numpy())

    seq = {}
    run(seq, 0)
    par = {}
    ts = [threading.Thread(target=run, args=(par, i)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for i in range(2):
        for a, b in zip(par[i], seq[0]):
            assert np.array_equal(a, b)
