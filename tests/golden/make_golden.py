"""Regenerate the golden fixtures in tests/golden/ from the REFERENCE'S OWN SOURCES.

Runs only where /root/reference exists (this container): it drives
oracle/_ref/libofdmref.so (reference src/*.cpp + substitute FFT, built by
`make -f oracle/Makefile ref`) on seeded inputs and stores inputs + outputs as small
.npz files.  The GPU box never reads /root/reference; tests load these fixtures.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import ctypes as C
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle as O  # noqa: E402
from paper_2209_03883_b200 import _native, gen  # noqa: E402
from paper_2209_03883_b200.configs import RadarConfig  # noqa: E402

OUT = Path(__file__).resolve().parent
TWO_PI = 6.283185307179586476925286766559


def p(a):
    return a.ctypes.data


def periodogram_fixtures(R):
    rng = np.random.default_rng(2209)
    cases = [(16, 8, 16, 8, 0), (64, 32, 128, 64, 1), (48, 20, 48, 40, 1), (37, 11, 74, 11, 0), (128, 64, 128, 64, 1)]
    for i, (n, m, np_, mp, w) in enumerate(cases):
        h = rng.normal(size=(n, m)) + 1j * rng.normal(size=(n, m))
        h = np.ascontiguousarray(h)
        out = np.empty((np_, mp))
        assert R.ref_periodogram(p(h), n, m, w, np_, mp, p(out)) == 0
        np.savez_compressed(OUT / f"periodogram_{i}.npz", kind="periodogram", h=h, window=w, n_prime=np_,
                            m_prime=mp, p=out)


def dft_ce_fixture(R):
    rng = np.random.default_rng(3883)
    n, m, L = 64, 24, 16
    h = np.ascontiguousarray(rng.normal(size=(n, m)) + 1j * rng.normal(size=(n, m)))
    out = np.empty_like(h)
    assert R.ref_dft_ce(p(h), p(out), n, m, L) == 0
    np.savez_compressed(OUT / "dft_ce_0.npz", kind="dft_ce", h=h, n_cp=L, out=out)


def receive_fixtures(R):
    # small grids through the reference receiver half of run_pipeline (pipeline.cpp:72-96)
    cases = [
        ("receive_ls_rect", RadarConfig("g0", 128, 32, 128, 32, 32, 4, 0, 0, 3, 4, 3, 3, 10.0, 10.0, range_hi=60.0)),
        ("receive_dftce_hamming_pad", RadarConfig("g1", 128, 32, 256, 64, 16, 16, 1, 1, 4, 4, 2, 5, -5.0, 15.0,
                                                  range_hi=60.0)),
    ]
    for name, cfg in cases:
        fb = gen.frames(cfg, 0, cfg.frames, threads=1)
        F, K = cfg.frames, cfg.max_targets
        d = np.zeros((F, K), np.int64)
        v = np.zeros((F, K), np.int64)
        w = np.zeros((F, K))
        cnt = np.zeros(F, np.int64)
        s2h = np.zeros(F)
        for f in range(F):
            c = C.c_long()
            s = C.c_double()
            e = C.c_double()
            dd = np.zeros(K, np.int64)
            vv = np.zeros(K, np.int64)
            ww = np.zeros(K)
            rc = R.ref_receive_frame(cfg.n, cfg.m, cfg.n_prime, cfg.m_prime, cfg.estimator, cfg.n_cp, cfg.window,
                                     cfg.pfa, p(fb.y[f]), p(fb.x[f]), float(fb.sigma2[f]), K, p(dd), p(vv), p(ww),
                                     C.byref(c), C.byref(s), C.byref(e), None)
            assert rc == 0
            d[f], v[f], w[f], cnt[f], s2h[f] = dd, vv, ww, c.value, s.value
        cfgv = np.array([cfg.n, cfg.m, cfg.n_prime, cfg.m_prime, cfg.estimator, cfg.n_cp, cfg.window], np.int64)
        np.savez_compressed(OUT / f"{name}.npz", kind="receive", cfg=cfgv, pfa=cfg.pfa, k=K, y=fb.y, x=fb.x,
                            sigma2=fb.sigma2, delay=d, doppler=v, power=w, count=cnt, s2h=s2h)


def sft_fixture(R):
    rng = np.random.default_rng(4455)
    n, m, F = 64, 48, 4
    hs, seeds, s2s = [], [], []
    for f in range(F):
        truth = []
        uk, ul = set(), set()
        while len(truth) < 5:
            k, l = int(rng.integers(n)), int(rng.integers(m))
            if k in uk or l in ul:
                continue
            uk.add(k)
            ul.add(l)
            truth.append((k, l, (0.5 + 1.5 * rng.random()) * np.exp(1j * TWO_PI * rng.random())))
        a = np.arange(n)[:, None]
        b = np.arange(m)[None, :]
        h = sum(A * np.exp(1j * TWO_PI * (a * k / n + b * l / m)) for k, l, A in truth)
        s2 = 0.01 * f
        h = h + np.sqrt(s2 / 2) * (rng.normal(size=(n, m)) + 1j * rng.normal(size=(n, m)))
        hs.append(np.ascontiguousarray(h))
        seeds.append(1000 + f)
        s2s.append(s2)
    ME = 64
    out = {k: [] for k in ("ek", "el", "ea_re", "ea_im", "n_entries", "residual", "converged", "iterations",
                           "samples_used")}
    for f in range(F):
        ek = np.zeros(ME, np.int64)
        el = np.zeros(ME, np.int64)
        ar = np.zeros(ME)
        ai = np.zeros(ME)
        ne = C.c_int64()
        res = C.c_double()
        conv = C.c_int32()
        its = C.c_int64()
        su = C.c_int64()
        rc = R.ref_sft_iterate(p(hs[f]), n, m, 8, 0.0, seeds[f], s2s[f], 1e-2, 8, 0.25, 0.35, ME, p(ek), p(el), p(ar),
                               p(ai), C.byref(ne), C.byref(res), C.byref(conv), C.byref(its), C.byref(su))
        assert rc == 0
        for k, v in (("ek", ek), ("el", el), ("ea_re", ar), ("ea_im", ai), ("n_entries", ne.value),
                     ("residual", res.value), ("converged", conv.value), ("iterations", its.value),
                     ("samples_used", su.value)):
            out[k].append(v)
    np.savez_compressed(OUT / "sft_64x48.npz", kind="sft", h=np.stack(hs), seed=np.array(seeds, np.uint64),
                        sigma2=np.array(s2s), i_max=8, **{k: np.array(v) for k, v in out.items()})


def frame_fixture(R):
    # generator pin: reference make_random_frame + apply_channel (validity-checked targets)
    n, m, ncp = 128, 32, 32
    df = 491.5e6 / 1024
    ranges = np.array([10.0, 25.5, 33.3])
    vels = np.array([3.0, -5.5, 7.25])
    y = np.empty((n, m), np.complex128)
    x = np.empty((n, m), np.complex128)
    s2 = C.c_double()
    rc = R.ref_make_frame_pair(n, m, df, 77e9, ncp, 16, p(ranges), p(vels), 3, 5.0, 4242, p(y), p(x), C.byref(s2))
    assert rc == 0, rc
    np.savez_compressed(OUT / "frame_gen_0.npz", kind="frame", n=n, m=m, n_cp=ncp, df=df, qam=16, ranges=ranges,
                        vels=vels, snr_db=5.0, seed=4242, y=y, x=x, sigma2=s2.value)


def ofdm_fixtures(R):
    """ofdm_modulate / ofdm_demodulate (waveform.cpp:133-166) on seeded grids / streams."""
    rng = np.random.default_rng(1333)
    for i, (n, m, ncp) in enumerate([(64, 12, 16), (256, 6, 0), (48, 5, 12)]):
        x = np.ascontiguousarray(rng.normal(size=(n, m)) + 1j * rng.normal(size=(n, m)))
        stream = np.empty((m, n + ncp), np.complex128)
        assert R.ref_ofdm_modulate(p(x), n, m, ncp, p(stream)) == 0
        noisy = np.ascontiguousarray(stream + 0.1 * (rng.normal(size=stream.shape) + 1j * rng.normal(size=stream.shape)))
        grid = np.empty((n, m), np.complex128)
        assert R.ref_ofdm_demodulate(p(noisy), n, m, ncp, p(grid)) == 0
        np.savez_compressed(OUT / f"ofdm_{i}.npz", kind="ofdm", x=x, n_cp=ncp, stream=stream, noisy=noisy, grid=grid)


def noise_fixtures(R):
    """estimate_noise_power (periodogram.cpp:146-152): maps with odd/even counts and ties."""
    rng = np.random.default_rng(146)
    maps = [rng.exponential(size=(32, 16)), rng.exponential(size=(7, 9)),
            np.round(rng.exponential(size=(16, 16)) * 4) / 4, np.zeros((8, 8))]
    for i, mp_ in enumerate(maps):
        mp_ = np.ascontiguousarray(mp_)
        pf = 0.3968 if i % 2 else 1.0
        s2 = R.ref_estimate_noise_power(p(mp_), mp_.shape[0], mp_.shape[1], pf)
        np.savez_compressed(OUT / f"noise_{i}.npz", kind="noise", p=mp_, pf=pf, sigma2=s2)


def io_fixture():
    """The reference's own writers (io.cpp:28-110, oracle/_ref/libofdmref_io.so) on a small map
    with zeros, sub-floor cells and a wide dynamic range, and on a detection list."""
    import tempfile
    W = O.ref_io()
    rng = np.random.default_rng(28)
    pm = rng.exponential(size=(16, 8)) * 10.0 ** rng.uniform(-40, 3, size=(16, 8))
    pm[0, 0] = 0.0
    pm[3, 5] = 1e-290
    pm = np.ascontiguousarray(pm)
    d = np.array([328, 1, 17], np.int64)
    v = np.array([45, -1, -128], np.int64)
    pw = np.array([12.5, 3.3e-7, 0.0])
    rg = np.array([100.0982666015625, 0.30517578125, 5.18798828125])
    vl = np.array([30.057, -0.6679, -85.5])
    with tempfile.TemporaryDirectory() as td:
        files = {}
        assert W.ref_write_map_csv(p(pm), 16, 8, f"{td}/map.csv".encode()) == 0
        assert W.ref_write_map_pgm(p(pm), 16, 8, f"{td}/map.pgm".encode()) == 0
        assert W.ref_write_detections_csv(p(d), p(v), p(pw), p(rg), p(vl), 3, f"{td}/det.csv".encode()) == 0
        for k in ("map.csv", "map.pgm", "det.csv"):
            files[k] = np.frombuffer(open(f"{td}/{k}", "rb").read(), np.uint8)
    np.savez_compressed(OUT / "io_0.npz", kind="io", p=pm, d=d, v=v, pw=pw, rg=rg, vl=vl, map_csv=files["map.csv"],
                        map_pgm=files["map.pgm"], det_csv=files["det.csv"])


def sft_noise_fixtures(R):
    """run_pipeline with the FPS-SFT detector in estimate-noise mode: the reference's
    sigma2_used and the channel estimate it came from (estimate_noise_from_slice is internal
    to pipeline.cpp, so it is pinned through run_pipeline)."""
    cases = [(64, 32, 16, 2, 10.0, 77), (48, 20, 12, 1, 0.0, 1234), (128, 64, 32, 3, -5.0, 99)]
    for i, (n, m, ncp, cnt, snr, seed) in enumerate(cases):
        df = 491.5e6 / n
        ranges = np.array([1.0, 2.5, 3.3][:cnt])
        vels = np.array([3.0, -5.5, 7.25][:cnt])
        h = np.empty((n, m), np.complex128)
        s2 = C.c_double()
        assert R.ref_sft_noise_case(n, m, df, 77e9, ncp, p(ranges), p(vels), cnt, snr, seed, p(h), C.byref(s2)) == 0
        np.savez_compressed(OUT / f"sft_noise_{i}.npz", kind="sft_noise", h=h, seed=seed, sigma2=s2.value)


MANIFEST_CASES = [
    # (command, seed, n, m, df, fc, ncp, qam, np, mp, window, pfa, est, det, K, est_noise, i_max,
    #  ranges, vels, phases, snr, extra, wall_ms)
    ("run", 7, 1024, 256, 491.5e6 / 1024, 77e9, 256, 4, 1024, 256, 0, 0.01, 0, 0, 3, 0, 10,
     [100.0, 31.25], [30.0, -12.5], None, 10.0, [], 12.5),
    ("rmse", 20220908, 2048, 512, 491.5e6 / 2048, 77e9, 256, 16, 4096, 2048, 1, 1e-05, 1, 1, 8, 1, 8,
     [5.5], [-80.0], [0.25], float("inf"), [("snr_db", "-10:20:5"), ("trials", "200")], 123456.789),
]


def manifest_fixtures():
    import tempfile
    W = O.ref_io()
    for i, c in enumerate(MANIFEST_CASES):
        (cmd, seed, n, m, df, fc, ncp, qam, np_, mp, win, pfa, est, det, K, en, imax, rg, vl, ph, snr, extra,
         wall) = c
        rg_a = np.ascontiguousarray(rg, np.float64)
        vl_a = np.ascontiguousarray(vl, np.float64)
        ph_a = np.ascontiguousarray(ph, np.float64) if ph is not None else None
        ks = (C.c_char_p * max(1, len(extra)))(*[k.encode() for k, _ in extra])
        vs = (C.c_char_p * max(1, len(extra)))(*[v.encode() for _, v in extra])
        with tempfile.TemporaryDirectory() as td:
            path = f"{td}/run.json"
            rc = W.ref_write_run_manifest(path.encode(), cmd.encode(), seed, n, m, df, fc, ncp, qam, np_, mp, win, pfa,
                                          est, det, K, en, imax, p(rg_a), p(vl_a),
                                          p(ph_a) if ph_a is not None else None, len(rg), snr, ks, vs, len(extra),
                                          wall)
            assert rc == 0
            data = np.frombuffer(open(path, "rb").read(), np.uint8)
        np.savez_compressed(OUT / f"manifest_{i}.npz", kind="manifest", case=i, run_json=data)


if __name__ == "__main__":
    R = O.ref()
    periodogram_fixtures(R)
    dft_ce_fixture(R)
    receive_fixtures(R)
    sft_fixture(R)
    frame_fixture(R)
    ofdm_fixtures(R)
    noise_fixtures(R)
    io_fixture()
    sft_noise_fixtures(R)
    manifest_fixtures()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)
