"""Every frame of every BASELINE config through the CUDA path (C-ABI) against the CPU oracle.

VERDICT r01 "Next round" item 1 / SURVEY.md §8d parity rules:
  cfg0  1 frame      LS, rectangular, top-3
  cfg1  64 frames    DFT-CE L=128, Hamming, top-3           (+ every map within 1e-4 of max)
  cfg2  256 frames   ZC-precoded 2048x512 -> 4096x2048, top-8 (+ every map within 1e-4 of max)
  cfg3  1024 frames  FPS-SFT 1024x1024: (k, l), amplitudes, iterations, samples, convergence;
                     plus the reference's bench_estimators support check (metrics.cpp:220-231):
                     the SFT detections' support equals the 1024x1024 periodogram top-10's
  cfg4  8192 frames  exactly the bench's GPU-generated batch (bench.py: gen.frames_device(cfg4, 0, 8192))

Detections must be bit-exact in bins and order; a difference is accepted only as an
"fp32-unresolvable tie" when the oracle's own fp64 margin at the deciding comparison is
< 1e-5 relative (tests/parity.py), and every tie is recorded with its margin.  Peak powers
within 1e-4 relative, sigma_h^2 within 1e-6.  Set OFDMR_PARITY_REPORT=path to write the
per-config ok/tie/fail report (profiles/parity_r02.json is one such run).
"""
from __future__ import annotations

import concurrent.futures as cf
import json
import os
import time

import numpy as np
import pytest
import torch

import oracle as O
from paper_2209_03883_b200 import configs, gen
from paper_2209_03883_b200.receiver import Receiver
from tests.parity import POWER_REL, classify_detail

pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 1
MAP_TOL = 1e-4
REPORT: dict = {}


def _write_report():
    path = os.environ.get("OFDMR_PARITY_REPORT")
    if not path:
        return
    REPORT["_meta"] = {"gpu": torch.cuda.get_device_name(0), "host_threads": THREADS, "base_seed": 20220908,
                       "tie_rule": "oracle fp64 margin < 1e-5 relative at the deciding comparison",
                       "power_tol": POWER_REL, "map_tol": MAP_TOL}
    d = os.path.dirname(path)
    if d:
        os.makedirs(d, exist_ok=True)
    with open(path, "w") as f:
        json.dump(REPORT, f, indent=1, sort_keys=True)


def _rc(cfg):
    return O.rx_config(cfg.n, cfg.m, cfg.n_prime, cfg.m_prime, cfg.estimator, cfg.n_cp, cfg.window, cfg.pfa)


def _compare_dets(cfg, name, stats, f_global, got, ref, ref_s2h, gpu_s2h, y, x, s2, k):
    """One frame: bins/order (tie-classified on the oracle's fp64 map), powers, sigma_h^2."""
    assert abs(gpu_s2h - ref_s2h) <= 1e-6 * ref_s2h, (name, f_global, gpu_s2h, ref_s2h)
    rd = {(a, b): w for a, b, w in ref}
    for a, b, w in got:
        if (a, b) in rd:
            assert abs(w - rd[(a, b)]) <= POWER_REL * rd[(a, b)], (name, f_global, (a, b), w, rd[(a, b)])
    if [(a, b) for a, b, _ in got] == [(a, b) for a, b, _ in ref]:
        stats["ok"] += 1
        return
    _, _, eta, pmap = O.receive_frame(_rc(cfg), y, x, s2, k, want_map=True)
    verdict, margin, why = classify_detail(got, ref, pmap, eta, k)
    stats[verdict] += 1
    stats.setdefault("cases", []).append({"frame": int(f_global), "verdict": verdict, "fp64_margin": margin,
                                          "why": why, "gpu": [(a, b) for a, b, _ in got],
                                          "oracle": [(a, b) for a, b, _ in ref]})
    assert verdict != "fail", (name, f_global, why, got, ref)


def _pipeline_all(cfg, name, y, x, s2, kf, chunk, check_maps=False):
    """GPU pipeline over all frames (device tensors y, x, s2, kf), oracle on host copies."""
    F = y.shape[0]
    stats = {"frames": F, "ok": 0, "tie": 0, "fail": 0, "overflow_recomputed": 0, "zero_cell": 0}
    rc = _rc(cfg)
    K = cfg.max_targets
    t_gpu = t_orc = 0.0
    max_map_err = 0.0
    with Receiver.from_config(cfg) as rx:
        for c0 in range(0, F, chunk):
            c1 = min(F, c0 + chunk)
            kk = kf[c0:c1] if kf is not None else None
            t0 = time.perf_counter()
            dets, pm = rx.pipeline(y[c0:c1], x[c0:c1], s2[c0:c1], k_per_frame=kk, want_map=check_maps)
            st = rx.last_status.cpu().numpy()
            torch.cuda.synchronize()
            t_gpu += time.perf_counter() - t0
            stats["overflow_recomputed"] += rx.last_recomputed
            stats["zero_cell"] += int(((st & 1) != 0).sum())
            yh = np.ascontiguousarray(y[c0:c1].cpu().numpy())
            xh = np.ascontiguousarray(x[c0:c1].cpu().numpy())
            sh = np.ascontiguousarray(s2[c0:c1].cpu().numpy(), np.float64)
            kh = None if kk is None else np.ascontiguousarray(kk.cpu().numpy(), np.int32)
            t0 = time.perf_counter()
            d, v, w, cnt, s2h, eta = O.receive_batch(rc, yh, xh, sh, K, kh, threads=THREADS)
            t_orc += time.perf_counter() - t0
            gs2h = dets.sigma2_h.cpu().numpy()
            for f in range(c1 - c0):
                k = int(kh[f]) if kh is not None else K
                ref = [(int(d[f, i]), int(v[f, i]), float(w[f, i])) for i in range(int(cnt[f]))]
                _compare_dets(cfg, name, stats, c0 + f, dets.frame(f), ref, float(s2h[f]), float(gs2h[f]), yh[f], xh[f],
                              float(sh[f]), k)
            if check_maps:
                pmh = pm.cpu().numpy()

                def one(f):
                    _, _, _, rm = O.receive_frame(rc, yh[f], xh[f], float(sh[f]), K, want_map=True)
                    return float(np.abs(pmh[f] - rm).max() / rm.max())

                with cf.ThreadPoolExecutor(THREADS) as ex:
                    errs = list(ex.map(one, range(c1 - c0)))
                max_map_err = max(max_map_err, max(errs))
                assert max(errs) <= MAP_TOL, (name, c0, max(errs))
    stats["gpu_s"] = round(t_gpu, 3)
    stats["oracle_s"] = round(t_orc, 3)
    if check_maps:
        stats["max_map_rel_err"] = max_map_err
    assert stats["fail"] == 0
    REPORT[name] = stats
    _write_report()
    return stats


def test_full_cfg0(cuda):
    cfg = configs.CFG0
    fb = gen.frames(cfg, 0, 1)
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    _pipeline_all(cfg, "cfg0", t(fb.y), t(fb.x), t(fb.sigma2), None, 1, check_maps=True)


def test_full_cfg1(cuda):
    cfg = configs.CFG1
    fb = gen.frames(cfg, 0, cfg.frames)
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    s = _pipeline_all(cfg, "cfg1", t(fb.y), t(fb.x), t(fb.sigma2), None, 64, check_maps=True)
    assert s["frames"] == 64


def test_full_cfg2(cuda):
    cfg = configs.CFG2
    g = gen.frames_device(cfg, 0, cfg.frames)
    s = _pipeline_all(cfg, "cfg2", g["y"], g["x"], g["sigma2"], None, 16, check_maps=True)
    assert s["frames"] == 256


def test_full_cfg4_bench_batch(cuda):
    cfg = configs.CFG4
    g = gen.frames_device(cfg, 0, cfg.frames)  # the bench's batch (bench.py, world size 1)
    s = _pipeline_all(cfg, "cfg4", g["y"], g["x"], g["sigma2"], g["n_targets"], 1024)
    assert s["frames"] == 8192


def test_full_cfg3_sft_and_support(cuda):
    c3 = configs.CFG3
    F, chunk = c3.frames, 64
    stats = {"frames": F, "ok": 0, "fail": 0, "max_amp_rel_err": 0.0,
             "support_gpu_sft_eq_gpu_periodogram": 0, "support_oracle_sft_eq_oracle_periodogram": 0,
             "support_gpu_sft_eq_oracle_periodogram": 0, "support_gpu_sft_subset_of_gpu_periodogram": 0,
             "support_oracle_sft_subset_of_oracle_periodogram": 0, "sft_detections_gpu_total": 0,
             "periodogram_detections_gpu_total": 0,
             "note": "FPS-SFT with BASELINE's i_max = 8 recovers a subset of the 10 on-grid targets on most "
                     "frames (the same subset in the oracle); the reference's bench_estimators support "
                     "precondition (metrics.cpp:220-231) is met on the frames counted as 'eq'"}
    dev = torch.device("cuda", 0)
    pr = Receiver(c3.n, c3.m, c3.n, c3.m, window="rectangular", estimator="ls", max_targets=c3.max_targets,
                  pfa=c3.pfa)
    sr = Receiver(16, 16)
    ok_sup = []
    for c0 in range(0, F, chunk):
        h, s2, _, _ = gen.sparse_frames(c3.n, c3.m, c3.targets, c3.snr_db, c3.base_seed, c0, chunk)
        seeds = np.array([gen.derive_seed(c3.base_seed + c0 + f, 0x736674) for f in range(chunk)], np.uint64)
        hd = torch.from_numpy(h).to(dev)
        out = sr.sft(hd, seeds, s2, i_max=c3.i_max, pfa=c3.pfa, decimation=c3.decimation)
        sd = pr.sft_detections(out, c3.n, c3.m, torch.from_numpy(s2).to(dev), c3.pfa)  # sft.cpp:461-490 on the GPU
        pm = pr.periodogram(hd)
        pd = pr.detect(pm, torch.from_numpy(s2).to(dev))  # eta = -sigma2 ln(Pfa) * pf(rect) = bench_estimators'
        torch.cuda.synchronize()
        k, l = out["k"].cpu().numpy(), out["l"].cpu().numpy()
        amp, ne = out["amp"].cpu().numpy(), out["n_entries"].cpu().numpy()
        its, su, conv = (out["iterations"].cpu().numpy(), out["samples_used"].cpu().numpy(),
                         out["converged"].cpu().numpy())

        def oracle(f):
            ref = O.sft_iterate(h[f].astype(np.complex128), int(seeds[f]), float(s2[f]), i_max=c3.i_max, pfa=c3.pfa,
                                decimation=c3.decimation)
            p = O.periodogram(h[f].astype(np.complex128), 0, c3.n, c3.m)
            eta = O.detection_threshold(float(s2[f]), c3.pfa, 1.0)
            return ref, O.extract_peaks(p, eta, c3.max_targets)

        with cf.ThreadPoolExecutor(THREADS) as ex:
            res = list(ex.map(oracle, range(chunk)))
        for f in range(chunk):
            ref, ref_pdet = res[f]
            n = int(ne[f])
            got = [(int(k[f, i]), int(l[f, i])) for i in range(n)]
            good = (n == ref["n_entries"] and got == [(a, b) for a, b, _ in ref["entries"]]
                    and int(its[f]) == ref["iterations"] and int(su[f]) == ref["samples_used"]
                    and bool(conv[f]) == ref["converged"])
            ga = amp[f, :n, 0] + 1j * amp[f, :n, 1]
            ra = np.array([a for _, _, a in ref["entries"]])
            if good and n:
                err = float(np.abs(ga - ra).max() / np.abs(ra).max())
                stats["max_amp_rel_err"] = max(stats["max_amp_rel_err"], err)
                good = err <= 1e-4
            stats["ok" if good else "fail"] += 1
            assert good, (c0 + f, got, ref["entries"][:4], int(its[f]), ref["iterations"])
            # bench_estimators support check (metrics.cpp:220-231)
            sdet = sd.frame(f)
            ssup = sorted((a, b) for a, b, _ in sdet)
            psup = sorted((a, b) for a, b, _ in pd.frame(f))
            osdet = O.detections_from_spectrum(ref["entries"], c3.n, c3.m, float(s2[f]), c3.pfa, c3.max_targets)
            osup = sorted((a, b) for a, b, _ in osdet)
            # device detections_from_spectrum: bins and order exact, powers to fp32 rounding
            assert [(a, b) for a, b, _ in sdet] == [(a, b) for a, b, _ in osdet], (c0 + f, sdet, osdet)
            for (_, _, pg), (_, _, po) in zip(sdet, osdet):
                assert abs(pg - po) <= 1e-6 * po
            opsup = sorted((a, b) for a, b, _ in ref_pdet)
            stats["support_gpu_sft_eq_gpu_periodogram"] += ssup == psup
            stats["support_oracle_sft_eq_oracle_periodogram"] += osup == opsup
            stats["support_gpu_sft_eq_oracle_periodogram"] += ssup == opsup
            stats["support_gpu_sft_subset_of_gpu_periodogram"] += set(ssup) <= set(psup)
            stats["support_oracle_sft_subset_of_oracle_periodogram"] += set(osup) <= set(opsup)
            stats["sft_detections_gpu_total"] += len(ssup)
            stats["periodogram_detections_gpu_total"] += len(psup)
            ok_sup.append(ssup == psup)
            # the GPU reproduces the oracle's detections and support decisions on every frame
            assert ssup == osup, (c0 + f, ssup, osup)
            assert psup == opsup, (c0 + f, psup, opsup)
    pr.close()
    sr.close()
    REPORT["cfg3"] = stats
    _write_report()
    assert stats["fail"] == 0
