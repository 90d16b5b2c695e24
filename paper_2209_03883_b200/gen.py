"""Seeded synthetic inputs (csrc/gen.cpp via ctypes).  Input side only: the frames
both the CUDA receiver and the CPU oracle consume (SURVEY.md §8d "Inputs")."""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _native
from .configs import RadarConfig

MAX_T = 16


@dataclass
class FrameBatch:
    y: np.ndarray          # (F, N, M) complex64
    x: np.ndarray          # (F, N, M) complex64 (x_tx, precoded for cfg2)
    sigma2: np.ndarray     # (F,) float64 noise variance per cell
    n_targets: np.ndarray  # (F,) int32
    ranges: np.ndarray     # (F, MAX_T)
    vels: np.ndarray       # (F, MAX_T)
    snr_db: np.ndarray     # (F,)


def gen_params(cfg: RadarConfig) -> _native.GenParams:
    p = _native.GenParams()
    p.n, p.m = cfg.n, cfg.m
    p.df_hz, p.fc_hz = cfg.df_hz, 77e9
    p.n_cp = cfg.n_cp
    p.qam_order = cfg.qam
    p.zc_precode = 1 if cfg.zc_precode else 0
    p.zc_root = 1
    p.targets_min, p.targets_max = cfg.targets_min, cfg.targets_max
    p.range_lo, p.range_hi = cfg.range_lo, cfg.range_hi
    p.vel_lo, p.vel_hi = cfg.vel_lo, cfg.vel_hi
    p.snr_lo_db, p.snr_hi_db = cfg.snr_lo_db, cfg.snr_hi_db
    return p


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def frames(cfg: RadarConfig, first: int = 0, count: int | None = None, threads: int | None = None) -> FrameBatch:
    count = cfg.frames if count is None else count
    threads = threads or os.cpu_count() or 1
    y = np.empty((count, cfg.n, cfg.m), np.complex64)
    x = np.empty((count, cfg.n, cfg.m), np.complex64)
    s2 = np.empty(count, np.float64)
    nt = np.empty(count, np.int32)
    rg = np.zeros((count, MAX_T), np.float64)
    vl = np.zeros((count, MAX_T), np.float64)
    snr = np.empty(count, np.float64)
    p = gen_params(cfg)
    rc = _native.gen().ofdmr_gen_batch(C.byref(p), cfg.base_seed, first, count, _ptr(y), _ptr(x), _ptr(s2), _ptr(nt),
                                       _ptr(rg), _ptr(vl), _ptr(snr), MAX_T, threads)
    if rc:
        raise ValueError(f"generator failed with code {rc}")
    return FrameBatch(y, x, s2, nt, rg, vl, snr)


def sparse_frames(n: int, m: int, k: int, snr_db: float, base_seed: int, first: int, count: int,
                  threads: int | None = None):
    """cfg3 on-grid sparse H (make_sparse convention, tests/test_sft.cpp:20-50)."""
    threads = threads or os.cpu_count() or 1
    h = np.empty((count, n, m), np.complex64)
    s2 = np.empty(count, np.float64)
    tk = np.empty((count, k), np.int32)
    tl = np.empty((count, k), np.int32)
    rc = _native.gen().ofdmr_gen_sparse_batch(n, m, k, snr_db, base_seed, first, count, _ptr(h), _ptr(s2), _ptr(tk),
                                              _ptr(tl), threads)
    if rc:
        raise ValueError(f"sparse generator failed with code {rc}")
    return h, s2, tk, tl


def noise_grid(n: int, m: int, sigma2: float, seed: int) -> np.ndarray:
    """noise_grid (tests/test_periodogram.cpp:31-37) as complex128."""
    out = np.empty((n, m), np.complex128)
    _native.gen().ofdmr_gen_noise_grid(n, m, sigma2, seed, _ptr(out))
    return out


def derive_seed(base: int, stream: int) -> int:
    return int(_native.gen().ofdmr_derive_seed(base, stream))


def rng_u64(seed: int, count: int) -> np.ndarray:
    out = np.empty(count, np.uint64)
    _native.gen().ofdmr_rng_u64(seed, count, _ptr(out))
    return out


def frames_device(cfg: RadarConfig, first: int = 0, count: int | None = None, device=None):
    """GPU generator (csrc/gen_kernels.cu, include/ofdmr_gen.h): frames [first, first+count)
    generated in device memory, same streams and arithmetic order as `frames` (rare 1-ulp c64
    differences from the GPU's fp64 sin/cos/log/pow).  Frames that hit an MT19937 rejection
    draw (status bit 0, probability ~2^-50) are regenerated with the CPU generator.
    Returns a dict of torch tensors: y, x (complex64 [F, N, M]), sigma2 (float64), n_targets
    (int32), ranges, vels ([F, MAX_T] float64), snr_db (float64)."""
    import torch

    count = cfg.frames if count is None else count
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    out = {
        "y": torch.empty(count, cfg.n, cfg.m, dtype=torch.complex64, device=dev),
        "x": torch.empty(count, cfg.n, cfg.m, dtype=torch.complex64, device=dev),
        "sigma2": torch.empty(count, dtype=torch.float64, device=dev),
        "n_targets": torch.empty(count, dtype=torch.int32, device=dev),
        "ranges": torch.zeros(count, MAX_T, dtype=torch.float64, device=dev),
        "vels": torch.zeros(count, MAX_T, dtype=torch.float64, device=dev),
        "snr_db": torch.empty(count, dtype=torch.float64, device=dev),
    }
    status = torch.empty(count, dtype=torch.int32, device=dev)
    p = gen_params(cfg)
    stream = torch.cuda.current_stream(dev).cuda_stream
    rc = _native.lib().ofdmr_gen_device(C.byref(p), cfg.base_seed, first, count, out["y"].data_ptr(),
                                         out["x"].data_ptr(), out["sigma2"].data_ptr(), out["n_targets"].data_ptr(),
                                         out["ranges"].data_ptr(), out["vels"].data_ptr(), out["snr_db"].data_ptr(),
                                         MAX_T, status.data_ptr(), C.c_void_p(stream))
    if rc:
        raise RuntimeError(f"ofdmr_gen_device failed ({rc}): {_native.last_error()}")
    bad = torch.nonzero(status).flatten().tolist()
    for i in bad:  # exact CPU regeneration of the (astronomically rare) rejection frames
        fb = frames(cfg, first + i, 1, threads=1)
        out["y"][i] = torch.from_numpy(fb.y[0]).to(dev)
        out["x"][i] = torch.from_numpy(fb.x[0]).to(dev)
        out["sigma2"][i] = float(fb.sigma2[0])
        out["n_targets"][i] = int(fb.n_targets[0])
        out["ranges"][i] = torch.from_numpy(fb.ranges[0]).to(dev)
        out["vels"][i] = torch.from_numpy(fb.vels[0]).to(dev)
        out["snr_db"][i] = float(fb.snr_db[0])
    out["regenerated_on_cpu"] = len(bad)
    return out
