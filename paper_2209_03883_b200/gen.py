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
