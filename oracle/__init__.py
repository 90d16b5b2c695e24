"""ORACLE — TEST INFRASTRUCTURE ONLY.

Python bindings for
  * oracle/liboracle.so        — the plain-C fp64 restatement (oracle/oracle.c), and
  * oracle/_ref/libofdmref.so  — the reference's own sources + substitute FFT (built
                                 by oracle/Makefile where /root/reference exists).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package, and only as the checker / timed CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libofdmref.so"

vp = C.c_void_p


class RxConfig(C.Structure):
    _fields_ = [("n", C.c_int32), ("m", C.c_int32), ("n_prime", C.c_int32), ("m_prime", C.c_int32),
                ("estimator", C.c_int32), ("n_cp", C.c_int32), ("window", C.c_int32), ("pfa", C.c_double)]


class SftConfig(C.Structure):
    _fields_ = [("i_max", C.c_int64), ("detect_threshold", C.c_double), ("seed", C.c_uint64),
                ("sigma2", C.c_double), ("pfa", C.c_double), ("decimation", C.c_int64),
                ("frac_tol", C.c_double), ("amp_tol", C.c_double)]


class SftResult(C.Structure):
    _fields_ = [("n_entries", C.c_int64), ("residual_energy", C.c_double), ("converged", C.c_int32),
                ("iterations", C.c_int64), ("samples_used", C.c_int64)]


_orc = None
_ref = None


def orc() -> C.CDLL:
    global _orc
    if _orc is None:
        if not ORACLE_SO.exists():
            raise ImportError(f"{ORACLE_SO} missing: run `make -f oracle/Makefile`")
        _orc = C.CDLL(str(ORACLE_SO))
        _orc.orc_detection_threshold.restype = C.c_int
        _orc.orc_division_noise_power.restype = C.c_double
        _orc.orc_division_noise_power.argtypes = [C.c_double, vp, C.c_size_t]
        _orc.orc_power_factor.restype = C.c_double
        _orc.orc_power_factor.argtypes = [vp, C.c_size_t, vp, C.c_size_t]
        _orc.orc_extract_peaks.restype = C.c_long
        _orc.orc_extract_peaks.argtypes = [vp, C.c_size_t, C.c_size_t, vp, C.c_size_t, vp, vp, vp]
        _orc.orc_estimate_noise_power.restype = C.c_double
        _orc.orc_estimate_noise_power.argtypes = [vp, C.c_size_t, C.c_double]
        _orc.orc_derive_seed.restype = C.c_uint64
        _orc.orc_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        _orc.orc_slope_admissible.argtypes = [C.c_long, C.c_long, C.c_size_t, C.c_size_t]
        _orc.orc_detections_from_spectrum.restype = C.c_long
        _orc.orc_detections_from_spectrum.argtypes = [vp, vp, vp, vp, C.c_long, C.c_size_t, C.c_size_t, C.c_double,
                                                      C.c_double, C.c_long, vp, vp, vp]
        _orc.orc_rng_u64.argtypes = [C.c_uint64, C.c_long, vp]
        _orc.orc_receive_batch.argtypes = [C.POINTER(RxConfig), vp, vp, vp, C.c_long, vp, C.c_int32, vp, vp, vp, vp,
                                           vp, vp, C.c_int]
        _orc.orc_receive_frame.argtypes = [C.POINTER(RxConfig), vp, vp, C.c_double, C.c_int32, vp, vp, vp, vp, vp,
                                           vp, vp]
        _orc.orc_sft_iterate.argtypes = [vp, C.c_size_t, C.c_size_t, C.POINTER(SftConfig), C.c_long, vp, vp, vp, vp,
                                         C.POINTER(SftResult)]
        _orc.orc_fft.argtypes = [vp, C.c_size_t, C.c_int]
        sz = C.c_size_t
        _orc.orc_spectral_division.argtypes = [vp, vp, vp, sz, sz]
        _orc.orc_dft_ce.argtypes = [vp, vp, sz, sz, sz]
        _orc.orc_make_window.argtypes = [C.c_int, sz, sz, vp, vp]
        _orc.orc_periodogram.argtypes = [vp, sz, sz, vp, vp, sz, sz, vp]
        _orc.orc_detection_threshold.argtypes = [C.c_double, C.c_double, C.c_double, vp]
        _orc.orc_ofdm_modulate.argtypes = [vp, sz, sz, sz, vp]
        _orc.orc_estimate_noise_from_slice.restype = C.c_double
        _orc.orc_estimate_noise_from_slice.argtypes = [vp, sz, sz, C.c_uint64]
        _orc.orc_ofdm_demodulate.argtypes = [vp, sz, sz, sz, vp]
    return _orc


REF_IO_SO = HERE / "_ref" / "libofdmref_io.so"
_ref_io = None


def ref_io() -> C.CDLL:
    """The reference's own output writers (io.cpp) behind oracle/ref_shim/ref_io_capi.cpp."""
    global _ref_io
    if _ref_io is None:
        if not REF_IO_SO.exists():
            raise ImportError(f"{REF_IO_SO} missing (built from /root/reference by `make -f oracle/Makefile ref`)")
        _ref_io = C.CDLL(str(REF_IO_SO))
        i64 = C.c_int64
        _ref_io.ref_write_map_csv.argtypes = [vp, i64, i64, C.c_char_p]
        _ref_io.ref_write_map_pgm.argtypes = [vp, i64, i64, C.c_char_p]
        _ref_io.ref_write_detections_csv.argtypes = [vp, vp, vp, vp, vp, i64, C.c_char_p]
        i32, d = C.c_int32, C.c_double
        _ref_io.ref_write_run_manifest.argtypes = [C.c_char_p, C.c_char_p, C.c_uint64, i64, i64, d, d, i64, i32, i64,
                                                   i64, i32, d, i32, i32, i64, i32, i64, vp, vp, vp, i32, d, vp, vp,
                                                   i32, d]
    return _ref_io


def ref_available() -> bool:
    return REF_SO.exists()


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not REF_SO.exists():
            raise ImportError(f"{REF_SO} missing (built from /root/reference by `make -f oracle/Makefile ref`)")
        _ref = C.CDLL(str(REF_SO))
        i64, d = C.c_int64, C.c_double
        _ref.ref_run_pipeline.argtypes = [i64, i64, i64, i64, d, d, i64, C.c_int, d, C.c_int, vp, vp, C.c_int32, d,
                                          C.c_uint64, vp, vp, vp, vp, vp]
        _ref.ref_mse_sweep.argtypes = [i64, i64, i64, i64, d, d, i64, C.c_int, d, C.c_int, vp, vp, C.c_int32, vp,
                                       C.c_int32, i64, C.c_uint64, vp]
        _ref.ref_rmse_sweep.argtypes = [i64, i64, i64, i64, d, d, i64, C.c_int, d, C.c_int, vp, vp, C.c_int32, vp,
                                        C.c_int32, i64, C.c_uint64, vp]
        _ref.ref_receive_frame.argtypes = [i64, i64, i64, i64, C.c_int, i64, C.c_int, d, vp, vp, d, i64, vp, vp, vp,
                                           vp, vp, vp, vp]
        _ref.ref_receive_batch.argtypes = [i64, i64, i64, i64, C.c_int, i64, C.c_int, d, vp, vp, vp, i64, vp, i64, vp,
                                           vp, vp, vp, C.c_int]
        _ref.ref_periodogram.argtypes = [vp, i64, i64, C.c_int, i64, i64, vp]
        _ref.ref_dft_ce.argtypes = [vp, vp, i64, i64, i64]
        _ref.ref_spectral_division.argtypes = [vp, vp, vp, i64, i64]
        _ref.ref_extract_peaks.restype = C.c_long
        _ref.ref_extract_peaks.argtypes = [vp, i64, i64, d, i64, vp, vp, vp]
        _ref.ref_window_power_factor.restype = d
        _ref.ref_window_power_factor.argtypes = [C.c_int, i64, i64]
        _ref.ref_detection_threshold.argtypes = [d, d, d, vp]
        _ref.ref_bins_to_physics.argtypes = [C.c_long, C.c_long, i64, i64, i64, i64, d, d, i64, vp, vp]
        _ref.ref_sft_iterate.argtypes = [vp, i64, i64, i64, d, C.c_uint64, d, d, i64, d, d, i64, vp, vp, vp, vp, vp,
                                         vp, vp, vp, vp]
        _ref.ref_sft_batch_c64.argtypes = [vp, i64, i64, i64, i64, vp, vp, d, i64, i64, vp, vp, vp, vp, vp, C.c_int]
        _ref.ref_make_frame_pair.argtypes = [i64, i64, d, d, i64, C.c_int, vp, vp, i64, d, C.c_uint64, vp, vp, vp]
        _ref.ref_rng_u64.argtypes = [C.c_uint64, i64, vp]
        _ref.ref_bench_estimators.argtypes = [i64, i64, d, d, C.c_int, C.c_int, d, d, vp, C.c_int32, i64, i64,
                                              C.c_uint64, vp, vp, vp, vp]
        _ref.ref_run_pipeline_q.argtypes = [i64, i64, i64, i64, d, d, i64, C.c_int, d, C.c_int, vp, vp, C.c_int32,
                                            C.c_int, d, C.c_uint64, vp, vp, vp]
        _ref.ref_run_pipeline_sft.argtypes = [i64, i64, d, d, i64, C.c_int, C.c_int, vp, vp, C.c_int32, d, C.c_uint64,
                                              C.c_int, i64, i64, vp, vp, vp, vp, vp]
        _ref.ref_sft_noise_case.argtypes = [i64, i64, d, d, i64, vp, vp, C.c_int32, d, C.c_uint64, vp, vp]
        _ref.ref_estimate_noise_power.restype = d
        _ref.ref_estimate_noise_power.argtypes = [vp, i64, i64, d]
        _ref.ref_ofdm_modulate.argtypes = [vp, i64, i64, i64, vp]
        _ref.ref_ofdm_demodulate.argtypes = [vp, i64, i64, i64, vp]
    return _ref


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


# ------------------------------------------------------------------ restatement --

def fft(x: np.ndarray, inverse: bool = False) -> np.ndarray:
    a = np.ascontiguousarray(x, np.complex128).copy()
    orc().orc_fft(_p(a), a.size, 1 if inverse else -1)
    return a


def spectral_division(y: np.ndarray, x: np.ndarray) -> np.ndarray:
    y = np.ascontiguousarray(y, np.complex128)
    x = np.ascontiguousarray(x, np.complex128)
    h = np.empty_like(y)
    rc = orc().orc_spectral_division(_p(y), _p(x), _p(h), C.c_size_t(y.shape[0]), C.c_size_t(y.shape[1]))
    if rc:
        raise ValueError("spectral_division: zero cell in X")
    return h


def dft_ce(h: np.ndarray, n_cp: int) -> np.ndarray:
    h = np.ascontiguousarray(h, np.complex128)
    out = np.empty_like(h)
    rc = orc().orc_dft_ce(_p(h), _p(out), C.c_size_t(h.shape[0]), C.c_size_t(h.shape[1]), C.c_size_t(n_cp))
    if rc:
        raise ValueError("dft_ce: truncation length exceeds N")
    return out


def make_window(kind: int, n: int, m: int):
    wk = np.empty(n)
    wl = np.empty(m)
    orc().orc_make_window(C.c_int(kind), C.c_size_t(n), C.c_size_t(m), _p(wk), _p(wl))
    return wk, wl


def power_factor(kind: int, n: int, m: int) -> float:
    wk, wl = make_window(kind, n, m)
    return orc().orc_power_factor(_p(wk), n, _p(wl), m)


def periodogram(h: np.ndarray, kind: int, n_prime: int, m_prime: int) -> np.ndarray:
    h = np.ascontiguousarray(h, np.complex128)
    n, m = h.shape
    wk, wl = make_window(kind, n, m)
    p = np.empty((n_prime, m_prime))
    rc = orc().orc_periodogram(_p(h), C.c_size_t(n), C.c_size_t(m), _p(wk), _p(wl), C.c_size_t(n_prime),
                               C.c_size_t(m_prime), _p(p))
    if rc:
        raise ValueError("periodogram: N' >= N and M' >= M required")
    return p


def detection_threshold(sigma2: float, pfa: float, pf: float) -> float:
    eta = C.c_double()
    rc = orc().orc_detection_threshold(C.c_double(sigma2), C.c_double(pfa), C.c_double(pf), C.byref(eta))
    if rc:
        raise ValueError("threshold: bad arguments")
    return eta.value


def extract_peaks(p: np.ndarray, eta: float, max_targets: int):
    p = np.ascontiguousarray(p, np.float64)
    mask = (p >= eta).astype(np.uint8)
    d = np.zeros(max_targets, np.int64)
    v = np.zeros(max_targets, np.int64)
    w = np.zeros(max_targets, np.float64)
    n = orc().orc_extract_peaks(_p(p), p.shape[0], p.shape[1], _p(mask), max_targets, _p(d), _p(v), _p(w))
    return [(int(d[i]), int(v[i]), float(w[i])) for i in range(n)]


def division_noise_power(sigma2: float, x: np.ndarray) -> float:
    x = np.ascontiguousarray(x, np.complex128)
    return orc().orc_division_noise_power(sigma2, _p(x), x.size)


def estimate_noise_power(p: np.ndarray, pf: float) -> float:
    p = np.ascontiguousarray(p, np.float64)
    return orc().orc_estimate_noise_power(_p(p), p.size, pf)


def estimate_noise_from_slice(h: np.ndarray, seed: int) -> float:
    """pipeline.cpp:26-43 (FPS-SFT estimate-noise mode) on an N x M grid (fp64)."""
    h = np.ascontiguousarray(h, np.complex128)
    return orc().orc_estimate_noise_from_slice(_p(h), h.shape[0], h.shape[1], seed)


def ofdm_modulate(x: np.ndarray, n_cp: int) -> np.ndarray:
    """waveform.cpp:133-149 on an N x M grid -> stream [M][N_cp + N] (fp64)."""
    x = np.ascontiguousarray(x, np.complex128)
    n, m = x.shape
    out = np.zeros((m, n + n_cp), np.complex128)
    if orc().orc_ofdm_modulate(_p(x), n, m, n_cp, _p(out)) != 0:
        raise ValueError("n_cp > N")
    return out


def ofdm_demodulate(stream: np.ndarray, n: int, m: int, n_cp: int) -> np.ndarray:
    """waveform.cpp:152-166: stream [M][N_cp + N] -> N x M grid (fp64)."""
    s = np.ascontiguousarray(stream, np.complex128).reshape(m, n + n_cp)
    out = np.zeros((n, m), np.complex128)
    orc().orc_ofdm_demodulate(_p(s), n, m, n_cp, _p(out))
    return out


def rx_config(n, m, n_prime, m_prime, estimator, n_cp, window, pfa) -> RxConfig:
    c = RxConfig()
    c.n, c.m, c.n_prime, c.m_prime = n, m, n_prime, m_prime
    c.estimator, c.n_cp, c.window, c.pfa = estimator, n_cp, window, pfa
    return c


def receive_frame(cfg: RxConfig, y: np.ndarray, x: np.ndarray, sigma2: float, max_targets: int,
                  want_map: bool = False):
    """run_pipeline's receiver half on one c64 frame (upcast to fp64)."""
    y = np.ascontiguousarray(y, np.complex64)
    x = np.ascontiguousarray(x, np.complex64)
    d = np.zeros(max(max_targets, 1), np.int64)
    v = np.zeros(max(max_targets, 1), np.int64)
    w = np.zeros(max(max_targets, 1), np.float64)
    cnt = C.c_long()
    s2h = C.c_double()
    eta = C.c_double()
    pmap = np.empty((cfg.n_prime, cfg.m_prime)) if want_map else None
    rc = orc().orc_receive_frame(C.byref(cfg), _p(y), _p(x), sigma2, max_targets, _p(d), _p(v), _p(w), C.byref(cnt),
                                 C.byref(s2h), C.byref(eta), _p(pmap) if pmap is not None else None)
    if rc:
        raise ValueError("oracle receive_frame: config error")
    dets = [(int(d[i]), int(v[i]), float(w[i])) for i in range(cnt.value)]
    return dets, s2h.value, eta.value, pmap


def receive_batch(cfg: RxConfig, y: np.ndarray, x: np.ndarray, sigma2: np.ndarray, k_max: int,
                  k_per_frame: np.ndarray | None = None, threads: int | None = None):
    F = y.shape[0]
    threads = threads or os.cpu_count() or 1
    d = np.zeros((F, k_max), np.int64)
    v = np.zeros((F, k_max), np.int64)
    w = np.zeros((F, k_max), np.float64)
    cnt = np.zeros(F, np.int64)
    s2h = np.zeros(F)
    eta = np.zeros(F)
    kp = None if k_per_frame is None else np.ascontiguousarray(k_per_frame, np.int32)
    rc = orc().orc_receive_batch(C.byref(cfg), _p(y), _p(x), _p(np.ascontiguousarray(sigma2, np.float64)), F,
                                 _p(kp) if kp is not None else None, k_max, _p(d), _p(v), _p(w), _p(cnt), _p(s2h),
                                 _p(eta), threads)
    if rc:
        raise ValueError("oracle receive_batch: config error")
    return d, v, w, cnt, s2h, eta


def sft_iterate(h: np.ndarray, seed: int, sigma2: float = 0.0, i_max: int = 10, detect_threshold: float = 0.0,
                pfa: float = 1e-2, decimation: int = 8, frac_tol: float = 0.25, amp_tol: float = 0.35,
                max_entries: int = 256):
    h = np.ascontiguousarray(h, np.complex128)
    c = SftConfig(i_max, detect_threshold, seed, sigma2, pfa, decimation, frac_tol, amp_tol)
    k = np.zeros(max_entries, np.int64)
    l = np.zeros(max_entries, np.int64)
    ar = np.zeros(max_entries)
    ai = np.zeros(max_entries)
    res = SftResult()
    rc = orc().orc_sft_iterate(_p(h), h.shape[0], h.shape[1], C.byref(c), max_entries, _p(k), _p(l), _p(ar), _p(ai),
                               C.byref(res))
    if rc:
        raise ValueError("sft_iterate: empty grid")
    n = min(res.n_entries, max_entries)
    ents = [(int(k[i]), int(l[i]), complex(ar[i], ai[i])) for i in range(n)]
    return dict(entries=ents, residual=res.residual_energy, converged=bool(res.converged),
                iterations=int(res.iterations), samples_used=int(res.samples_used), n_entries=int(res.n_entries))


def detections_from_spectrum(entries, n: int, m: int, sigma2: float, pfa: float, max_targets: int):
    ne = len(entries)
    k = np.array([e[0] for e in entries] + [0], np.int64)
    l = np.array([e[1] for e in entries] + [0], np.int64)
    ar = np.array([e[2].real for e in entries] + [0.0])
    ai = np.array([e[2].imag for e in entries] + [0.0])
    d = np.zeros(max(max_targets, 1), np.int64)
    v = np.zeros(max(max_targets, 1), np.int64)
    w = np.zeros(max(max_targets, 1))
    cnt = orc().orc_detections_from_spectrum(_p(k), _p(l), _p(ar), _p(ai), ne, n, m, sigma2, pfa, max_targets, _p(d),
                                             _p(v), _p(w))
    return [(int(d[i]), int(v[i]), float(w[i])) for i in range(cnt)]


def rng_u64(seed: int, count: int) -> np.ndarray:
    out = np.empty(count, np.uint64)
    orc().orc_rng_u64(seed, count, _p(out))
    return out


def derive_seed(base: int, stream: int) -> int:
    return int(orc().orc_derive_seed(base, stream))


def ref_scenario_args(n, m, n_prime, m_prime, df, fc, n_cp, window, pfa, estimator, ranges, vels):
    r = np.ascontiguousarray(ranges, np.float64)
    v = np.ascontiguousarray(vels, np.float64)
    return (n, m, n_prime, m_prime, df, fc, n_cp, window, pfa, estimator, _p(r), _p(v), len(r)), (r, v)


def ref_run_pipeline(scn, snr_db: float, seed: int):
    """The reference's run_pipeline on a fixed scenario (oracle/_ref, test infrastructure)."""
    args, keep = ref_scenario_args(*scn)
    k = max(args[-1], 1)
    d = np.zeros(k, np.int64)
    v = np.zeros(k, np.int64)
    r = np.zeros(k)
    vel = np.zeros(k)
    cnt = C.c_long()
    rc = ref().ref_run_pipeline(*args, snr_db, seed, _p(d), _p(v), _p(r), _p(vel), C.byref(cnt))
    assert rc == 0
    n = cnt.value
    return d[:n], v[:n], r[:n], vel[:n]


def ref_rmse_sweep(scn, snr_grid, trials: int, seed: int) -> np.ndarray:
    """The reference's rmse_sweep (metrics.cpp:92-120): rows [snr][range_rmse, vel_rmse, miss_rate]."""
    args, keep = ref_scenario_args(*scn)
    g = np.ascontiguousarray(snr_grid, np.float64)
    rows = np.zeros((len(g), 3))
    rc = ref().ref_rmse_sweep(*args, _p(g), len(g), trials, seed, _p(rows))
    assert rc == 0
    return rows


def ref_mse_sweep(scn, snr_grid, trials: int, seed: int) -> np.ndarray:
    """The reference's mse_sweep (metrics.cpp:122-143): per-SNR channel MSE."""
    args, keep = ref_scenario_args(*scn)
    g = np.ascontiguousarray(snr_grid, np.float64)
    rows = np.zeros(len(g))
    rc = ref().ref_mse_sweep(*args, _p(g), len(g), trials, seed, _p(rows))
    assert rc == 0
    return rows


def ref_make_frame_pair(n, m, df, fc, n_cp, qam, ranges, vels, snr_db: float, seed: int):
    """run_pipeline's frame for `seed` (make_random_frame + apply_channel, pipeline.cpp:65-70) from
    the reference sources: (y, x) complex128 N x M and the realization's sigma2."""
    r = np.ascontiguousarray(ranges, np.float64)
    v = np.ascontiguousarray(vels, np.float64)
    y = np.empty((n, m), np.complex128)
    x = np.empty((n, m), np.complex128)
    s2 = C.c_double()
    rc = ref().ref_make_frame_pair(n, m, df, fc, n_cp, qam, _p(r), _p(v), len(r), snr_db, seed, _p(y), _p(x),
                                   C.byref(s2))
    if rc:
        raise ValueError(f"ref_make_frame_pair failed ({rc})")
    return y, x, s2.value


def ref_run_pipeline_sft(n, m, df, fc, n_cp, qam, estimator, ranges, vels, snr_db: float, seed: int,
                         estimate_noise: bool, i_max: int, max_targets: int):
    """The reference's run_pipeline with the FPS-SFT detector: ([(delay, doppler, power)], sigma2_used)."""
    r = np.ascontiguousarray(ranges, np.float64)
    v = np.ascontiguousarray(vels, np.float64)
    k = max(max_targets, 1)
    d = np.zeros(k, np.int64)
    dp = np.zeros(k, np.int64)
    w = np.zeros(k)
    cnt = C.c_long()
    s2u = C.c_double()
    rc = ref().ref_run_pipeline_sft(n, m, df, fc, n_cp, qam, estimator, _p(r), _p(v), len(r), snr_db, seed,
                                    1 if estimate_noise else 0, i_max, max_targets, _p(d), _p(dp), _p(w),
                                    C.byref(cnt), C.byref(s2u))
    if rc:
        raise ValueError(f"ref_run_pipeline_sft failed ({rc})")
    return [(int(d[i]), int(dp[i]), float(w[i])) for i in range(cnt.value)], s2u.value


def sft_pipeline_frame(y: np.ndarray, x: np.ndarray, sigma2: float, estimator: int, n_cp: int, sft_seed: int,
                       noise_seed: int | None, i_max: int, pfa: float, max_targets: int):
    """The FPS-SFT branch of run_pipeline (pipeline.cpp:47-58, 79, 97-113) restated on one frame with
    the oracle's functions (fp64 on the upcast inputs): ([(delay, doppler, power)], sigma2_used, spectrum)."""
    h = spectral_division(y, x)
    if estimator == 1:
        h = dft_ce(h, n_cp)
    s2 = division_noise_power(sigma2, x)
    if noise_seed is not None:
        s2 = estimate_noise_from_slice(h, noise_seed)
    spec = sft_iterate(h, sft_seed, s2, i_max=i_max, pfa=pfa)
    return detections_from_spectrum(spec["entries"], h.shape[0], h.shape[1], s2, pfa, max_targets), s2, spec


def ref_bench_estimators(n, m, df, fc, qam, window, pfa, snr_db, sizes, k, repeats, seed):
    """The reference's bench_estimators (metrics.cpp:145-253): rows (n, periodogram_ms, sft_ms,
    speedup, samples_used); raises RuntimeError when its support precondition fails."""
    sz = np.ascontiguousarray(sizes, np.int64)
    pg, sf, sp = np.zeros(len(sz)), np.zeros(len(sz)), np.zeros(len(sz))
    su = np.zeros(len(sz), np.int64)
    rc = ref().ref_bench_estimators(n, m, df, fc, qam, window, pfa, snr_db, _p(sz), len(sz), k, repeats, seed,
                                    _p(pg), _p(sf), _p(sp), _p(su))
    if rc == 4:
        raise RuntimeError("bench: detector support sets differ")
    if rc:
        raise ValueError(f"ref_bench_estimators failed ({rc})")
    return [(int(sz[i]), float(pg[i]), float(sf[i]), float(sp[i]), int(su[i])) for i in range(len(sz))]


def ref_run_pipeline_qam(scn, qam: int, snr_db: float, seed: int):
    """ref_run_pipeline with an explicit QAM order: (delay bins, doppler bins, None, None)."""
    args, keep = ref_scenario_args(*scn)
    k = max(args[-1], 1)
    d = np.zeros(k, np.int64)
    v = np.zeros(k, np.int64)
    cnt = C.c_long()
    rc = ref().ref_run_pipeline_q(*args, qam, snr_db, seed, _p(d), _p(v), C.byref(cnt))
    if rc:
        raise ValueError(f"ref_run_pipeline_q failed ({rc})")
    return d[:cnt.value], v[:cnt.value], None, None
