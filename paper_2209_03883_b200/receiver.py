"""Host-side mirror of the reference receiver API (namespace ofdmradar)
over the CUDA C-ABI (include/ofdmr_b200.h).

Same names, argument meaning and error behaviour as the reference:
  spectral_division  estimation.hpp:9      dft_ce            estimation.hpp:14
  estimate_channel   pipeline.hpp:24-25    make_window       periodogram.hpp:32
  periodogram        periodogram.hpp:39-40 detection_threshold periodogram.hpp:52
  threshold_mask     periodogram.hpp:55    extract_peaks     periodogram.hpp:60-61
  bins_to_physics    periodogram.hpp:64    sft_iterate       sft.hpp:62
  detections_from_spectrum sft.hpp:67-70   sft_detect        sft.hpp:73-75
ConfigError mirrors ofdmradar::ConfigError (errors.hpp:9-12).  Grids are torch complex64
tensors on a CUDA device ((N, M) or batched (F, N, M)); numpy inputs are uploaded.
Every compute call goes through libofdmr_b200.so; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native
from .configs import EST_DFT_CE, EST_LS, WINDOW_HAMMING, WINDOW_RECT, RadarConfig

KSPEED_OF_LIGHT = 3.0e8
TWO_PI = 6.283185307179586476925286766559


class ConfigError(ValueError):
    """Bad parameters / shapes / zero X cell (ofdmradar::ConfigError, CLI exit code 2)."""


class CudaError(RuntimeError):
    pass


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = _native.last_error()
    if rc == 2:
        raise ConfigError(msg)
    raise CudaError(msg or f"ofdmr error {rc}")


def _window_code(w) -> int:
    if isinstance(w, int):
        return w
    s = str(w).lower()
    if s in ("rect", "rectangular"):
        return WINDOW_RECT
    if s == "hamming":
        return WINDOW_HAMMING
    raise ConfigError(f"unknown window {w!r}")


def _estimator_code(e) -> int:
    if isinstance(e, int):
        return e
    s = str(e).lower()
    if s in ("ls", "zcp-ls"):
        return EST_LS
    if s == "dft-ce":
        return EST_DFT_CE
    raise ConfigError(f"unknown estimator {e!r}")


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise CudaError("the receiver runs on a CUDA device; none is available")
    return torch.device("cuda", torch.cuda.current_device())


def _as_grid(a, dev: torch.device, dtype=torch.complex64) -> torch.Tensor:
    if isinstance(a, np.ndarray):
        a = torch.from_numpy(np.ascontiguousarray(a))
    if not isinstance(a, torch.Tensor):
        raise ConfigError("expected a tensor or ndarray")
    if a.dtype != dtype:
        a = a.to(dtype)
    a = a.to(dev)
    return a.contiguous()


def _batched(t: torch.Tensor) -> tuple[torch.Tensor, bool]:
    if t.dim() == 2:
        return t.unsqueeze(0), True
    if t.dim() == 3:
        return t, False
    raise ConfigError("grids must be (N, M) or (F, N, M)")


@dataclass
class Detections:
    """Batched detection records ([frame][max_targets]) + counts (Detection, periodogram.hpp:12-18)."""

    delay_bin: torch.Tensor
    doppler_bin: torch.Tensor
    peak_power: torch.Tensor
    counts: torch.Tensor
    sigma2_h: torch.Tensor | None = None

    def frame(self, i: int) -> list[tuple[int, int, float]]:
        n = int(self.counts[i])
        d = self.delay_bin[i, :n].tolist()
        v = self.doppler_bin[i, :n].tolist()
        p = self.peak_power[i, :n].tolist()
        return list(zip(d, v, p))


@dataclass
class SparseSpectrum:
    """SparseSpectrum (sft.hpp:41-47) for one frame."""

    entries: list[tuple[int, int, complex]] = field(default_factory=list)
    residual_energy: float = 0.0
    converged: bool = False
    iterations: int = 0
    samples_used: int = 0


class Receiver:
    """One ofdmr_context: the per-configuration receiver on one CUDA device."""

    def __init__(self, n: int, m: int, n_prime: int | None = None, m_prime: int | None = None,
                 window="hamming", estimator="ls", n_cp: int = 0, max_targets: int = 64, pfa: float = 1e-2,
                 chunk_frames: int = 0, device: int | None = None):
        self._lib = _native.lib()
        dev = _device() if device is None else torch.device("cuda", device)
        self.device = dev
        cfg = _native.OfdmrConfig()
        cfg.n_subcarriers, cfg.n_symbols = n, m
        cfg.n_prime = n if n_prime is None else n_prime
        cfg.m_prime = m if m_prime is None else m_prime
        cfg.window = _window_code(window)
        cfg.estimator = _estimator_code(estimator)
        cfg.n_cp = n_cp
        cfg.max_targets = max_targets
        cfg.pfa = pfa
        cfg.chunk_frames = chunk_frames
        cfg.device = dev.index if dev.index is not None else 0
        self.cfg = cfg
        handle = C.c_void_p()
        with torch.cuda.device(dev):
            _check(self._lib.ofdmr_create(C.byref(cfg), C.byref(handle)))
        self._h = handle

    @classmethod
    def from_config(cls, rc: RadarConfig, chunk_frames: int = 0, device: int | None = None) -> "Receiver":
        return cls(rc.n, rc.m, rc.n_prime, rc.m_prime, rc.window, rc.estimator, rc.n_cp, rc.max_targets, rc.pfa,
                   chunk_frames, device)

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.ofdmr_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- plumbing --------------------------------------------------------------
    def _stream(self) -> None:
        s = torch.cuda.current_stream(self.device).cuda_stream
        _check(self._lib.ofdmr_set_stream(self._h, C.c_void_p(s)))

    def set_profiling(self, on: bool) -> None:
        _check(self._lib.ofdmr_set_profiling(self._h, 1 if on else 0))

    def get_profile(self):
        """(ms[3], launches[3]) per stage: colpass, rowpass+detect, merge (syncs)."""
        ms = np.zeros(3, np.float64)
        n = np.zeros(3, np.int64)
        _check(self._lib.ofdmr_get_profile(self._h, ms.ctypes.data, n.ctypes.data))
        return ms, n

    @property
    def launch_count(self) -> int:
        return int(self._lib.ofdmr_launch_count(self._h))

    def _shape_check(self, t: torch.Tensor) -> None:
        if t.shape[-2:] != (self.cfg.n_subcarriers, self.cfg.n_symbols):
            raise ConfigError("grid shape does not match the receiver configuration")

    def _k(self, k_per_frame, frames: int):
        if k_per_frame is None:
            return None
        k = torch.as_tensor(k_per_frame, dtype=torch.int32).to(self.device).contiguous()
        if k.numel() != frames:
            raise ConfigError("k_per_frame must have one entry per frame")
        return k

    def _dets(self, frames: int) -> Detections:
        K = self.cfg.max_targets
        z = dict(device=self.device)
        return Detections(torch.zeros(frames, K, dtype=torch.int32, **z), torch.zeros(frames, K, dtype=torch.int32, **z),
                          torch.zeros(frames, K, dtype=torch.float32, **z), torch.zeros(frames, dtype=torch.int32, **z))

    @staticmethod
    def _raise_status(status: torch.Tensor) -> None:
        if bool((status & 1).any()):
            raise ConfigError("spectral_division: zero cell in X")

    # -- reference API ------------------------------------------------------------
    def spectral_division(self, y, x, check: bool = True) -> torch.Tensor:
        """estimation.cpp:10-21."""
        y, single = _batched(_as_grid(y, self.device))
        x, _ = _batched(_as_grid(x, self.device))
        if y.shape != x.shape:
            raise ConfigError("spectral_division: shape mismatch")
        self._shape_check(y)
        h = torch.empty_like(y)
        st = torch.empty(y.shape[0], dtype=torch.int32, device=self.device)
        self._stream()
        _check(self._lib.ofdmr_spectral_division(self._h, y.data_ptr(), x.data_ptr(), h.data_ptr(), st.data_ptr(),
                                                 y.shape[0]))
        if check:
            self._raise_status(st)
        return h[0] if single else h

    def dft_ce(self, h) -> torch.Tensor:
        """estimation.cpp:23-39 with L = n_cp."""
        h, single = _batched(_as_grid(h, self.device))
        self._shape_check(h)
        out = torch.empty_like(h)
        self._stream()
        _check(self._lib.ofdmr_dft_ce(self._h, h.data_ptr(), out.data_ptr(), h.shape[0]))
        return out[0] if single else out

    def estimate_channel(self, y, x_tx, check: bool = True) -> torch.Tensor:
        """pipeline.cpp:47-58."""
        y, single = _batched(_as_grid(y, self.device))
        x, _ = _batched(_as_grid(x_tx, self.device))
        if y.shape != x.shape:
            raise ConfigError("spectral_division: shape mismatch")
        self._shape_check(y)
        h = torch.empty_like(y)
        st = torch.empty(y.shape[0], dtype=torch.int32, device=self.device)
        self._stream()
        _check(self._lib.ofdmr_estimate_channel(self._h, y.data_ptr(), x.data_ptr(), h.data_ptr(), st.data_ptr(),
                                                y.shape[0]))
        if check:
            self._raise_status(st)
        return h[0] if single else h

    def periodogram(self, h) -> torch.Tensor:
        """periodogram.cpp:39-75 (N' x M' fp32, Doppler fft-shifted)."""
        h, single = _batched(_as_grid(h, self.device))
        self._shape_check(h)
        p = torch.empty(h.shape[0], self.cfg.n_prime, self.cfg.m_prime, dtype=torch.float32, device=self.device)
        self._stream()
        _check(self._lib.ofdmr_periodogram(self._h, h.data_ptr(), p.data_ptr(), h.shape[0]))
        return p[0] if single else p

    def _p_batch(self, p):
        p = _as_grid(p, self.device, torch.float32)
        if p.dim() == 2:
            p = p.unsqueeze(0)
        if p.shape[-2:] != (self.cfg.n_prime, self.cfg.m_prime):
            raise ConfigError("extract_peaks: mask shape mismatch")
        return p

    def detect(self, p, sigma2_h, k_per_frame=None) -> Detections:
        """detection_threshold + threshold_mask + extract_peaks (periodogram.cpp:77-136)."""
        p = self._p_batch(p)
        F = p.shape[0]
        if isinstance(sigma2_h, torch.Tensor):
            s2 = sigma2_h.to(self.device, torch.float64).reshape(-1).expand(F).contiguous()
        else:
            s2 = torch.as_tensor(np.broadcast_to(np.asarray(sigma2_h, np.float64), (F,)).copy()).to(self.device)
        if bool((s2 < 0).any()):
            raise ConfigError("threshold: sigma2 must be >= 0")
        k = self._k(k_per_frame, F)
        d = self._dets(F)
        self._stream()
        _check(self._lib.ofdmr_detect(self._h, p.data_ptr(), s2.data_ptr(), k.data_ptr() if k is not None else None,
                                      d.delay_bin.data_ptr(), d.doppler_bin.data_ptr(), d.peak_power.data_ptr(),
                                      d.counts.data_ptr(), F))
        return d

    def ofdm_demodulate(self, stream) -> torch.Tensor:
        """ofdm_demodulate (waveform.cpp:152-166): stream of M (N_cp + N) samples per frame
        -> N x M grid (CP strip + unscaled forward FFT_N per symbol)."""
        n, m, ncp = self.cfg.n_subcarriers, self.cfg.n_symbols, self.cfg.n_cp
        st = _as_grid(stream, self.device)
        single = st.dim() == 1 or (st.dim() == 2 and st.shape == (m, n + ncp))
        st = st.reshape(1 if single else st.shape[0], -1)
        if st.shape[1] != m * (n + ncp):
            raise ConfigError("stream length must be M*(N+Ncp)")
        st = st.contiguous()
        out = torch.empty(st.shape[0], n, m, dtype=torch.complex64, device=self.device)
        self._stream()
        _check(self._lib.ofdmr_ofdm_demodulate(self._h, st.data_ptr(), out.data_ptr(), st.shape[0]))
        return out[0] if single else out

    def ofdm_modulate(self, x) -> torch.Tensor:
        """ofdm_modulate (waveform.cpp:133-149): N x M grid -> M x (N_cp + N) stream per frame
        (IFFT_N x 1/N per symbol, cyclic prefix = last N_cp samples)."""
        n, m, ncp = self.cfg.n_subcarriers, self.cfg.n_symbols, self.cfg.n_cp
        x, single = _batched(_as_grid(x, self.device))
        if tuple(x.shape[1:]) != (n, m):
            raise ConfigError("grid shape does not match config")
        out = torch.empty(x.shape[0], m, n + ncp, dtype=torch.complex64, device=self.device)
        self._stream()
        _check(self._lib.ofdmr_ofdm_modulate(self._h, x.data_ptr(), out.data_ptr(), x.shape[0]))
        return out[0] if single else out

    def map_to_pgm(self, p) -> torch.Tensor:
        """write_map_pgm's pixels (io.cpp:94-110) for a batch of maps, on the device: uint8
        (F, N', M'); io.write_pgm_bytes adds the header."""
        p = self._p_batch(p)
        out = torch.empty(p.shape, dtype=torch.uint8, device=self.device)
        self._stream()
        _check(self._lib.ofdmr_map_to_pgm(self._h, p.data_ptr(), out.data_ptr(), p.shape[0]))
        return out

    def estimate_noise_power(self, p) -> torch.Tensor:
        """estimate_noise_power (periodogram.cpp:146-152) per frame: the order statistic
        P[count / 2] of the map / ln 2 / window power factor (fp64, device)."""
        p = self._p_batch(p)
        F = p.shape[0]
        out = torch.empty(F, dtype=torch.float64, device=self.device)
        self._stream()
        _check(self._lib.ofdmr_estimate_noise_power(self._h, p.data_ptr(), out.data_ptr(), F))
        return out

    def extract_peaks(self, p, eta, k_per_frame=None) -> Detections:
        """extract_peaks (periodogram.cpp:89-136) on the mask p >= eta."""
        p = self._p_batch(p)
        F = p.shape[0]
        e = torch.as_tensor(np.broadcast_to(np.asarray(eta, np.float64), (F,)).copy()).to(self.device)
        k = self._k(k_per_frame, F)
        d = self._dets(F)
        self._stream()
        _check(self._lib.ofdmr_extract_peaks(self._h, p.data_ptr(), e.data_ptr(),
                                             k.data_ptr() if k is not None else None, d.delay_bin.data_ptr(),
                                             d.doppler_bin.data_ptr(), d.peak_power.data_ptr(), d.counts.data_ptr(), F))
        return d

    def pipeline(self, y, x_tx, sigma2, k_per_frame=None, want_map: bool = False, check: bool = True,
                 estimate_noise: bool = False):
        """Receiver half of run_pipeline (pipeline.cpp:72-96).  Returns (Detections, map|None).
        estimate_noise=True is the detector's estimate_noise mode (pipeline.cpp:86-87): the
        threshold uses estimate_noise_power(P) instead of sigma2 (which is then ignored);
        Detections.sigma2_h holds the estimate (the reference's sigma2_used)."""
        y, _ = _batched(_as_grid(y, self.device))
        x, _ = _batched(_as_grid(x_tx, self.device))
        if y.shape != x.shape:
            raise ConfigError("spectral_division: shape mismatch")
        self._shape_check(y)
        F = y.shape[0]
        if estimate_noise:
            h = self.estimate_channel(y, x, check=check)
            pm = self.periodogram(h)
            s2e = self.estimate_noise_power(pm)
            d = self.detect(pm, s2e, k_per_frame)
            d.sigma2_h = s2e
            return d, (pm if want_map else None)
        s2 = torch.as_tensor(np.broadcast_to(np.asarray(sigma2, np.float64), (F,)).copy()).to(self.device) \
            if not isinstance(sigma2, torch.Tensor) else sigma2.to(self.device, torch.float64).contiguous()
        k = self._k(k_per_frame, F)
        d = self._dets(F)
        d.sigma2_h = torch.empty(F, dtype=torch.float64, device=self.device)
        pmap = (torch.empty(F, self.cfg.n_prime, self.cfg.m_prime, dtype=torch.float32, device=self.device)
                if want_map else None)
        st = torch.empty(F, dtype=torch.int32, device=self.device)
        self.last_status = st  # per-frame status of the last pipeline call (bit 0 zero cell, bit 1 overflow)
        self._stream()
        _check(self._lib.ofdmr_pipeline(self._h, y.data_ptr(), x.data_ptr(), s2.data_ptr(),
                                        k.data_ptr() if k is not None else None, d.delay_bin.data_ptr(),
                                        d.doppler_bin.data_ptr(), d.peak_power.data_ptr(), d.counts.data_ptr(),
                                        d.sigma2_h.data_ptr(), pmap.data_ptr() if pmap is not None else None,
                                        st.data_ptr(), F))
        if check:
            over = torch.nonzero(st & 2).flatten()
            self.last_recomputed = int(over.numel())  # frames re-run on the exact general path
            if over.numel():
                # status bit 1: candidate-list overflow on the fused path, or an |x|^2 outside the fp32
                # normal range (zero / denormal / huge x cell): recompute those frames exactly on the
                # general path, whose status then decides the zero-cell error (bit 0)
                idx = over
                sub = self._dets(idx.numel())
                sub.sigma2_h = torch.empty(idx.numel(), dtype=torch.float64, device=self.device)
                ys, xs, ss = y[idx].contiguous(), x[idx].contiguous(), s2[idx].contiguous()
                ks = k[idx].contiguous() if k is not None else None
                st2 = torch.empty(idx.numel(), dtype=torch.int32, device=self.device)
                _check(self._lib.ofdmr_pipeline_general(
                    self._h, ys.data_ptr(), xs.data_ptr(), ss.data_ptr(), ks.data_ptr() if ks is not None else None,
                    sub.delay_bin.data_ptr(), sub.doppler_bin.data_ptr(), sub.peak_power.data_ptr(),
                    sub.counts.data_ptr(), sub.sigma2_h.data_ptr(), None, st2.data_ptr(), idx.numel()))
                d.delay_bin[idx] = sub.delay_bin
                d.doppler_bin[idx] = sub.doppler_bin
                d.peak_power[idx] = sub.peak_power
                d.counts[idx] = sub.counts
                d.sigma2_h[idx] = sub.sigma2_h
                st[idx] = st2
            self._raise_status(st)
        return d, pmap

    def pipeline_raw(self, y: torch.Tensor, x: torch.Tensor, s2: torch.Tensor, k: torch.Tensor | None,
                     d: Detections, frames: int, status: torch.Tensor | None = None) -> None:
        """Pre-allocated pipeline call for timing loops (no host sync); per-frame status flags go to
        `status` when given (checked by the caller after the timed region)."""
        _check(self._lib.ofdmr_pipeline(self._h, y.data_ptr(), x.data_ptr(), s2.data_ptr(),
                                        k.data_ptr() if k is not None else None, d.delay_bin.data_ptr(),
                                        d.doppler_bin.data_ptr(), d.peak_power.data_ptr(), d.counts.data_ptr(),
                                        None, None, status.data_ptr() if status is not None else None, frames))

    def pipeline_host(self, y: np.ndarray, x_tx: np.ndarray, sigma2: np.ndarray, k_per_frame=None):
        """Host-buffer pipeline (H2D / D2H inside the call).  Returns numpy records."""
        F = y.shape[0]
        for a in (y, x_tx):
            if a.dtype != np.complex64 or not a.flags["C_CONTIGUOUS"]:
                raise ConfigError("host frames must be C-contiguous complex64")
        s2 = np.ascontiguousarray(sigma2, np.float64)
        k = None if k_per_frame is None else np.ascontiguousarray(k_per_frame, np.int32)
        K = self.cfg.max_targets
        d = np.zeros((F, K), np.int32)
        dp = np.zeros((F, K), np.int32)
        pw = np.zeros((F, K), np.float32)
        cnt = np.zeros(F, np.int32)
        self._stream()
        _check(self._lib.ofdmr_pipeline_host(self._h, y.ctypes.data, x_tx.ctypes.data, s2.ctypes.data,
                                             k.ctypes.data if k is not None else None, d.ctypes.data, dp.ctypes.data,
                                             pw.ctypes.data, cnt.ctypes.data, F))
        return d, dp, pw, cnt

    def pipeline_host_ptr(self, y_ptr: int, x_ptr: int, s2_ptr: int, k_ptr, d_ptr: int, dp_ptr: int, pw_ptr: int,
                          cnt_ptr: int, frames: int) -> None:
        """Same as pipeline_host on raw (pinned) host pointers, for the e2e timing loop."""
        self._stream()
        _check(self._lib.ofdmr_pipeline_host(self._h, y_ptr, x_ptr, s2_ptr, k_ptr, d_ptr, dp_ptr, pw_ptr, cnt_ptr,
                                             frames))

    @staticmethod
    def _sft_config(i_max, detect_threshold, pfa, decimation, frac_tol, amp_tol, max_entries):
        c = _native.OfdmrSftConfig()
        c.i_max, c.detect_threshold, c.pfa, c.decimation = i_max, detect_threshold, pfa, decimation
        c.frac_tol, c.amp_tol, c.max_entries = frac_tol, amp_tol, max_entries
        return c

    def _f64_dev(self, v, F: int) -> torch.Tensor:
        if isinstance(v, torch.Tensor):
            return v.to(self.device, torch.float64).reshape(-1).expand(F).contiguous()
        return torch.as_tensor(np.broadcast_to(np.asarray(v, np.float64), (F,)).copy()).to(self.device)

    @staticmethod
    def _raise_sft_status(status: torch.Tensor) -> None:
        if bool((status & 1).any()):
            raise ConfigError("spectral_division: zero cell in X")
        if bool((status & 4).any()):
            raise ConfigError("sft: more than 128 accepted tones or 64 entries in a frame")

    def sft(self, h, seeds, sigma2, i_max: int = 10, detect_threshold: float = 0.0, pfa: float = 1e-2,
            decimation: int = 8, frac_tol: float = 0.25, amp_tol: float = 0.35, max_entries: int = 64,
            stream_ordered: bool = False):
        """sft_iterate (sft.cpp:185-459) over a batch; returns dict of device tensors.  The slope /
        offset draws run on the device from the per-frame seeds.  stream_ordered=True: no host sync,
        out["status"] bit 2 flags a frame beyond the on-chip limits (else ConfigError here)."""
        h, single = _batched(_as_grid(h, self.device))
        F, n, m = h.shape
        seeds = np.ascontiguousarray(np.broadcast_to(np.asarray(seeds, np.uint64), (F,)))
        s2 = np.ascontiguousarray(np.broadcast_to(np.asarray(sigma2, np.float64), (F,)))
        c = self._sft_config(i_max, detect_threshold, pfa, decimation, frac_tol, amp_tol, max_entries)
        z = dict(device=self.device)
        out = dict(k=torch.zeros(F, max_entries, dtype=torch.int32, **z),
                   l=torch.zeros(F, max_entries, dtype=torch.int32, **z),
                   amp=torch.zeros(F, max_entries, 2, dtype=torch.float64, **z),
                   n_entries=torch.zeros(F, dtype=torch.int32, **z),
                   iterations=torch.zeros(F, dtype=torch.int32, **z),
                   samples_used=torch.zeros(F, dtype=torch.int64, **z),
                   converged=torch.zeros(F, dtype=torch.int32, **z),
                   residual=torch.zeros(F, dtype=torch.float64, **z))
        if stream_ordered:
            out["status"] = torch.zeros(F, dtype=torch.int32, **z)
        self._stream()
        _check(self._lib.ofdmr_sft(self._h, h.data_ptr(), n, m, C.byref(c), seeds.ctypes.data, s2.ctypes.data,
                                   out["k"].data_ptr(), out["l"].data_ptr(), out["amp"].data_ptr(),
                                   out["n_entries"].data_ptr(), out["iterations"].data_ptr(),
                                   out["samples_used"].data_ptr(), out["converged"].data_ptr(),
                                   out["residual"].data_ptr(),
                                   out["status"].data_ptr() if stream_ordered else None, F))
        return out

    def sft_detections(self, out: dict, n: int, m: int, sigma2, pfa: float = 1e-2, k_per_frame=None) -> Detections:
        """detections_from_spectrum (sft.cpp:461-490) on the device for a batch of sft() outputs."""
        F = out["n_entries"].shape[0]
        me = out["k"].shape[1]
        s2 = self._f64_dev(sigma2, F)
        k = self._k(k_per_frame, F)
        d = self._dets(F)
        self._stream()
        _check(self._lib.ofdmr_sft_detections(self._h, out["k"].data_ptr(), out["l"].data_ptr(), out["amp"].data_ptr(),
                                              out["n_entries"].data_ptr(), me, n, m, s2.data_ptr(), pfa,
                                              k.data_ptr() if k is not None else None, d.delay_bin.data_ptr(),
                                              d.doppler_bin.data_ptr(), d.peak_power.data_ptr(), d.counts.data_ptr(), F))
        d.sigma2_h = s2
        return d

    def sft_detect(self, h, seeds, sigma2, pfa: float = 1e-2, i_max: int = 10, decimation: int = 8,
                   frac_tol: float = 0.25, amp_tol: float = 0.35, detect_threshold: float = 0.0, k_per_frame=None,
                   check: bool = True) -> Detections:
        """sft_detect (sft.cpp:492-500) over a batch: sft_iterate with sigma2 / pfa, then
        detections_from_spectrum, all on the device (ofdmr_sft_detect)."""
        h, _ = _batched(_as_grid(h, self.device))
        F, n, m = h.shape
        seeds = np.ascontiguousarray(np.broadcast_to(np.asarray(seeds, np.uint64), (F,)))
        s2 = self._f64_dev(sigma2, F)
        c = self._sft_config(i_max, detect_threshold, pfa, decimation, frac_tol, amp_tol, 64)
        k = self._k(k_per_frame, F)
        d = self._dets(F)
        st = torch.empty(F, dtype=torch.int32, device=self.device)
        self._stream()
        _check(self._lib.ofdmr_sft_detect(self._h, h.data_ptr(), n, m, C.byref(c), seeds.ctypes.data, s2.data_ptr(),
                                          k.data_ptr() if k is not None else None, d.delay_bin.data_ptr(),
                                          d.doppler_bin.data_ptr(), d.peak_power.data_ptr(), d.counts.data_ptr(),
                                          st.data_ptr(), F))
        self.last_status = st
        if check:
            self._raise_sft_status(st)
        d.sigma2_h = s2
        return d

    def pipeline_sft(self, y, x_tx, sigma2, sft_seeds, noise_seeds=None, i_max: int = 10, decimation: int = 8,
                     pfa: float | None = None, k_per_frame=None, check: bool = True) -> Detections:
        """The FPS-SFT branch of run_pipeline (pipeline.cpp:97-113) on a batch of frames, one
        C-ABI call (ofdmr_pipeline_sft): estimate_channel -> division_noise_power -> [estimate_noise_
        from_slice when noise_seeds is given] -> sft_iterate -> detections_from_spectrum.
        sft_seeds[f] / noise_seeds[f] are run_pipeline's derive_seed(seed, 0x736674) /
        derive_seed(seed, 0x6e6573).  Detections.sigma2_h = PipelineResult::sigma2_used."""
        y, _ = _batched(_as_grid(y, self.device))
        x, _ = _batched(_as_grid(x_tx, self.device))
        if y.shape != x.shape:
            raise ConfigError("spectral_division: shape mismatch")
        self._shape_check(y)
        F = y.shape[0]
        s2 = self._f64_dev(sigma2, F)
        ss = np.ascontiguousarray(np.broadcast_to(np.asarray(sft_seeds, np.uint64), (F,)))
        ns = None if noise_seeds is None else np.ascontiguousarray(
            np.broadcast_to(np.asarray(noise_seeds, np.uint64), (F,)))
        c = self._sft_config(i_max, 0.0, self.cfg.pfa if pfa is None else pfa, decimation, 0.25, 0.35, 64)
        k = self._k(k_per_frame, F)
        d = self._dets(F)
        d.sigma2_h = torch.empty(F, dtype=torch.float64, device=self.device)
        st = torch.empty(F, dtype=torch.int32, device=self.device)
        self._stream()
        _check(self._lib.ofdmr_pipeline_sft(self._h, y.data_ptr(), x.data_ptr(), s2.data_ptr(), ss.ctypes.data,
                                            ns.ctypes.data if ns is not None else None, C.byref(c),
                                            k.data_ptr() if k is not None else None, d.delay_bin.data_ptr(),
                                            d.doppler_bin.data_ptr(), d.peak_power.data_ptr(), d.counts.data_ptr(),
                                            d.sigma2_h.data_ptr(), st.data_ptr(), F))
        self.last_status = st
        if check:
            self._raise_sft_status(st)
        return d

    def estimate_noise_from_slice(self, h, seeds) -> torch.Tensor:
        """estimate_noise_from_slice (pipeline.cpp:26-43), the FPS-SFT detector's estimate-noise
        mode: seeds[f] is the Rng seed (run_pipeline passes derive_seed(seed, 0x6e6573))."""
        h, single = _batched(_as_grid(h, self.device))
        F, n, m = h.shape
        seeds = np.ascontiguousarray(np.broadcast_to(np.asarray(seeds, np.uint64), (F,)))
        out = torch.empty(F, dtype=torch.float64, device=self.device)
        self._stream()
        _check(self._lib.ofdmr_sft_estimate_noise(self._h, h.data_ptr(), n, m, seeds.ctypes.data, out.data_ptr(), F))
        return out[0] if single else out


class MultiReceiver:
    """ofdmr_multi (include/ofdmr_b200.h): one context per listed device, frames sharded in
    contiguous ranges (shard.shard_range), detections gathered to the host (pipeline_host) or to
    the first device by peer copies (pipeline on per-device shards)."""

    def __init__(self, rc: RadarConfig, devices, chunk_frames: int = 0):
        self._lib = _native.lib()
        cfg = _native.OfdmrConfig()
        cfg.n_subcarriers, cfg.n_symbols, cfg.n_prime, cfg.m_prime = rc.n, rc.m, rc.n_prime, rc.m_prime
        cfg.window, cfg.estimator, cfg.n_cp = rc.window, rc.estimator, rc.n_cp
        cfg.max_targets, cfg.pfa, cfg.chunk_frames, cfg.device = rc.max_targets, rc.pfa, chunk_frames, 0
        self.cfg = cfg
        self.devices = [int(d) for d in devices]
        arr = (C.c_int32 * len(self.devices))(*self.devices)
        h = C.c_void_p()
        rc_ = self._lib.ofdmr_multi_create(C.byref(cfg), arr, len(self.devices), C.byref(h))
        if rc_:
            msg = self._lib.ofdmr_multi_last_error().decode()
            raise ConfigError(msg) if rc_ == 2 else CudaError(msg)
        self._h = h

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.ofdmr_multi_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _check(self, rc_: int) -> None:
        if rc_:
            msg = self._lib.ofdmr_multi_last_error().decode()
            raise ConfigError(msg) if rc_ == 2 else CudaError(msg)

    def shard_range(self, frames: int, rank: int) -> tuple[int, int]:
        lo, hi = C.c_int64(), C.c_int64()
        self._lib.ofdmr_shard_range(frames, rank, len(self.devices), C.byref(lo), C.byref(hi))
        return lo.value, hi.value

    def pipeline_host(self, y: np.ndarray, x_tx: np.ndarray, sigma2, k_per_frame=None):
        """ofdmr_multi_pipeline_host: numpy records (delay, doppler, power, counts)."""
        F = y.shape[0]
        y = np.ascontiguousarray(y, np.complex64)
        x = np.ascontiguousarray(x_tx, np.complex64)
        s2 = np.ascontiguousarray(sigma2, np.float64)
        k = None if k_per_frame is None else np.ascontiguousarray(k_per_frame, np.int32)
        K = self.cfg.max_targets
        d, dp = np.zeros((F, K), np.int32), np.zeros((F, K), np.int32)
        pw, cnt = np.zeros((F, K), np.float32), np.zeros(F, np.int32)
        self._check(self._lib.ofdmr_multi_pipeline_host(self._h, y.ctypes.data, x.ctypes.data, s2.ctypes.data,
                                                        k.ctypes.data if k is not None else None, d.ctypes.data,
                                                        dp.ctypes.data, pw.ctypes.data, cnt.ctypes.data, F))
        return d, dp, pw, cnt

    def pipeline(self, ys, xs, s2s, ks=None) -> tuple[Detections, torch.Tensor]:
        """ofdmr_multi_pipeline on per-device shards (lists of tensors, shard r on devices[r]);
        returns the gathered Detections and status on the first device."""
        F = sum(int(t.shape[0]) for t in ys)
        for r, t in enumerate(ys):
            lo, hi = self.shard_range(F, r)
            if int(t.shape[0]) != hi - lo:
                raise ConfigError("shard sizes must follow ofdmr_shard_range")
        G = len(self.devices)
        vp = C.c_void_p
        arr = lambda ts: (vp * G)(*[t.data_ptr() if t is not None else None for t in ts])  # noqa: E731
        dev0 = torch.device("cuda", self.devices[0])
        K = self.cfg.max_targets
        z = dict(device=dev0)
        d = Detections(torch.zeros(F, K, dtype=torch.int32, **z), torch.zeros(F, K, dtype=torch.int32, **z),
                       torch.zeros(F, K, dtype=torch.float32, **z), torch.zeros(F, dtype=torch.int32, **z))
        st = torch.zeros(F, dtype=torch.int32, **z)
        for dv in set(self.devices):
            torch.cuda.synchronize(dv)  # inputs produced on torch's streams are ready
        self._check(self._lib.ofdmr_multi_pipeline(self._h, arr(ys), arr(xs), arr(s2s),
                                                   arr(ks) if ks is not None else None, d.delay_bin.data_ptr(),
                                                   d.doppler_bin.data_ptr(), d.peak_power.data_ptr(),
                                                   d.counts.data_ptr(), st.data_ptr(), F))
        return d, st


# ---------------------------------------------------------------------------------
# Module-level functions with the reference's names (single frame, value semantics).

_ctx_cache: dict = {}


def _ctx(n, m, np_, mp, window, estimator, n_cp, max_targets=64, pfa=1e-2) -> Receiver:
    key = (torch.cuda.current_device(), n, m, np_, mp, window, estimator, n_cp, max_targets, pfa)
    r = _ctx_cache.get(key)
    if r is None:
        r = Receiver(n, m, np_, mp, window, estimator, n_cp, max_targets, pfa)
        _ctx_cache[key] = r
    return r


@dataclass
class Window2d:
    """Window2d (periodogram.hpp:21-30)."""

    kind: int
    subcarrier: np.ndarray
    symbol: np.ndarray

    def power_factor(self) -> float:
        return float(_native.lib().ofdmr_window_power_factor(self.kind, len(self.subcarrier), len(self.symbol)))


def make_window(kind, n: int, m: int) -> Window2d:
    """periodogram.cpp:25-37."""
    k = _window_code(kind)
    wk = np.empty(n, np.float64)
    wl = np.empty(m, np.float64)
    _check(_native.lib().ofdmr_make_window(k, n, m, wk.ctypes.data_as(_native.P_f64), wl.ctypes.data_as(_native.P_f64)))
    return Window2d(k, wk, wl)


def spectral_division(y, x) -> torch.Tensor:
    y = _as_grid(y, _device())
    if y.dim() != 2:
        raise ConfigError("spectral_division takes one (N, M) grid")
    if tuple(_as_grid(x, _device()).shape) != tuple(y.shape):
        raise ConfigError("spectral_division: shape mismatch")
    n, m = y.shape
    return _ctx(n, m, n, m, WINDOW_RECT, EST_LS, 0).spectral_division(y, x)


def dft_ce(h, n_cp: int) -> torch.Tensor:
    h = _as_grid(h, _device())
    n, m = h.shape
    if n_cp > n:
        raise ConfigError("dft_ce: truncation length exceeds N")
    return _ctx(n, m, n, m, WINDOW_RECT, EST_DFT_CE, n_cp).dft_ce(h)


def periodogram(h, window: Window2d, n_prime: int, m_prime: int) -> torch.Tensor:
    h = _as_grid(h, _device())
    n, m = h.shape
    if n_prime < n or m_prime < m:
        raise ConfigError("periodogram: N' >= N and M' >= M required")
    if len(window.subcarrier) != n or len(window.symbol) != m:
        raise ConfigError("periodogram: window shape mismatch")
    return _ctx(n, m, n_prime, m_prime, window.kind, EST_LS, 0).periodogram(h)


def detection_threshold(sigma2: float, pfa: float, window_power_factor: float) -> float:
    eta = C.c_double()
    _check(_native.lib().ofdmr_detection_threshold(sigma2, pfa, window_power_factor, C.byref(eta)))
    return eta.value


def threshold_mask(p: torch.Tensor, eta: float) -> torch.Tensor:
    """periodogram.cpp:83-87 (elementwise, device-side)."""
    return (p.double() >= eta).to(torch.uint8)


@dataclass
class Detection:
    delay_bin: int
    doppler_bin: int
    peak_power: float
    range_m: float = 0.0
    velocity_mps: float = 0.0


def bins_to_physics(det: Detection, rc: RadarConfig) -> Detection:
    """periodogram.cpp:138-144 (fp64, host)."""
    r = C.c_double()
    v = C.c_double()
    _native.lib().ofdmr_bins_to_physics(det.delay_bin, det.doppler_bin, rc.n, rc.n_cp, rc.n_prime, rc.m_prime,
                                        rc.df_hz, 77e9, C.byref(r), C.byref(v))
    det.range_m, det.velocity_mps = r.value, v.value
    return det


def extract_peaks(p: torch.Tensor, eta: float, max_targets: int, rc: RadarConfig | None = None) -> list[Detection]:
    """extract_peaks (periodogram.cpp:89-136) on the mask p >= eta (the mask argument is
    represented by its threshold); physics filled when a RadarConfig is given."""
    p = _as_grid(p, _device(), torch.float32)
    np_, mp = p.shape
    if max_targets > 64:
        raise ConfigError("extract_peaks: max_targets <= 64 on the GPU path")
    if np_ < 16 or mp < 16:
        # the device contexts take power-of-two dimensions >= 16 (include/ofdmr_b200.h)
        raise ConfigError("extract_peaks: maps smaller than 16 x 16 are not supported on the GPU path")
    r = _ctx(np_, mp, np_, mp, WINDOW_RECT, EST_LS, 0, max_targets)
    d = r.extract_peaks(p, eta)
    out = [Detection(a, b, c) for a, b, c in d.frame(0)]
    if rc is not None:
        for det in out:
            bins_to_physics(det, rc)
    return out


def sft_iterate(h, seed: int, sigma2: float = 0.0, i_max: int = 10, detect_threshold: float = 0.0,
                pfa: float = 1e-2, decimation: int = 8, frac_tol: float = 0.25, amp_tol: float = 0.35) -> SparseSpectrum:
    """sft.cpp:185-459 for one grid."""
    h = _as_grid(h, _device())
    n, m = h.shape
    r = _ctx(16, 16, 16, 16, WINDOW_RECT, EST_LS, 0)
    o = r.sft(h, [seed], [sigma2], i_max, detect_threshold, pfa, decimation, frac_tol, amp_tol, 64)
    ne = int(o["n_entries"][0])
    k = o["k"][0].tolist()
    l = o["l"][0].tolist()
    a = o["amp"][0].cpu().numpy()
    ents = [(k[i], l[i], complex(a[i, 0], a[i, 1])) for i in range(min(ne, 64))]
    return SparseSpectrum(ents, float(o["residual"][0]), bool(o["converged"][0]), int(o["iterations"][0]),
                          int(o["samples_used"][0]))


def detections_from_spectrum(spec: SparseSpectrum, n: int, m: int, sigma2: float, pfa: float, max_targets: int,
                             rc: RadarConfig | None = None) -> list[Detection]:
    """sft.cpp:461-490 through the device entry point (ofdmr_sft_detections): threshold, bin
    mapping and the (power desc, delay, Doppler) ranking in fp64 on the GPU; peak_power is the
    fp64 |A|^2 N M of the matching entry, physics as sft.cpp:476-479 when a RadarConfig is given."""
    if sigma2 < 0:
        raise ConfigError("threshold: sigma2 must be >= 0")
    if not (0 < pfa <= 1):
        raise ConfigError("threshold: pfa must lie in (0,1]")
    if not spec.entries or max_targets <= 0:
        return []
    if len(spec.entries) > 64 or max_targets > 64:
        raise ConfigError("detections_from_spectrum: at most 64 entries / targets on the GPU path")
    dev = _device()
    r = _ctx(16, 16, 16, 16, WINDOW_RECT, EST_LS, 0, max_targets)
    ne = len(spec.entries)
    out = {"k": torch.tensor([[e[0] for e in spec.entries]], dtype=torch.int32, device=dev),
           "l": torch.tensor([[e[1] for e in spec.entries]], dtype=torch.int32, device=dev),
           "amp": torch.tensor([[[e[2].real, e[2].imag] for e in spec.entries]], dtype=torch.float64, device=dev),
           "n_entries": torch.tensor([ne], dtype=torch.int32, device=dev)}
    d = r.sft_detections(out, n, m, [sigma2], pfa)
    nm = float(n) * float(m)
    amp = {(int(k) % n, int(l) % m): a for k, l, a in spec.entries}
    dets = []
    for db, vb, _ in d.frame(0):
        a = amp[((n - db) % n, vb % m)]
        det = Detection(db, vb, (a.real * a.real + a.imag * a.imag) * nm)
        if rc is not None:
            det.range_m = KSPEED_OF_LIGHT * db / (2.0 * n * rc.df_hz)
            det.velocity_mps = KSPEED_OF_LIGHT * vb / (2.0 * 77e9 * m * rc.symbol_time)
        dets.append(det)
    return dets


def sft_detect(h, seed: int, sigma2: float, pfa: float, max_targets: int, **kw) -> list[Detection]:
    """sft.cpp:492-500 (one grid): sft_iterate + detections_from_spectrum on the device."""
    h = _as_grid(h, _device())
    n, m = h.shape
    r = _ctx(16, 16, 16, 16, WINDOW_RECT, EST_LS, 0, max_targets)
    d = r.sft_detect(h, [seed], [sigma2], pfa=pfa, **kw)
    return [Detection(a, b, c) for a, b, c in d.frame(0)]
