"""GPU counterpart of the reference's estimator timing harness, bench_estimators
(metrics.cpp:145-253): for each subcarrier count N, K distinct on-bin targets inside the CP
window and the velocity-model bound, one frame from the seeded generator, the LS channel
estimate, and then the two detectors on the SAME channel estimate:

  periodogram   periodogram(h, window, N, M) -> threshold -> extract_peaks(K)   (ofdmr_periodogram + ofdmr_detect)
  FPS-SFT       sft_iterate(h, {seed = derive_seed(run_seed, 0x736674), sigma2_h, pfa})
                -> detections_from_spectrum(K)                                   (ofdmr_sft_detect)

Their support sets must agree before anything is timed (metrics.cpp:220-231); then both are
timed `repeats` times and the medians reported with periodogram_ms / sft_ms (the paper's headline
claim is this ratio).  Every step is the reference's, with the reference's random
streams:
  targets   Rng(derive_seed(seed, N)): delay 1 + uniform_int(n_cp - 2), Doppler
            uniform_int(2 D + 1) - D with D = max(1, floor(0.1 v_bound / v_res) - 1), redrawn while
            within 2 bins of an accepted target in either axis (metrics.cpp:160-186)
  frame     run seed derive_seed(seed, 31 N + 7): make_random_frame + apply_channel
            (ofdmr_gen_device_explicit, metrics.cpp:188-192)
GPU timings are CUDA-event medians on the context stream; besides the single-frame latency the
reference measures, the batched rate of each detector over `batch` copies of the frame is
reported (the GPU's natural operating point).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math

import numpy as np

from . import _native, gen
from .configs import RadarConfig

C_LIGHT = 3.0e8
K_VELOCITY_MARGIN = 0.1  # channel.hpp:25


@dataclasses.dataclass
class BenchRow:
    n: int
    m: int
    k: int
    periodogram_ms: float
    sft_ms: float
    speedup: float
    samples_used: int
    support: list
    periodogram_batch_frames_per_s: float | None = None
    sft_batch_frames_per_s: float | None = None


class _Rng:
    """Rng (rng.hpp): MT19937-64 via the generator library; uniform_int with the reference's
    rejection rule."""

    def __init__(self, seed: int):
        self.seed = seed
        self.buf = gen.rng_u64(seed, 4096)
        self.pos = 0

    def next(self) -> int:
        if self.pos >= len(self.buf):
            self.buf = gen.rng_u64(self.seed, 2 * len(self.buf))
        v = int(self.buf[self.pos])
        self.pos += 1
        return v

    def uniform_int(self, n: int) -> int:
        m64 = (1 << 64) - 1
        limit = m64 - m64 % n
        while True:
            v = self.next()
            if v < limit:
                return v % n


def _targets(cfg: RadarConfig, k_targets: int, seed: int):
    """metrics.cpp:160-186."""
    ts = (1.0 / cfg.df_hz) + cfg.n_cp * ((1.0 / cfg.df_hz) / cfg.n)
    v_res = C_LIGHT / (2.0 * cfg.m * 77e9 * ts)
    v_bound = C_LIGHT * cfg.df_hz / (2.0 * 77e9)
    max_doppler = max(1, int(K_VELOCITY_MARGIN * v_bound / v_res) - 1)
    rng = _Rng(gen.derive_seed(seed, cfg.n))
    used_d, used_v, ranges, vels = [], [], [], []
    while len(ranges) < k_targets:
        db = 1 + rng.uniform_int(cfg.n_cp - 2)
        vb = rng.uniform_int(2 * max_doppler + 1) - max_doppler
        if any(abs(d - db) < 2 or abs(v - vb) < 2 for d, v in zip(used_d, used_v)):
            continue
        used_d.append(db)
        used_v.append(vb)
        ranges.append(C_LIGHT * db / (2.0 * cfg.n * cfg.df_hz))
        vels.append(C_LIGHT * vb / (2.0 * 77e9 * cfg.m * ts))
    return np.array(ranges), np.array(vels), list(zip(used_d, used_v))


def bench_estimators(base: RadarConfig, sizes, k_targets: int, repeats: int, seed: int, snr_db: float = 40.0,
                     batch: int = 256, bandwidth_hz: float | None = None, device=None) -> list[BenchRow]:
    """metrics.cpp:145-253 on the GPU.  `base` supplies M, QAM, window and P_fa; the bandwidth
    N * df is kept (bandwidth_hz, default the base's) while N sweeps `sizes` with n_cp = N / 4,
    N' = N, M' = M (metrics.cpp:152-158).  snr_db is the scenario's channel SNR (fig6: 40 dB)."""
    import torch

    from .receiver import ConfigError, Receiver

    if repeats < 1:
        raise ConfigError("bench: repeats must be >= 1")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    bandwidth = bandwidth_hz if bandwidth_hz is not None else base.df_hz * base.n
    lib = _native.lib()
    rows = []
    for n in sizes:
        cfg = base.replace(n=n, n_prime=n, m_prime=base.m, n_cp=n // 4, max_targets=k_targets,
                           snr_lo_db=snr_db, snr_hi_db=snr_db, zc_precode=False)
        df = bandwidth / n
        # RadarConfig derives df from its fixed B; the spacing goes through the generator params
        ranges, vels, support_truth = _targets(_with_df(cfg, df), k_targets, seed)
        p = gen.gen_params(cfg)
        p.df_hz = df
        y = torch.empty(1, n, cfg.m, dtype=torch.complex64, device=dev)
        x = torch.empty_like(y)
        s2 = torch.empty(1, dtype=torch.float64, device=dev)
        st = torch.empty(1, dtype=torch.int32, device=dev)
        stream = torch.cuda.current_stream(dev).cuda_stream
        rc = lib.ofdmr_gen_device_explicit(C.byref(p), seed, n * 31 + 7, 1, ranges.ctypes.data_as(_native.P_f64),
                                           vels.ctypes.data_as(_native.P_f64), len(ranges), float(snr_db),
                                           y.data_ptr(), x.data_ptr(), s2.data_ptr(), st.data_ptr(), None,
                                           C.c_void_p(stream))
        if rc or int(st.item()):
            raise RuntimeError(f"generator failed ({rc}, status {int(st.item())})")
        run_seed = gen.derive_seed(seed, n * 31 + 7)
        with Receiver(n, cfg.m, n, cfg.m, window=cfg.window, estimator="ls", max_targets=k_targets,
                      pfa=cfg.pfa, device=dev.index) as rx:
            h = rx.spectral_division(y, x)
            # sigma2_h = realization.sigma2 * mean(1 / |x|^2) (metrics.cpp:193-195), fp64 on the c64 x
            xx = x.to(torch.complex128)
            s2h = s2 * (1.0 / (xx.real ** 2 + xx.imag ** 2)).sum(dim=(1, 2)) / float(n * cfg.m)
            sft_seed = gen.derive_seed(run_seed, 0x736674)

            def run_periodogram(hh, s2b):
                return rx.detect(rx.periodogram(hh), s2b)

            def run_sft(hh, s2b, seeds):
                return rx.sft_detect(hh, seeds, s2b, pfa=cfg.pfa, i_max=10)

            det_p = run_periodogram(h, s2h)
            det_s = run_sft(h, s2h, [sft_seed])
            sup_p = sorted((a, b) for a, b, _ in det_p.frame(0))
            sup_s = sorted((a, b) for a, b, _ in det_s.frame(0))
            if sup_p != sup_s:
                raise RuntimeError(f"bench: detector support sets differ at N={n}: {sup_p} vs {sup_s}")
            # samples_used of the SFT run (SparseSpectrum stats)
            o = rx.sft(h, [sft_seed], s2h.cpu().numpy(), i_max=10, pfa=cfg.pfa)
            samples = int(o["samples_used"][0])

            def timed(fn, reps):
                ts_ = []
                for _ in range(reps):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    rx._stream()
                    e0.record()
                    fn()
                    e1.record()
                    torch.cuda.synchronize()
                    ts_.append(e0.elapsed_time(e1))
                return float(np.median(ts_))

            timed(lambda: run_periodogram(h, s2h), 2)
            timed(lambda: run_sft(h, s2h, [sft_seed]), 2)
            tp = timed(lambda: run_periodogram(h, s2h), max(repeats, 5))
            tsft = timed(lambda: run_sft(h, s2h, [sft_seed]), max(repeats, 5))
            # batched: `batch` copies of the frame per call
            hb = h.reshape(1, n, cfg.m).expand(batch, n, cfg.m).contiguous()
            s2b = s2h.expand(batch).contiguous()
            seeds_b = [sft_seed] * batch
            tpb = timed(lambda: run_periodogram(hb, s2b), 3)
            tsb = timed(lambda: run_sft(hb, s2b, seeds_b), 3)
            del hb
        rows.append(BenchRow(n, cfg.m, k_targets, tp, tsft, tp / tsft, samples, sup_p,
                             batch / (tpb / 1e3), batch / (tsb / 1e3)))
    return rows


def _with_df(cfg: RadarConfig, df: float):
    """A view of cfg whose df_hz is `df` (RadarConfig derives it from the fixed bandwidth)."""

    class _V:
        pass

    v = _V()
    v.n, v.m, v.n_cp, v.df_hz = cfg.n, cfg.m, cfg.n_cp, df
    return v
