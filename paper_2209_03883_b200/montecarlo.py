"""Monte-Carlo callers on the GPU receiver.

`rmse_sweep` mirrors the reference's `rmse_sweep` (src/metrics.cpp:92-120) and `mse_sweep` its
`mse_sweep` (metrics.cpp:122-143).  rmse_sweep: for every SNR of
the grid, `trials` runs of run_pipeline on a fixed scenario (run seed derive_seed(seed, t),
max_targets = number of targets), detections matched to the truths by `match_detections`
(metrics.cpp:36-72) and reduced to range / velocity RMSE and miss rate.  The frames come from
the GPU generator (`ofdmr_gen_device_explicit`, the same streams as run_pipeline's generator
half) and are processed in batches by the fused GPU pipeline; only the detection records
(bins) travel to the host, where the physics conversion (periodogram.cpp:138-144), the
resolutions (waveform.cpp:41-54) and the greedy matching run in fp64 in the reference's
operation order.

Differences from the reference: the frames are quantised to c64 and the receiver computes in
fp32 (fp64 for σ_h² and η), so a trial's detections can differ from the fp64 reference only
at fp32-unresolvable near-ties (SURVEY.md §8d parity rules); the host-side reduction is exact
(tests/test_montecarlo.py pins it against the reference's own rmse_sweep).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _native
from .configs import RadarConfig

C_LIGHT = 3.0e8  # kSpeedOfLight, waveform.hpp:14


@dataclass
class RmseRow:
    snr_db: float
    estimator: str
    range_rmse_m: float
    velocity_rmse_mps: float
    miss_rate: float
    trials: int


def symbol_time(cfg: RadarConfig) -> float:
    """WaveformConfig::symbol_time (waveform.hpp:32-35): T + n_cp * (T / N)."""
    t = 1.0 / cfg.df_hz
    return t + float(cfg.n_cp) * (t / float(cfg.n))


def resolutions(cfg: RadarConfig, fc: float = 77e9) -> dict:
    """waveform.cpp:41-54 (the fields match_detections uses)."""
    df = cfg.df_hz
    ts = symbol_time(cfg)
    cp_time = float(cfg.n_cp) * ((1.0 / df) / float(cfg.n))
    return {
        "range_resolution_m": C_LIGHT / (2.0 * float(cfg.n) * df),
        "velocity_resolution_mps": C_LIGHT / (2.0 * float(cfg.m) * fc * ts),
        "unambiguous_velocity_mps": C_LIGHT / (2.0 * fc * ts),
        "cp_range_limit_m": C_LIGHT * cp_time / 2.0,
    }


def bins_to_physics(delay_bin: int, doppler_bin: int, cfg: RadarConfig, fc: float = 77e9) -> tuple[float, float]:
    """periodogram.cpp:138-144 bins_to_physics."""
    r = C_LIGHT * float(delay_bin) / (2.0 * float(cfg.n_prime) * cfg.df_hz)
    v = C_LIGHT * float(doppler_bin) / (2.0 * fc * float(cfg.m_prime) * symbol_time(cfg))
    return r, v


class MatchStats:
    def __init__(self):
        self.sum_sq_range = 0.0
        self.sum_sq_velocity = 0.0
        self.misses = 0
        self.truths = 0


def match_detections(dets: list[tuple[float, float]], truths: list[tuple[float, float]], res: dict,
                     stats: MatchStats) -> None:
    """metrics.cpp:36-72: greedy nearest neighbour in resolution-normalised (range, velocity),
    miss penalties d_max and v_un/2, matched errors capped at the penalties."""
    pen_r = res["cp_range_limit_m"]
    pen_v = res["unambiguous_velocity_mps"] / 2.0
    det_used = [False] * len(dets)
    truth_used = [False] * len(truths)
    for _ in range(min(len(dets), len(truths))):
        best = math.inf
        bi = bj = 0
        for i, (tr, tv) in enumerate(truths):
            if truth_used[i]:
                continue
            for j, (dr_m, dv_m) in enumerate(dets):
                if det_used[j]:
                    continue
                dr = (tr - dr_m) / res["range_resolution_m"]
                dv = (tv - dv_m) / res["velocity_resolution_mps"]
                d = dr * dr + dv * dv
                if d < best:
                    best, bi, bj = d, i, j
        if not math.isfinite(best):
            break
        truth_used[bi] = True
        det_used[bj] = True
        er = min(abs(truths[bi][0] - dets[bj][0]), pen_r)
        ev = min(abs(truths[bi][1] - dets[bj][1]), pen_v)
        stats.sum_sq_range += er * er
        stats.sum_sq_velocity += ev * ev
    for i in range(len(truths)):
        if not truth_used[i]:
            stats.misses += 1
            stats.sum_sq_range += pen_r * pen_r
            stats.sum_sq_velocity += pen_v * pen_v
    stats.truths += len(truths)


def finish_row(snr: float, estimator: str, stats: MatchStats, trials: int) -> RmseRow:
    return RmseRow(snr, estimator, math.sqrt(stats.sum_sq_range / float(stats.truths)),
                   math.sqrt(stats.sum_sq_velocity / float(stats.truths)),
                   float(stats.misses) / float(stats.truths), trials)


def rmse_sweep(cfg: RadarConfig, ranges, vels, snr_grid_db, trials: int, seed: int, batch: int = 2048,
               device=None) -> list[RmseRow]:
    """metrics.cpp:92-120 on the GPU (generator + fused receiver); see the module docstring."""
    import torch

    from . import gen
    from .receiver import ConfigError, Receiver

    if trials < 1:
        raise ValueError("rmse_sweep: trials must be >= 1")
    ranges = np.ascontiguousarray(ranges, np.float64)
    vels = np.ascontiguousarray(vels, np.float64)
    T = len(ranges)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    rcfg = cfg.replace(max_targets=max(T, 1), per_frame_k=False)
    truths = list(zip(ranges.tolist(), vels.tolist()))
    res = resolutions(cfg)
    est_name = {0: "ls", 1: "dft-ce"}.get(cfg.estimator, "?")
    p = gen.gen_params(cfg)
    lib = _native.lib()
    rows = []
    B = min(batch, trials)
    K = rcfg.max_targets
    pin = dict(dtype=torch.int32, pin_memory=True)
    with Receiver.from_config(rcfg, device=dev.index) as rx:
        # two batch slots: the GPU generates and receives batch j while the host matches batch j - 1
        slots = []
        for _ in range(2):
            slots.append(dict(
                y=torch.empty(B, cfg.n, cfg.m, dtype=torch.complex64, device=dev),
                x=torch.empty(B, cfg.n, cfg.m, dtype=torch.complex64, device=dev),
                s2=torch.empty(B, dtype=torch.float64, device=dev),
                gst=torch.empty(B, dtype=torch.int32, device=dev),
                pst=torch.empty(B, dtype=torch.int32, device=dev),
                d=rx._dets(B),
                h_delay=torch.empty(B, K, **pin), h_dopp=torch.empty(B, K, **pin), h_cnt=torch.empty(B, **pin),
                h_gst=torch.empty(B, **pin), h_pst=torch.empty(B, **pin), ev=torch.cuda.Event()))

        def enqueue(sl, snr, t0, nb):
            stream = torch.cuda.current_stream(dev).cuda_stream
            rc = lib.ofdmr_gen_device_explicit(C.byref(p), seed, t0, nb, ranges.ctypes.data_as(_native.P_f64),
                                               vels.ctypes.data_as(_native.P_f64), T, float(snr), sl["y"].data_ptr(),
                                               sl["x"].data_ptr(), sl["s2"].data_ptr(), sl["gst"].data_ptr(), None,
                                               C.c_void_p(stream))
            if rc:
                raise RuntimeError(f"ofdmr_gen_device_explicit failed ({rc})")
            d = sl["d"]
            rx._stream()
            rc = rx._lib.ofdmr_pipeline(rx._h, sl["y"].data_ptr(), sl["x"].data_ptr(), sl["s2"].data_ptr(), None,
                                        d.delay_bin.data_ptr(), d.doppler_bin.data_ptr(), d.peak_power.data_ptr(),
                                        d.counts.data_ptr(), None, None, sl["pst"].data_ptr(), nb)
            if rc:
                raise RuntimeError(f"ofdmr_pipeline failed ({rc})")
            for src, dst in ((d.delay_bin, "h_delay"), (d.doppler_bin, "h_dopp"), (d.counts, "h_cnt"),
                             (sl["gst"], "h_gst"), (sl["pst"], "h_pst")):
                sl[dst][:nb].copy_(src[:nb], non_blocking=True)
            sl["ev"].record()

        def finish(sl, nb, stats):
            sl["ev"].synchronize()
            if int(sl["h_gst"][:nb].sum()):
                raise RuntimeError("generator rejection draw (regenerate on the CPU)")
            pst = sl["h_pst"][:nb].numpy()
            if (pst & 1).any():
                raise ConfigError("spectral_division: zero cell in X")
            dd, vv, cc = sl["h_delay"][:nb].numpy(), sl["h_dopp"][:nb].numpy(), sl["h_cnt"][:nb].numpy()
            over = np.flatnonzero(pst & 2)
            if over.size:  # fused-path candidate overflow: those frames exactly, as Receiver.pipeline does
                dets, _ = rx.pipeline(sl["y"][torch.as_tensor(over, device=dev)],
                                      sl["x"][torch.as_tensor(over, device=dev)],
                                      sl["s2"][torch.as_tensor(over, device=dev)])
                dd, vv, cc = dd.copy(), vv.copy(), cc.copy()
                dd[over] = dets.delay_bin.cpu().numpy()
                vv[over] = dets.doppler_bin.cpu().numpy()
                cc[over] = dets.counts.cpu().numpy()
            for i in range(nb):
                phys = [bins_to_physics(int(dd[i, j]), int(vv[i, j]), cfg) for j in range(int(cc[i]))]
                match_detections(phys, truths, res, stats)

        # batches of every SNR point in one stream of work: the host matches batch j - 1 (which may
        # belong to the previous SNR point) while the GPU generates and receives batch j
        all_stats = [MatchStats() for _ in snr_grid_db]
        pending = None
        bi = 0
        for si, snr in enumerate(snr_grid_db):
            for t0 in range(0, trials, B):
                nb = min(B, trials - t0)
                sl = slots[bi % 2]
                bi += 1
                enqueue(sl, snr, t0, nb)
                if pending is not None:
                    finish(*pending)
                pending = (sl, nb, all_stats[si])
        if pending is not None:
            finish(*pending)
        for si, snr in enumerate(snr_grid_db):
            rows.append(finish_row(float(snr), est_name, all_stats[si], trials))
    return rows


@dataclass
class MseRow:
    snr_db: float
    estimator: str
    channel_mse: float


def mse_sweep(cfg: RadarConfig, ranges, vels, snr_grid_db, trials: int, seed: int, batch: int = 512,
              device=None) -> list[MseRow]:
    """metrics.cpp:122-143 on the GPU: per trial, the generator's true channel (c128) against
    estimate_channel on the GPU (LS or DFT-CE per cfg.estimator), channel_mse per trial on the
    device, accumulated over trials in trial order on the host (as the reference does)."""
    import torch

    from . import gen
    from .receiver import Receiver

    if trials < 1:
        raise ValueError("mse_sweep: trials must be >= 1")
    ranges = np.ascontiguousarray(ranges, np.float64)
    vels = np.ascontiguousarray(vels, np.float64)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    est_name = {0: "ls", 1: "dft-ce"}.get(cfg.estimator, "?")
    p = gen.gen_params(cfg)
    lib = _native.lib()
    B = min(batch, trials)
    y = torch.empty(B, cfg.n, cfg.m, dtype=torch.complex64, device=dev)
    x = torch.empty(B, cfg.n, cfg.m, dtype=torch.complex64, device=dev)
    ht = torch.empty(B, cfg.n, cfg.m, dtype=torch.complex128, device=dev)
    s2 = torch.empty(B, dtype=torch.float64, device=dev)
    st = torch.empty(B, dtype=torch.int32, device=dev)
    mse = torch.empty(B, dtype=torch.float64, device=dev)
    rows = []
    with Receiver.from_config(cfg, device=dev.index) as rx:
        for snr in snr_grid_db:
            acc = 0.0
            for t0 in range(0, trials, B):
                nb = min(B, trials - t0)
                stream = torch.cuda.current_stream(dev).cuda_stream
                rc = lib.ofdmr_gen_device_explicit(C.byref(p), seed, t0, nb, ranges.ctypes.data_as(_native.P_f64),
                                                   vels.ctypes.data_as(_native.P_f64), len(ranges), float(snr),
                                                   y.data_ptr(), x.data_ptr(), s2.data_ptr(), st.data_ptr(),
                                                   ht.data_ptr(), C.c_void_p(stream))
                if rc or int(st[:nb].sum().item()):
                    raise RuntimeError(f"ofdmr_gen_device_explicit failed ({rc})")
                h = rx.estimate_channel(y[:nb], x[:nb])
                rc = lib.ofdmr_channel_mse(h.data_ptr(), ht.data_ptr(), cfg.n * cfg.m, nb, mse.data_ptr(),
                                           C.c_void_p(stream))
                if rc:
                    raise RuntimeError(f"ofdmr_channel_mse failed ({rc})")
                for v in mse[:nb].cpu().numpy().tolist():
                    acc += v
            rows.append(MseRow(float(snr), est_name, acc / float(trials)))
    return rows
