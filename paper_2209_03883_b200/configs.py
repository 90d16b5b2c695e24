"""The five BASELINE.json configurations (pinned decisions D1-D12).

Every input is synthetic (seeded generator, csrc/gen.cpp); there is no dataset.
"""
from __future__ import annotations

import dataclasses
import math

B_HZ = 491.5e6          # D8: literally 491.5 MHz
FC_HZ = 77e9
WINDOW_RECT, WINDOW_HAMMING = 0, 1
EST_LS, EST_DFT_CE = 0, 1


@dataclasses.dataclass(frozen=True)
class RadarConfig:
    name: str
    n: int                  # subcarriers N
    m: int                  # OFDM symbols M
    n_prime: int
    m_prime: int
    n_cp: int               # CP samples == DFT-CE taps L (D1)
    qam: int
    estimator: int
    window: int
    max_targets: int
    frames: int
    targets_min: int
    targets_max: int
    snr_lo_db: float
    snr_hi_db: float
    zc_precode: bool = False
    per_frame_k: bool = False   # cfg4: K_f = the frame's target count (D6)
    range_lo: float = 5.0
    range_hi: float = 300.0
    vel_lo: float = -80.0
    vel_hi: float = 80.0
    pfa: float = 1e-2
    base_seed: int = 20220908   # recorded with every report (D9)

    @property
    def df_hz(self) -> float:
        return B_HZ / self.n

    @property
    def symbol_time(self) -> float:
        t = 1.0 / self.df_hz
        return t + self.n_cp * (t / self.n)

    def replace(self, **kw) -> "RadarConfig":
        return dataclasses.replace(self, **kw)


CFG0 = RadarConfig("cfg0", 1024, 256, 1024, 256, 256, 4, EST_LS, WINDOW_RECT, 3, 1, 3, 3, 10.0, 10.0)
CFG1 = RadarConfig("cfg1", 1024, 256, 1024, 256, 128, 4, EST_DFT_CE, WINDOW_HAMMING, 3, 64, 3, 3, -10.0, -10.0)
CFG2 = RadarConfig("cfg2", 2048, 512, 4096, 2048, 256, 16, EST_DFT_CE, WINDOW_HAMMING, 8, 256, 8, 8, 0.0, 20.0,
                   zc_precode=True)
CFG4 = RadarConfig("cfg4", 1024, 256, 1024, 256, 128, 4, EST_DFT_CE, WINDOW_HAMMING, 8, 8192, 3, 8, -10.0, 20.0,
                   per_frame_k=True)


@dataclasses.dataclass(frozen=True)
class SftRunConfig:
    """cfg3: FPS-SFT on 1024 x 1024 on-grid sparse channel estimates (D11, D12)."""

    name: str = "cfg3"
    n: int = 1024
    m: int = 1024
    targets: int = 10
    snr_db: float = 15.0
    i_max: int = 8
    decimation: int = 8
    frac_tol: float = 0.25
    amp_tol: float = 0.35
    pfa: float = 1e-2
    frames: int = 1024
    max_targets: int = 10
    base_seed: int = 20220908

    @property
    def sigma2(self) -> float:
        return self.targets / 10 ** (self.snr_db / 10.0)


CFG3 = SftRunConfig()

ALL = {"cfg0": CFG0, "cfg1": CFG1, "cfg2": CFG2, "cfg3": CFG3, "cfg4": CFG4}


def pf(cfg: RadarConfig) -> float:
    """Window2d::power_factor (periodogram.cpp:11-16) in fp64."""
    if cfg.window == WINDOW_RECT:
        return 1.0
    two_pi = 6.283185307179586476925286766559
    sk = sum((0.54 - 0.46 * math.cos(two_pi * k / (cfg.n - 1))) ** 2 for k in range(cfg.n))
    sl = sum((0.54 - 0.46 * math.cos(two_pi * l / (cfg.m - 1))) ** 2 for l in range(cfg.m))
    return sk * sl / (cfg.n * cfg.m)
