"""B200-native OFDM radar receiver hot path (arXiv 2209.03883): LS / ZC-LS channel
estimate, DFT-CE, 2-D periodogram with top-K peaks, FPS-SFT — hand-written sm_100a
CUDA kernels behind a C-ABI (include/ofdmr_b200.h)."""
from .configs import ALL as CONFIGS  # noqa: F401

__all__ = ["CONFIGS"]
