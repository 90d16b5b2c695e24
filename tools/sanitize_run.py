"""Small end-to-end run of every kernel family for compute-sanitizer (memcheck / racecheck)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_03883_b200 import configs, gen  # noqa: E402
from paper_2209_03883_b200.receiver import Receiver  # noqa: E402

torch.cuda.set_device(0)
fb = gen.frames(configs.CFG4, 0, 4)
with Receiver.from_config(configs.CFG4) as rx:          # fused cluster kernel
    rx.pipeline(fb.y, fb.x, fb.sigma2, k_per_frame=fb.n_targets)
    rx.pipeline(fb.y, fb.x, fb.sigma2, want_map=True)   # chunked fast kernels
fb0 = gen.frames(configs.CFG0, 0, 2)
with Receiver.from_config(configs.CFG0) as rx:          # persistent ticket kernel (LS)
    rx.pipeline(fb0.y, fb0.x, fb0.sigma2)
    rx.periodogram(fb0.y)
with Receiver(64, 32, 128, 64, window="hamming", estimator="dft-ce", n_cp=16, max_targets=4) as rx:  # generic
    f2 = gen.frames(configs.CFG1.replace(n=64, m=32, n_prime=128, m_prime=64, n_cp=16, max_targets=4), 0, 2)
    rx.pipeline(f2.y, f2.x, f2.sigma2, want_map=True)
h, s2, _, _ = gen.sparse_frames(64, 32, 4, 20.0, 7, 0, 2)
with Receiver(16, 16) as rx:                            # FPS-SFT
    rx.sft(h, np.array([1, 2], np.uint64), s2, i_max=6)
torch.cuda.synchronize()
print("sanitize run ok")
