"""GPU frame generator: exactness against the CPU generator on a sample and device rate."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_03883_b200 import configs, gen  # noqa: E402

cfg = configs.CFG4
F = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
ref = gen.frames(cfg, 100, 16)
d = gen.frames_device(cfg, 100, 16)
torch.cuda.synchronize()
y = d["y"].cpu().numpy().view(np.float32)
r = ref.y.view(np.float32)
diff = y != r
print(f"sample 16 frames: x exact {np.array_equal(d['x'].cpu().numpy(), ref.x)}, "
      f"sigma2 exact {np.array_equal(d['sigma2'].cpu().numpy(), ref.sigma2)}, "
      f"y floats differing {diff.sum()} of {diff.size} ({diff.mean():.2e}), max |dy| {np.abs(y - r).max():.3e}")
for i in range(2):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    d = gen.frames_device(cfg, 0, F)
    e1.record()
    torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"GPU generator: {F} cfg4 frames in {ms:.1f} ms = {F / ms * 1e3:,.0f} frames/s")
t0 = time.perf_counter()
gen.frames(cfg, 0, 64)
dt = time.perf_counter() - t0
print(f"CPU generator ({os.cpu_count()} threads): {64 / dt:,.0f} frames/s")
