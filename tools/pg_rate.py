"""Device-only rate of ofdmr_periodogram (1024 x 256, rect) for the library named by OFDMR_LIB."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_03883_b200.receiver import Receiver  # noqa: E402

F = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
win = sys.argv[2] if len(sys.argv) > 2 else "rectangular"
h = torch.randn(64, 1024, 256, dtype=torch.complex64, device="cuda").repeat(-(-F // 64), 1, 1)[:F].contiguous()
p = torch.empty(F, 1024, 256, dtype=torch.float32, device="cuda")
rx = Receiver(1024, 256, window=win)
ts = []
for i in range(8):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    rx._stream()
    e0.record()
    rx._lib.ofdmr_periodogram(rx._h, h.data_ptr(), p.data_ptr(), F)
    e1.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(e0.elapsed_time(e1))
ms = float(np.median(ts))
print(f"{os.path.basename(os.environ.get('OFDMR_LIB', 'default'))} {win}: {ms:.3f} ms  {F / ms * 1e3:,.0f} frames/s "
      f"{F * 3 * 2**20 / ms / 1e6:,.0f} GB/s")
