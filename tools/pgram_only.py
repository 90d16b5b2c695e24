"""Run only the batched periodogram (H -> P) on the fast path, for profiling."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_03883_b200.receiver import Receiver  # noqa: E402

F = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
h = (torch.randn(F, 1024, 256, dtype=torch.complex64, device="cuda"))
p = torch.empty(F, 1024, 256, dtype=torch.float32, device="cuda")
rx = Receiver(1024, 256, window="rectangular")
for _ in range(reps):
    rx._stream()
    rx._lib.ofdmr_periodogram(rx._h, h.data_ptr(), p.data_ptr(), F)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
rx._lib.ofdmr_periodogram(rx._h, h.data_ptr(), p.data_ptr(), F)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"periodogram {F} frames: {ms:.3f} ms, {F / ms * 1e3:.0f} frames/s, {F * 3 * 2**20 / ms / 1e6:.1f} GB/s")
