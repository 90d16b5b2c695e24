"""Per-phase clock64 breakdown of the warp-specialised periodogram (debug build
libofdmr_b200_t3.so from tools/build_timing.sh): column warp 0 and row warp 0 of every CTA."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("OFDMR_LIB", os.path.join(ROOT, "paper_2209_03883_b200", "libofdmr_b200_t3.so"))
from paper_2209_03883_b200 import _native  # noqa: E402
from paper_2209_03883_b200.receiver import Receiver  # noqa: E402

NAMES = ["col: tile wait", "col: load+DFT32+tw", "col: G-free wait", "col: G store", "row: loop top", "row: G-ready wait", "row: DFT32+handoff", "row: FFT256+P"]
F = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
win = sys.argv[2] if len(sys.argv) > 2 else "rectangular"
h = torch.randn(64, 1024, 256, dtype=torch.complex64, device="cuda").repeat(-(-F // 64), 1, 1)[:F].contiguous()
p = torch.empty(F, 1024, 256, dtype=torch.float32, device="cuda")
rx = Receiver(1024, 256, window=win)
lib = _native.lib()
lib.ofdmr_debug_pg3_phase_cycles.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros(8, np.uint64)
for _ in range(2):
    rx._stream()
    lib.ofdmr_periodogram(rx._h, h.data_ptr(), p.data_ptr(), F)
torch.cuda.synchronize()
lib.ofdmr_debug_pg3_phase_cycles(buf.ctypes.data, 1)
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
e0.record()
lib.ofdmr_periodogram(rx._h, h.data_ptr(), p.data_ptr(), F)
e1.record()
torch.cuda.synchronize()
lib.ofdmr_debug_pg3_phase_cycles(buf.ctypes.data, 1)
ms = e0.elapsed_time(e1)
print(f"frames {F}: {ms:.3f} ms, {F / ms * 1e3:,.0f} frames/s")
ct, rt = buf[:4].sum(), buf[4:8].sum()
for i, n in enumerate(NAMES):
    tot = ct if i < 4 else rt
    print(f"{n:22s} {buf[i] / tot * 100:6.2f}%   {buf[i] / F:10.0f} cycles/frame (summed over CTAs)")
