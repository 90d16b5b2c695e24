"""Per-phase clock64 breakdown of the fused periodogram kernel (debug build libofdmr_b200_timing.so)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("OFDMR_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                "paper_2209_03883_b200", "libofdmr_b200_timing.so"))
from paper_2209_03883_b200 import _native  # noqa: E402
from paper_2209_03883_b200.receiver import Receiver  # noqa: E402

NAMES = ["col_load", "col_fft", "G_wait", "G_store", "group_barrier", "row_pass"]
F = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
win = sys.argv[2] if len(sys.argv) > 2 else "rectangular"
h = torch.randn(64, 1024, 256, dtype=torch.complex64, device="cuda").repeat(-(-F // 64), 1, 1)[:F].contiguous()
p = torch.empty(F, 1024, 256, dtype=torch.float32, device="cuda")
rx = Receiver(1024, 256, window=win)
lib = _native.lib()
lib.ofdmr_debug_pg_phase_cycles.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros(8, np.uint64)
for _ in range(2):
    rx._stream()
    lib.ofdmr_periodogram(rx._h, h.data_ptr(), p.data_ptr(), F)
torch.cuda.synchronize()
lib.ofdmr_debug_pg_phase_cycles(buf.ctypes.data, 1)
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
e0.record()
lib.ofdmr_periodogram(rx._h, h.data_ptr(), p.data_ptr(), F)
e1.record()
torch.cuda.synchronize()
lib.ofdmr_debug_pg_phase_cycles(buf.ctypes.data, 1)
ms = e0.elapsed_time(e1)
tot = buf[:6].sum()
print(f"frames {F}: {ms:.3f} ms, {F / ms * 1e3:,.0f} frames/s, {F * 3 * 2**20 / ms / 1e6:,.0f} GB/s")
for n, v in zip(NAMES, buf[:6]):
    print(f"{n:14s} {v / tot * 100:6.2f}%   {v / F:10.0f} cycles/frame (summed over CTAs)")
lib.ofdmr_debug_info.restype = C.c_longlong
lib.ofdmr_debug_info.argtypes = [C.c_void_p, C.c_char_p]
print("clusters in use", lib.ofdmr_debug_info(rx._h, b"pg_clusters"))
