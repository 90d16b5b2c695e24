"""Per-phase clock64 breakdown of the fused DFT-CE kernel (debug build libofdmr_b200_timing.so)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("OFDMR_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                "paper_2209_03883_b200", "libofdmr_b200_timing.so"))
from paper_2209_03883_b200 import _native, configs, gen  # noqa: E402
from paper_2209_03883_b200.receiver import Receiver  # noqa: E402

NAMES = ["A_load", "A_fft", "A_store", "A_reduce+sync", "B_rowfft", "C_load", "C_fft", "-",
         "C_detect+edges", "finish_sync", "resolve+topk+out"]
cfg = configs.CFG4
F = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
pool = gen.frames(cfg, 0, 64)
reps = -(-F // 64)
y = torch.from_numpy(pool.y).cuda().repeat(reps, 1, 1)[:F].contiguous()
x = torch.from_numpy(pool.x).cuda().repeat(reps, 1, 1)[:F].contiguous()
s2 = torch.from_numpy(np.tile(pool.sigma2, reps)[:F]).cuda()
kf = torch.from_numpy(np.tile(pool.n_targets, reps)[:F].astype(np.int32)).cuda()
rx = Receiver.from_config(cfg)
d = rx._dets(F)
lib = _native.lib()
lib.ofdmr_debug_phase_cycles.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros(16, np.uint64)
for _ in range(2):
    rx._stream()
    rx.pipeline_raw(y, x, s2, kf, d, F)
torch.cuda.synchronize()
lib.ofdmr_debug_phase_cycles(buf.ctypes.data, 1)
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
e0.record()
rx._stream()
rx.pipeline_raw(y, x, s2, kf, d, F)
e1.record()
torch.cuda.synchronize()
lib.ofdmr_debug_phase_cycles(buf.ctypes.data, 1)
ms = e0.elapsed_time(e1)
tot = buf[:11].sum()
print(f"frames {F}: {ms:.3f} ms, {F / ms * 1e3:.0f} frames/s")
for n, v in zip(NAMES, buf[:11]):
    print(f"{n:16s} {v / tot * 100:6.2f}%   {v / F / 2:10.0f} cycles/frame/CTA")
