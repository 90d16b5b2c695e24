"""clock64 phase breakdown of the cfg2 column pass (colpass2048.cu; debug build from
tools/build_variant.sh t colpass2048 -DOFDMR_PHASE_TIMING): thread 0 of every CTA."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("OFDMR_LIB", os.path.join(ROOT, "paper_2209_03883_b200", "libofdmr_b200_t.so"))
from paper_2209_03883_b200 import _native, configs, gen  # noqa: E402
from paper_2209_03883_b200.receiver import Receiver  # noqa: E402

NAMES = ["LS ring + tile", "IFFT_2048 / taps / FFT -> H'", "4 x (modulate + IFFT_1024)", "4 x (stage + G store)"]
cfg = configs.CFG2
frames = int(sys.argv[1]) if len(sys.argv) > 1 else 64
fb = gen.frames(cfg, 0, 8)
rep = -(-frames // 8)
y = torch.from_numpy(fb.y).cuda().repeat(rep, 1, 1)[:frames].contiguous()
x = torch.from_numpy(fb.x).cuda().repeat(rep, 1, 1)[:frames].contiguous()
s2 = torch.from_numpy(np.tile(fb.sigma2, rep)[:frames]).cuda()
rx = Receiver.from_config(cfg)
dets = rx._dets(frames)
lib = _native.lib()
lib.ofdmr_debug_c2_phase_cycles.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros(8, np.uint64)
rx._stream()
rx.pipeline_raw(y, x, s2, None, dets, frames)
torch.cuda.synchronize()
lib.ofdmr_debug_c2_phase_cycles(buf.ctypes.data, 1)
rx.pipeline_raw(y, x, s2, None, dets, frames)
torch.cuda.synchronize()
lib.ofdmr_debug_c2_phase_cycles(buf.ctypes.data, 1)
tot = buf[:4].sum()
for i, n in enumerate(NAMES):
    print(f"{n:32s} {buf[i] / tot * 100:6.2f}%   {buf[i] / frames:12.0f} cycles/frame (summed over CTAs)")
