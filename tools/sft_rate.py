"""cfg3 FPS-SFT batch rate through Receiver.sft (whole call: host draws, uploads, kernel, overflow
check) and the sft kernel alone (development tool)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_03883_b200 import configs, gen  # noqa: E402
from paper_2209_03883_b200.receiver import Receiver  # noqa: E402

c3 = configs.CFG3
h, s2, _, _ = gen.sparse_frames(c3.n, c3.m, c3.targets, c3.snr_db, c3.base_seed, 0, 64)
seeds = np.array([gen.derive_seed(c3.base_seed + f, 0x736674) for f in range(c3.frames)], np.uint64)
s2t = np.tile(s2, c3.frames // 64)
hd = torch.from_numpy(h).cuda().repeat(c3.frames // 64, 1, 1).contiguous()
rx = Receiver(16, 16)
call = lambda: rx.sft(hd, seeds, s2t, i_max=c3.i_max, pfa=c3.pfa, decimation=c3.decimation)  # noqa: E731
out = call()
torch.cuda.synchronize()
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    out = call()
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
ms = float(np.median(ts)) * 1e3
print(f"{os.path.basename(os.environ.get('OFDMR_LIB', 'default'))} cfg3 sft: {c3.frames} frames {ms:.3f} ms "
      f"{c3.frames / ms * 1e3:,.0f} frames/s; iterations[0] {int(out['iterations'][0])} "
      f"entries[0] {int(out['n_entries'][0])}")
