"""Device-only rate of the default pipeline dispatch (fused kernel for cfg4) for the library
named by OFDMR_LIB: 8192 frames, 3 warm-up + 5 timed launches, median frames/s."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_03883_b200 import configs, gen  # noqa: E402
from paper_2209_03883_b200.receiver import Receiver  # noqa: E402

cfg = configs.CFG4
F = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
pool = gen.frames(cfg, 0, 64)
reps = -(-F // 64)
y = torch.from_numpy(pool.y).cuda().repeat(reps, 1, 1)[:F].contiguous()
x = torch.from_numpy(pool.x).cuda().repeat(reps, 1, 1)[:F].contiguous()
s2 = torch.from_numpy(np.tile(pool.sigma2, reps)[:F]).cuda()
kf = torch.from_numpy(np.tile(pool.n_targets, reps)[:F].astype(np.int32)).cuda()
rx = Receiver.from_config(cfg)
d = rx._dets(F)
ts = []
for i in range(8):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    rx._stream()
    e0.record()
    rx.pipeline_raw(y, x, s2, kf, d, F)
    e1.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(e0.elapsed_time(e1))
ms = float(np.median(ts))
print(f"{os.path.basename(os.environ.get('OFDMR_LIB', 'default'))}: {ms:.3f} ms  {F / ms * 1e3:,.0f} frames/s")
