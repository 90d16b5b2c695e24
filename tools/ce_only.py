"""Run only the fused cfg4 pipeline (device-resident), for profiling: F frames, R repeats."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_03883_b200 import configs, gen  # noqa: E402
from paper_2209_03883_b200.receiver import Receiver  # noqa: E402

cfg = configs.CFG4
F = int(sys.argv[1]) if len(sys.argv) > 1 else 1184
R = int(sys.argv[2]) if len(sys.argv) > 2 else 2
pool = gen.frames(cfg, 0, 64)
reps = -(-F // 64)
y = torch.from_numpy(pool.y).cuda().repeat(reps, 1, 1)[:F].contiguous()
x = torch.from_numpy(pool.x).cuda().repeat(reps, 1, 1)[:F].contiguous()
s2 = torch.from_numpy(np.tile(pool.sigma2, reps)[:F]).cuda()
kf = torch.from_numpy(np.tile(pool.n_targets, reps)[:F].astype(np.int32)).cuda()
rx = Receiver.from_config(cfg)
d = rx._dets(F)
for _ in range(R):
    rx._stream()
    rx.pipeline_raw(y, x, s2, kf, d, F)
torch.cuda.synchronize()
print("ok", F)
