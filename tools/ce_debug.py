"""Debug: position (in)dependence of the fused cfg4 pipeline on a tiled batch."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_03883_b200 import configs, gen  # noqa: E402
from paper_2209_03883_b200.receiver import Receiver  # noqa: E402

cfg = configs.CFG4
pool, F = int(sys.argv[1]) if len(sys.argv) > 1 else 256, int(sys.argv[2]) if len(sys.argv) > 2 else 8192
fb = gen.frames(cfg, 0, pool)
reps = F // pool
y = torch.from_numpy(fb.y).cuda().repeat(reps, 1, 1)
x = torch.from_numpy(fb.x).cuda().repeat(reps, 1, 1)
s2 = torch.from_numpy(np.tile(fb.sigma2, reps)).cuda()
kf = torch.from_numpy(np.tile(fb.n_targets, reps).astype(np.int32)).cuda()
with Receiver.from_config(cfg) as rx:
    outs = []
    for _ in range(2):
        dets, _ = rx.pipeline(y, x, s2, k_per_frame=kf)
        torch.cuda.synchronize()
        outs.append((dets.delay_bin.cpu().numpy().reshape(reps, pool, -1), dets.doppler_bin.cpu().numpy().reshape(reps, pool, -1),
                     dets.peak_power.cpu().numpy().reshape(reps, pool, -1), dets.counts.cpu().numpy().reshape(reps, pool),
                     dets.sigma2_h.cpu().numpy().reshape(reps, pool)))
d, v, p, c, sh = outs[0]
print("run-to-run equal:", all((a == b).all() for a, b in zip(outs[0][:4], outs[1][:4])))
for name, arr in (("delay", d), ("doppler", v), ("power", p), ("count", c), ("s2h", sh)):
    if arr is None:
        continue
    bad = np.argwhere((arr != arr[0:1]).reshape(reps, pool, -1).any(-1))
    print(name, "mismatching (rep, frame):", len(bad), bad[:10].tolist())
    for r, f in bad[:4]:
        print("   ", arr[0, f].ravel()[:8], "vs", arr[r, f].ravel()[:8])
