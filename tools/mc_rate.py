"""Monte-Carlo rmse_sweep rate (bench.py's scenario) and the share of the host-side matching
(development tool): the same sweep with the matching replaced by a no-op."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_03883_b200 import configs  # noqa: E402
from paper_2209_03883_b200 import montecarlo as mc  # noqa: E402

cfg = configs.CFG1
rng_t, vel_t = np.array([8.0, 17.5, 31.0]), np.array([-35.0, 12.0, 60.0])
grid = [-15.0, -5.0, 5.0]
mc.rmse_sweep(cfg, rng_t, vel_t, grid[:1], 2048, 1)
acc = {"t": 0.0}
orig_match, orig_phys = mc.match_detections, mc.bins_to_physics


def timed(f):
    def g(*a, **k):
        t = time.perf_counter()
        r = f(*a, **k)
        acc["t"] += time.perf_counter() - t
        return r
    return g


mc.match_detections, mc.bins_to_physics = timed(orig_match), timed(orig_phys)
torch.cuda.synchronize()
t0 = time.perf_counter()
rows = mc.rmse_sweep(cfg, rng_t, vel_t, grid, 4096, 2022)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"{3 * 4096 / dt:,.0f} trials/s; host matching + physics {acc['t'] / dt * 100:.0f} % of the wall time",
      [round(r.range_rmse_m, 6) for r in rows])
