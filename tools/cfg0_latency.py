"""cfg0 single-frame pipeline: per-call time with CUDA events around back-to-back calls (as
bench.py), host time per call, and the launches per call (development tool)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_03883_b200 import configs, gen  # noqa: E402
from paper_2209_03883_b200.receiver import Receiver  # noqa: E402

cfg = configs.CFG0
fb = gen.frames(cfg, 0, 1)
y = torch.from_numpy(fb.y).cuda().contiguous()
x = torch.from_numpy(fb.x).cuda().contiguous()
s2 = torch.from_numpy(fb.sigma2).cuda()
rx = Receiver.from_config(cfg)
d = rx._dets(1)
rx._stream()
for _ in range(10):
    rx.pipeline_raw(y, x, s2, None, d, 1)
torch.cuda.synchronize()
n0 = rx.launch_count
reps = 200
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
for _ in range(reps):
    rx.pipeline_raw(y, x, s2, None, d, 1)
e1.record()
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"cfg0: {e0.elapsed_time(e1) / reps * 1e3:.1f} us/call (events), host enqueue {(t1 - t0) / reps * 1e6:.1f} us/call, "
      f"launches/call {(rx.launch_count - n0) / reps:.1f}")
