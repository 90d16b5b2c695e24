"""One GPU-generator launch over 1024 cfg4 frames (for profiling)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_03883_b200 import configs, gen  # noqa: E402

cfg = configs.CFG4
fb = gen.frames_device(cfg, 0, 1024)
torch.cuda.synchronize()
print("ok", fb["y"].shape)
