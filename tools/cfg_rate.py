"""Device rate and per-stage kernel time of the receiver pipeline on one BASELINE config
(development tool): python tools/cfg_rate.py cfg2 [frames] [pool]."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_03883_b200 import configs, gen  # noqa: E402
from paper_2209_03883_b200.receiver import Receiver  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = configs.ALL[name]
frames = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.frames
pool = int(sys.argv[3]) if len(sys.argv) > 3 else 8
fb = gen.frames(cfg, 0, pool)
rep = -(-frames // pool)
y = torch.from_numpy(fb.y).cuda().repeat(rep, 1, 1)[:frames].contiguous()
x = torch.from_numpy(fb.x).cuda().repeat(rep, 1, 1)[:frames].contiguous()
s2 = torch.from_numpy(np.tile(fb.sigma2, rep)[:frames]).cuda()
kf = torch.from_numpy(np.tile(fb.n_targets, rep)[:frames].astype(np.int32)).cuda() if cfg.per_frame_k else None
rx = Receiver.from_config(cfg, chunk_frames=int(os.environ.get("CHUNK", "0")))
dets = rx._dets(frames)
rx._stream()
rx.pipeline_raw(y, x, s2, kf, dets, frames)
torch.cuda.synchronize()
ts = []
for i in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rx.pipeline_raw(y, x, s2, kf, dets, frames)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = float(np.median(ts))
rx.set_profiling(True)
rx.pipeline_raw(y, x, s2, kf, dets, frames)
torch.cuda.synchronize()
st, sn = rx.get_profile()
rx.set_profiling(False)
print(f"{os.path.basename(os.environ.get('OFDMR_LIB', 'default'))} {name}: {frames} frames {ms:.3f} ms "
      f"{frames / ms * 1e3:,.0f} frames/s; stages (col, row, merge) ms {np.round(st, 3).tolist()} launches {sn.tolist()}")
print("frame 0:", dets.delay_bin[0].tolist(), dets.doppler_bin[0].tolist(), dets.peak_power[0].tolist(),
      int(dets.counts[0]))
