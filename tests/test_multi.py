"""Multi-device C-ABI (ofdmr_multi) on the one GPU of the test box: three contexts
on device 0 (each on its own host thread and stream; no kernel waits on another context's) stand
in for three devices.  The sharded host path and the device-resident path with the peer-copy
gather must reproduce the single-context records exactly."""
import numpy as np
import pytest
import torch

from paper_2209_03883_b200 import configs, gen
from paper_2209_03883_b200.receiver import MultiReceiver, Receiver

pytestmark = pytest.mark.gpu


def test_multi_receiver_matches_single_context(cuda):
    cfg = configs.CFG4
    F = 37
    fb = gen.frames(cfg, 0, F)
    with Receiver.from_config(cfg) as rx:
        rd, rv, rp, rc = rx.pipeline_host(fb.y, fb.x, fb.sigma2, fb.n_targets)
    with MultiReceiver(cfg, [0, 0, 0]) as mr:
        d, v, p, c = mr.pipeline_host(fb.y, fb.x, fb.sigma2, fb.n_targets)
        for a, b in ((d, rd), (v, rv), (p, rp), (c, rc)):
            assert np.array_equal(a, b)
        ys, xs, ss, ks = [], [], [], []
        for r in range(3):
            lo, hi = mr.shard_range(F, r)
            ys.append(torch.from_numpy(fb.y[lo:hi]).cuda())
            xs.append(torch.from_numpy(fb.x[lo:hi]).cuda())
            ss.append(torch.from_numpy(fb.sigma2[lo:hi]).cuda())
            ks.append(torch.from_numpy(fb.n_targets[lo:hi].astype(np.int32)).cuda())
        dets, st = mr.pipeline(ys, xs, ss, ks)
        assert int(st.abs().sum()) == 0
        assert np.array_equal(dets.delay_bin.cpu().numpy(), rd)
        assert np.array_equal(dets.doppler_bin.cpu().numpy(), rv)
        assert np.array_equal(dets.peak_power.cpu().numpy(), rp)
        assert np.array_equal(dets.counts.cpu().numpy(), rc)
