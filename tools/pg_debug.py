import os, sys
import numpy as np
sys.path.insert(0, "/root/repo")
import oracle as O
from paper_2209_03883_b200.receiver import Receiver
n, m, F = 1024, 256, 96
rng = np.random.default_rng(11)
h = (rng.standard_normal((F, n, m)) + 1j * rng.standard_normal((F, n, m))).astype(np.complex64)
with Receiver(n, m, window=0) as rx:
    p = rx.periodogram(h).cpu().numpy()
    os.environ["OFDMR_PG_PERSIST"] = "1"
    q = rx.periodogram(h).cpu().numpy()
bad = [f for f in range(F) if np.abs(p[f] - q[f]).max() / q[f].max() > 1e-4]
print("mismatch frames", bad[:40], len(bad))
for f in [0, 1, 36, 37, 40, 74, 95] + bad[:3]:
    ref = O.periodogram(h[f].astype(np.complex128), 0, n, m)
    ep = np.abs(p[f] - ref).max() / ref.max(); eq = np.abs(q[f] - ref).max() / ref.max()
    d = np.abs(p[f] - ref) > 1e-4 * ref.max()
    rows = np.unique(np.nonzero(d)[0]); cols = np.unique(np.nonzero(d)[1])
    print(f, "fused err", ep, "persist err", eq, "bad rows", rows[:10], len(rows), "cols", cols[:10], len(cols))
