"""Parity helpers: compare GPU detections with the oracle, separating genuine
fp32-unresolvable near-ties (SURVEY.md §8d "Parity rules") from failures."""
from __future__ import annotations

import numpy as np

TIE_REL = 1e-5   # oracle fp64 margin below which an fp32 decision may legitimately flip
POWER_REL = 1e-4  # peak magnitude tolerance (BASELINE north_star)


def strict_local_maxima(p: np.ndarray, eta: float):
    """All strict wrapped 3x3 local maxima >= eta, sorted (value desc, index asc)."""
    rows, cols = p.shape
    nb = np.stack([np.roll(np.roll(p, dr, 0), dc, 1) for dr in (-1, 0, 1) for dc in (-1, 0, 1) if (dr, dc) != (0, 0)])
    is_max = (p > nb.max(0)) & (p >= eta)
    idx = np.flatnonzero(is_max)
    vals = p.ravel()[idx]
    order = np.lexsort((idx, -vals))
    return idx[order], vals[order], nb.max(0)


def classify(gpu_dets, ref_dets, pmap: np.ndarray, eta: float, k: int) -> str:
    """'ok' (identical bins and order), 'tie' (difference explained by a near-tie of the
    oracle's own fp64 values), or 'fail'."""
    g = [(int(a), int(b)) for a, b, _ in gpu_dets]
    r = [(int(a), int(b)) for a, b, _ in ref_dets]
    if g == r:
        return "ok"
    rows, cols = pmap.shape
    idx, vals, nbmax = strict_local_maxima(pmap, -np.inf)
    half = cols // 2

    def cell(d):
        return d[0] * cols + (d[1] + half)

    flat = pmap.ravel()
    nbf = nbmax.ravel()
    suspicious = set(g) ^ set(r)
    for d in suspicious:
        c = cell(d)
        v = flat[c]
        near_nb = abs(v - nbf[c]) <= TIE_REL * max(v, nbf[c])
        near_eta = abs(v - eta) <= TIE_REL * max(abs(eta), v)
        # near the K-th / (K+1)-th rank boundary among maxima >= eta
        above = vals[vals >= eta * (1 - TIE_REL)]
        near_rank = False
        if len(above) > k - 1:
            kth = above[min(k - 1, len(above) - 1)]
            nxt = above[k] if len(above) > k else eta
            near_rank = abs(kth - nxt) <= TIE_REL * kth and (abs(v - kth) <= TIE_REL * kth or abs(v - nxt) <= TIE_REL * kth)
        if not (near_nb or near_eta or near_rank):
            return "fail"
    if not suspicious:  # same set, different order: adjacent ranks must be near-equal
        for i, (a, b) in enumerate(zip(g, r)):
            if a != b:
                va, vb = flat[cell(a)], flat[cell(b)]
                if abs(va - vb) > TIE_REL * max(va, vb):
                    return "fail"
    return "tie"


def powers_close(gpu_dets, ref_dets) -> bool:
    rd = {(int(a), int(b)): w for a, b, w in ref_dets}
    for a, b, w in gpu_dets:
        key = (int(a), int(b))
        if key in rd and abs(w - rd[key]) > POWER_REL * abs(rd[key]):
            return False
    return True
