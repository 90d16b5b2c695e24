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


def _rel(a: float, b: float) -> float:
    den = max(abs(a), abs(b))
    return abs(a - b) / den if den > 0 else 0.0


def classify_detail(gpu_dets, ref_dets, pmap: np.ndarray, eta: float, k: int):
    """(verdict, margin, reason): verdict 'ok' (identical bins and order), 'tie' (every
    difference is explained by a near-tie of the oracle's own fp64 values: margin = the
    largest relative fp64 gap among the deciding comparisons, < TIE_REL) or 'fail'."""
    g = [(int(a), int(b)) for a, b, _ in gpu_dets]
    r = [(int(a), int(b)) for a, b, _ in ref_dets]
    if g == r:
        return "ok", None, ""
    rows, cols = pmap.shape
    idx, vals, nbmax = strict_local_maxima(pmap, -np.inf)
    half = cols // 2

    def cell(d):
        return d[0] * cols + (d[1] + half)

    flat = pmap.ravel()
    nbf = nbmax.ravel()
    suspicious = set(g) ^ set(r)
    worst, reasons = 0.0, []
    above = vals[vals >= eta * (1 - TIE_REL)]
    for d in suspicious:
        c = cell(d)
        v = flat[c]
        cands = {"neighbour": _rel(v, nbf[c]), "threshold": _rel(v, eta)}
        if len(above) > k - 1:
            kth = above[min(k - 1, len(above) - 1)]
            nxt = above[k] if len(above) > k else eta
            cands["rank_k"] = max(_rel(kth, nxt), min(_rel(v, kth), _rel(v, nxt)))
        why, m = min(cands.items(), key=lambda kv: kv[1])
        if m > TIE_REL:
            return "fail", m, f"{d}: smallest fp64 margin {m:.3g} ({why})"
        worst = max(worst, m)
        reasons.append(f"{d}:{why}")
    if not suspicious:  # same set, different order: adjacent ranks must be near-equal
        for a, b in zip(g, r):
            if a != b:
                m = _rel(flat[cell(a)], flat[cell(b)])
                if m > TIE_REL:
                    return "fail", m, f"order {a} vs {b}: margin {m:.3g}"
                worst = max(worst, m)
                reasons.append(f"order {a}/{b}")
    return "tie", worst, ";".join(reasons)


def classify(gpu_dets, ref_dets, pmap: np.ndarray, eta: float, k: int) -> str:
    """'ok', 'tie' or 'fail' (see classify_detail)."""
    return classify_detail(gpu_dets, ref_dets, pmap, eta, k)[0]


def powers_close(gpu_dets, ref_dets) -> bool:
    rd = {(int(a), int(b)): w for a, b, w in ref_dets}
    for a, b, w in gpu_dets:
        key = (int(a), int(b))
        if key in rd and abs(w - rd[key]) > POWER_REL * abs(rd[key]):
            return False
    return True
