"""Output writers of the reference (io.cpp:22-110), fed from this package's maps and records.

Byte-for-byte the reference formats: "%.12g" floats (format_double, io.cpp:22-26), CSV
headers and row order, and the 8-bit PGM heatmap (io.cpp:94-110).  The PGM pixels of a batch
of device maps are computed on the GPU (Receiver.map_to_pgm -> ofdmr_map_to_pgm) so only
N' x M' bytes per frame leave the device; the host only adds the header.
"""
from __future__ import annotations

import math
import os
from typing import Iterable, Sequence

import numpy as np


def format_double(v: float) -> str:
    """io.cpp:22-26 ("%.12g", the C library's rounding)."""
    return "%.12g" % v


def _db(v: float) -> float:
    return 10.0 * math.log10(max(float(v), 1e-300))


def write_detections_csv(path: str | os.PathLike, dets: Iterable[Sequence]) -> None:
    """io.cpp:28-37.  dets: (delay_bin, doppler_bin, range_m, velocity_mps, peak_power) per
    detection, in output order (e.g. Detections.frame() + bins_to_physics)."""
    lines = ["id,delay_bin,doppler_bin,range_m,velocity_mps,peak_power_db\n"]
    for i, (d, v, r, vel, pw) in enumerate(dets):
        lines.append(f"{i},{int(d)},{int(v)},{format_double(r)},{format_double(vel)},{format_double(_db(pw))}\n")
    with open(path, "wb") as fh:
        fh.write("".join(lines).encode())


def write_map_csv(path: str | os.PathLike, p) -> None:
    """io.cpp:39-49: one line per cell, Doppler column as the signed bin (col - cols/2)."""
    p = np.asarray(p, np.float64)
    rows, cols = p.shape
    half = cols // 2
    out = ["delay_bin,doppler_bin,power_db\n"]
    for r in range(rows):
        row = p[r]
        out.extend(f"{r},{c - half},{format_double(_db(row[c]))}\n" for c in range(cols))
    with open(path, "wb") as fh:
        fh.write("".join(out).encode())


def pgm_pixels(p) -> np.ndarray:
    """io.cpp:96-108 pixel values on the host (fp64, the reference's operation order)."""
    p = np.asarray(p, np.float64)
    peak = max(0.0, float(p.max())) if p.size else 0.0
    if peak <= 0.0:
        peak = 1.0
    floor_db = -60.0
    flat = p.ravel()
    px = np.empty(flat.size, np.uint8)
    lo = peak * 1e-30
    for i, v in enumerate(flat.tolist()):
        db = 10.0 * math.log10(max(v, lo) / peak)
        t = min(max((db - floor_db) / -floor_db, 0.0), 1.0)
        x = t * 255.0
        n = math.floor(x)
        px[i] = n + (1 if x - n >= 0.5 else 0)  # lround (half away from zero), x >= 0
    return px.reshape(p.shape)


def write_pgm_bytes(path: str | os.PathLike, pixels) -> None:
    """P5 header (io.cpp:102) + row-major pixel bytes (e.g. from Receiver.map_to_pgm)."""
    px = np.ascontiguousarray(np.asarray(pixels, np.uint8))
    rows, cols = px.shape
    with open(path, "wb") as fh:
        fh.write(f"P5\n{cols} {rows}\n255\n".encode())
        fh.write(px.tobytes())


def write_map_pgm(path: str | os.PathLike, p) -> None:
    """io.cpp:94-110 from a host map."""
    write_pgm_bytes(path, pgm_pixels(p))
