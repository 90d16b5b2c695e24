"""Output writers of the reference (io.cpp:22-110), fed from this package's maps and records.

Byte-for-byte the reference formats: "%.12g" floats (format_double, io.cpp:22-26), CSV
headers and row order, the 8-bit PGM heatmap (io.cpp:94-110) and the run.json manifest
(io.cpp:112-122 with the config.cpp:147-182 schema and nlohmann's number formatting).  The PGM pixels of a batch
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


# ------------------------------------------------------------------ run.json manifests --
TOOL_VERSION = "ofdmradar 1.0.0"  # io.hpp kToolVersion


def _json_float(v: float) -> str:
    """nlohmann::json number_float output: shortest round-trip digits, fixed notation for
    decimal exponents in (-4, 15] (with a trailing ".0" for integral values), otherwise
    d.ddde+XX."""
    if v != v or v in (math.inf, -math.inf):
        return "null"
    if v == 0.0:
        return "-0.0" if math.copysign(1.0, v) < 0 else "0.0"
    r = repr(float(v))
    neg = r.startswith("-")
    r = r.lstrip("-")
    mant, _, exp = r.partition("e")
    digits = mant.replace(".", "")
    point = (mant.index(".") if "." in mant else len(mant)) + (int(exp) if exp else 0)
    lead = len(digits) - len(digits.lstrip("0"))
    digits = digits.strip("0") or "0"
    point -= lead
    k, n = len(digits), point  # value = 0.digits x 10^n
    if k <= n <= 15:
        s = digits + "0" * (n - k) + ".0"
    elif 0 < n <= 15:
        s = digits[:n] + "." + digits[n:]
    elif -4 < n <= 0:
        s = "0." + "0" * (-n) + digits
    else:
        e = n - 1
        s = digits[0] + ("." + digits[1:] if k > 1 else "") + "e" + ("-" if e < 0 else "+") + f"{abs(e):02d}"
    return ("-" if neg else "") + s


def _json_str(s: str) -> str:
    out = ['"']
    for ch in s:
        o = ord(ch)
        if ch == '"':
            out.append('\\"')
        elif ch == "\\":
            out.append("\\\\")
        elif o < 0x20:
            out.append({8: "\\b", 9: "\\t", 10: "\\n", 12: "\\f", 13: "\\r"}.get(o, f"\\u{o:04x}"))
        else:
            out.append(ch)
    out.append('"')
    return "".join(out)


def _json_dump(v, ind: int, sort: bool) -> str:
    """nlohmann::json::dump(2) layout (sort=True would mimic a std::map-backed json; the
    reference's manifest and config objects keep insertion order)."""
    pad, pad1 = " " * ind, " " * (ind + 2)
    if isinstance(v, bool):
        return "true" if v else "false"
    if v is None:
        return "null"
    if isinstance(v, int):
        return str(v)
    if isinstance(v, float):
        return _json_float(v)
    if isinstance(v, str):
        return _json_str(v)
    if isinstance(v, dict):
        if not v:
            return "{}"
        items = sorted(v.items()) if sort else list(v.items())
        body = ",\n".join(f"{pad1}{_json_str(k)}: {_json_dump(x, ind + 2, sort)}" for k, x in items)
        return "{\n" + body + "\n" + pad + "}"
    if isinstance(v, (list, tuple)):
        if not v:
            return "[]"
        return "[\n" + ",\n".join(pad1 + _json_dump(x, ind + 2, sort) for x in v) + "\n" + pad + "]"
    raise TypeError(type(v))


def simulation_config(*, n: int, m: int, df_hz: float, fc_hz: float, n_cp: int, qam: int, n_prime: int,
                      m_prime: int, window: str, pfa: float, targets: Sequence[dict], snr_db: float, seed: int,
                      estimator: str = "ls", zcp=(1024, 1, 0), detector: str = "periodogram",
                      max_targets: int = 64, estimate_noise: bool = False, sft_i_max: int = 10,
                      amplitude_mode: str = "normalized", output_dir: str = "out") -> dict:
    """config.cpp:147-182 to_json schema of a SimulationConfig.  targets: dicts with
    range_m, velocity_mps, optional rcs (default 1.0) and phase."""
    tg = []
    for t in targets:
        d = {"range_m": float(t["range_m"]), "velocity_mps": float(t["velocity_mps"]), "rcs": float(t.get("rcs", 1.0))}
        if t.get("phase") is not None and t["phase"] == t["phase"]:
            d["phase"] = float(t["phase"])
        tg.append(d)
    return {
        "waveform": {"n_subcarriers": int(n), "n_symbols": int(m), "subcarrier_spacing_hz": float(df_hz),
                     "carrier_hz": float(fc_hz), "n_cp": int(n_cp), "qam_order": int(qam)},
        "targets": tg,
        "channel": {"snr_db": float(snr_db) if math.isfinite(snr_db) else "inf", "amplitude_mode": amplitude_mode,
                    "seed": int(seed)},
        "estimator": {"kind": estimator, "zcp": {"length": int(zcp[0]), "root": int(zcp[1]), "offset": int(zcp[2])}},
        "detector": {"kind": detector, "pfa": float(pfa), "window": window, "n_prime": int(n_prime),
                     "m_prime": int(m_prime), "max_targets": int(max_targets), "estimate_noise": bool(estimate_noise),
                     "sft": {"i_max": int(sft_i_max)}},
        "output": {"dir": output_dir},
    }


def write_run_manifest(path: str | os.PathLike, command: str, seed: int, config: dict,
                       extra: Sequence[tuple[str, str]] = (), wall_ms: float = 0.0) -> None:
    """io.cpp:112-122 run.json: tool, command, seed, params (sweep parameters, only when
    present), the resolved config, wall_ms."""
    cfg_txt = _json_dump(config, 2, False)  # config.cpp builds an insertion-ordered json
    parts = [f'  "tool": {_json_str(TOOL_VERSION)}', f'  "command": {_json_str(command)}', f'  "seed": {int(seed)}']
    if extra:
        params: dict = {}
        for k, v in extra:
            params[str(k)] = str(v)
        parts.append(f'  "params": {_json_dump(params, 2, False)}')
    parts.append(f'  "config": {cfg_txt}')
    parts.append(f'  "wall_ms": {_json_float(float(wall_ms))}')
    with open(path, "wb") as fh:
        fh.write(("{\n" + ",\n".join(parts) + "\n}\n").encode())
