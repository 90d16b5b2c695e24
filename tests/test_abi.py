"""CPU tests: the C-ABI library loads and exports every symbol include/ofdmr_b200.h
declares (no compute calls without a GPU); host-side helpers match the reference."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2209_03883_b200 import _native, configs

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "ofdmr_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ofdmr_[a-z_0-9]+)\s*\(", text)))


def test_header_symbols_exported_and_bound():
    lib = _native.lib()
    syms = declared_symbols()
    assert len(syms) >= 18
    bound = {name for name, _, _ in _native.RECEIVER_SYMBOLS}
    for s in syms:
        assert hasattr(lib, s), s
        assert s in bound, f"{s} declared but not bound in _native.py"


def test_library_is_sm100a():
    data = (ROOT / "paper_2209_03883_b200" / "libofdmr_b200.so").read_bytes()
    assert b"sm_100a" in data


def test_generator_symbols():
    g = _native.gen()
    for name, _, _ in _native.GEN_SYMBOLS:
        assert hasattr(g, name)
    # include/ofdmr_gen.h: the device generator lives in the CUDA library
    text = re.sub(r"/\*.*?\*/", "", (ROOT / "include" / "ofdmr_gen.h").read_text(), flags=re.S)
    declared = set(re.findall(r"\b(ofdmr_[a-z_0-9]+)\s*\(", text))
    assert declared == {name for name, _, _ in _native.DEVICE_GEN_SYMBOLS}
    lib = _native.lib()
    for s in declared:
        assert hasattr(lib, s), s


def test_host_helpers_match_reference_formulas():
    lib = _native.lib()
    eta = C.c_double()
    assert lib.ofdmr_detection_threshold(1.0, 0.01, 1.0, C.byref(eta)) == 0
    assert abs(eta.value - 4.6052) < 4.6052e-4
    assert lib.ofdmr_detection_threshold(1.0, 0.0, 1.0, C.byref(eta)) == 2
    assert "pfa" in _native.last_error()
    assert lib.ofdmr_detection_threshold(-1.0, 0.1, 1.0, C.byref(eta)) == 2
    assert "sigma2" in _native.last_error()
    # bins_to_physics known answers on Table I numerology (test_periodogram.cpp:248-264)
    r = C.c_double()
    v = C.c_double()
    lib.ofdmr_bins_to_physics(328, 45, 2048, 512, 2048, 560, 240e3, 77e9, C.byref(r), C.byref(v))
    assert abs(r.value - 100.10) < 100.10e-3 and abs(v.value - 30.06) < 30.06e-3
    lib.ofdmr_bins_to_physics(1, -1, 2048, 512, 2048, 560, 240e3, 77e9, C.byref(r), C.byref(v))
    assert abs(r.value - 0.30518) < 0.30518e-3 and abs(v.value + 0.6679) < 0.6679e-3
    # window power factor equals the oracle's fp64 value bit-for-bit
    import oracle as O
    for kind in (0, 1):
        assert lib.ofdmr_window_power_factor(kind, 1024, 256) == O.power_factor(kind, 1024, 256)
    assert abs(configs.pf(configs.CFG4) - O.power_factor(1, 1024, 256)) < 1e-12


def test_create_rejects_bad_config_without_gpu():
    lib = _native.lib()
    cfg = _native.OfdmrConfig(17 * 19, 256, 17 * 19, 256, 0, 0, 0, 3, 1e-2, 0, 0)
    h = C.c_void_p()
    assert lib.ofdmr_create(C.byref(cfg), C.byref(h)) == 2   # prime factors beyond 13: ConfigError
    cfg = _native.OfdmrConfig(1024, 8192, 1024, 8192, 0, 0, 0, 3, 1e-2, 0, 0)
    assert lib.ofdmr_create(C.byref(cfg), C.byref(h)) == 2   # above 4096: ConfigError
    cfg = _native.OfdmrConfig(1024, 256, 512, 256, 0, 0, 0, 3, 1e-2, 0, 0)
    assert lib.ofdmr_create(C.byref(cfg), C.byref(h)) == 2   # N' < N (periodogram.cpp:43)
    assert "N'" in _native.last_error()
    cfg = _native.OfdmrConfig(1024, 256, 1024, 256, 0, 1, 2048, 3, 1e-2, 0, 0)
    assert lib.ofdmr_create(C.byref(cfg), C.byref(h)) == 2   # dft_ce L > N (estimation.cpp:26)
