"""ctypes bindings for the in-tree native libraries.

The CUDA receiver library is REQUIRED: importing the receiver on a machine where
libofdmr_b200.so is missing raises immediately (there is no CPU fallback path).
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

PKG = Path(__file__).resolve().parent
import os

LIB_PATH = Path(os.environ["OFDMR_LIB"]) if os.environ.get("OFDMR_LIB") else PKG / "libofdmr_b200.so"
GEN_PATH = PKG / "libofdmr_gen.so"

vp = C.c_void_p
i32 = C.c_int32
i64 = C.c_int64
u64 = C.c_uint64
f64 = C.c_double
P_i32 = C.POINTER(C.c_int32)
P_f64 = C.POINTER(C.c_double)


class OfdmrConfig(C.Structure):
    """ofdmr_config (include/ofdmr_b200.h)."""

    _fields_ = [
        ("n_subcarriers", i32),
        ("n_symbols", i32),
        ("n_prime", i32),
        ("m_prime", i32),
        ("window", i32),
        ("estimator", i32),
        ("n_cp", i32),
        ("max_targets", i32),
        ("pfa", f64),
        ("chunk_frames", i32),
        ("device", i32),
    ]


class OfdmrSftConfig(C.Structure):
    """ofdmr_sft_config (include/ofdmr_b200.h) — SftConfig, sft.hpp:14-33."""

    _fields_ = [
        ("i_max", i32),
        ("detect_threshold", f64),
        ("pfa", f64),
        ("decimation", i32),
        ("frac_tol", f64),
        ("amp_tol", f64),
        ("max_entries", i32),
    ]


class GenParams(C.Structure):
    """ofdmr_gen_params (csrc/gen.cpp)."""

    _fields_ = [
        ("n", i32),
        ("m", i32),
        ("df_hz", f64),
        ("fc_hz", f64),
        ("n_cp", i32),
        ("qam_order", i32),
        ("zc_precode", i32),
        ("zc_root", i64),
        ("targets_min", i32),
        ("targets_max", i32),
        ("range_lo", f64),
        ("range_hi", f64),
        ("vel_lo", f64),
        ("vel_hi", f64),
        ("snr_lo_db", f64),
        ("snr_hi_db", f64),
    ]


# (name, restype, argtypes) for every symbol declared in include/ofdmr_b200.h
RECEIVER_SYMBOLS = [
    ("ofdmr_create", i32, [C.POINTER(OfdmrConfig), C.POINTER(vp)]),
    ("ofdmr_destroy", None, [vp]),
    ("ofdmr_set_stream", i32, [vp, vp]),
    ("ofdmr_last_error", C.c_char_p, []),
    ("ofdmr_launch_count", i64, [vp]),
    ("ofdmr_set_profiling", i32, [vp, i32]),
    ("ofdmr_get_profile", i32, [vp, vp, vp]),
    ("ofdmr_make_window", i32, [i32, i32, i32, P_f64, P_f64]),
    ("ofdmr_window_power_factor", f64, [i32, i32, i32]),
    ("ofdmr_detection_threshold", i32, [f64, f64, f64, P_f64]),
    ("ofdmr_bins_to_physics", None, [i64, i64, i32, i32, i32, i32, f64, f64, P_f64, P_f64]),
    ("ofdmr_spectral_division", i32, [vp, vp, vp, vp, vp, i64]),
    ("ofdmr_dft_ce", i32, [vp, vp, vp, i64]),
    ("ofdmr_estimate_channel", i32, [vp, vp, vp, vp, vp, i64]),
    ("ofdmr_periodogram", i32, [vp, vp, vp, i64]),
    ("ofdmr_detect", i32, [vp, vp, vp, vp, vp, vp, vp, vp, i64]),
    ("ofdmr_extract_peaks", i32, [vp, vp, vp, vp, vp, vp, vp, vp, i64]),
    ("ofdmr_estimate_noise_power", i32, [vp, vp, vp, i64]),
    ("ofdmr_ofdm_demodulate", i32, [vp, vp, vp, i64]),
    ("ofdmr_ofdm_modulate", i32, [vp, vp, vp, i64]),
    ("ofdmr_map_to_pgm", i32, [vp, vp, vp, i64]),
    ("ofdmr_pipeline", i32, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i64]),
    ("ofdmr_pipeline_general", i32, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i64]),
    ("ofdmr_pipeline_host", i32, [vp, vp, vp, vp, vp, vp, vp, vp, vp, i64]),
    ("ofdmr_sft", i32, [vp, vp, i32, i32, C.POINTER(OfdmrSftConfig), vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                        i64]),
    ("ofdmr_sft_detections", i32, [vp, vp, vp, vp, vp, i32, i32, i32, vp, C.c_double, vp, vp, vp, vp, vp, i64]),
    ("ofdmr_sft_detect", i32, [vp, vp, i32, i32, C.POINTER(OfdmrSftConfig), vp, vp, vp, vp, vp, vp, vp, vp, i64]),
    ("ofdmr_pipeline_sft", i32, [vp, vp, vp, vp, vp, vp, C.POINTER(OfdmrSftConfig), vp, vp, vp, vp, vp, vp, vp,
                                 i64]),
    ("ofdmr_sft_estimate_noise", i32, [vp, vp, i32, i32, vp, vp, i64]),
    ("ofdmr_shard_range", None, [i64, i32, i32, vp, vp]),
    ("ofdmr_multi_create", i32, [C.POINTER(OfdmrConfig), vp, i32, vp]),
    ("ofdmr_multi_destroy", None, [vp]),
    ("ofdmr_multi_devices", i32, [vp]),
    ("ofdmr_multi_context", vp, [vp, i32]),
    ("ofdmr_multi_last_error", C.c_char_p, []),
    ("ofdmr_multi_pipeline_host", i32, [vp, vp, vp, vp, vp, vp, vp, vp, vp, i64]),
    ("ofdmr_multi_pipeline", i32, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i64]),
]

# include/ofdmr_gen.h, device side (in the CUDA library)
DEVICE_GEN_SYMBOLS = [
    ("ofdmr_gen_device", i32, [C.POINTER(GenParams), u64, i64, i64, vp, vp, vp, vp, vp, vp, vp, i32, vp, vp]),
    ("ofdmr_gen_device_explicit", i32, [C.POINTER(GenParams), u64, i64, i64, P_f64, P_f64, i32, f64, vp, vp, vp, vp,
                                        vp, vp]),
    ("ofdmr_channel_mse", i32, [vp, vp, i64, i64, vp, vp]),
]

GEN_SYMBOLS = [
    ("ofdmr_derive_seed", u64, [u64, u64]),
    ("ofdmr_gen_frame", i32, [C.POINTER(GenParams), u64, i64, vp, vp, vp, vp, vp, vp, vp, i32]),
    ("ofdmr_gen_frame_explicit", i32, [C.POINTER(GenParams), vp, vp, i32, f64, u64, vp, vp, vp]),
    ("ofdmr_gen_batch", i32, [C.POINTER(GenParams), u64, i64, i64, vp, vp, vp, vp, vp, vp, vp, i32, C.c_int]),
    ("ofdmr_gen_sparse", i32, [i32, i32, i32, f64, u64, i64, vp, vp, vp, vp, vp, vp]),
    ("ofdmr_gen_sparse_batch", i32, [i32, i32, i32, f64, u64, i64, i64, vp, vp, vp, vp, C.c_int]),
    ("ofdmr_gen_noise_grid", i32, [i32, i32, f64, u64, vp]),
    ("ofdmr_rng_u64", None, [u64, i64, vp]),
]


def _bind(lib: C.CDLL, table) -> C.CDLL:
    for name, res, args in table:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = None
_gen = None


def lib() -> C.CDLL:
    """The CUDA receiver library; raises if it was not built (no silent fallback)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2209_03883_b200.build` "
                "(there is no CPU fallback for the receiver path)"
            )
        _lib = _bind(C.CDLL(str(LIB_PATH)), RECEIVER_SYMBOLS + DEVICE_GEN_SYMBOLS)
    return _lib


def gen() -> C.CDLL:
    global _gen
    if _gen is None:
        if not GEN_PATH.exists():
            raise ImportError(f"{GEN_PATH} is missing: build it with `python -m paper_2209_03883_b200.build`")
        _gen = _bind(C.CDLL(str(GEN_PATH)), GEN_SYMBOLS)
    return _gen


def last_error() -> str:
    msg = lib().ofdmr_last_error()
    return msg.decode() if msg else ""
