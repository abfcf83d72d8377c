"""ctypes binding of the C ABI declared in include/me_b200.h (libme_b200.so).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_1002_1168_b200/csrc``).  There is no CPU fallback: if the
library is missing, every entry point raises ``ImportError``; if it is present
but no sm_100 device exists, the compute entry points return ME_ERR_NO_DEVICE
and this module raises ``RuntimeError``.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libme_b200.so")

ME_OK, ME_ERR_INVALID_ARGUMENT, ME_ERR_OUT_OF_RANGE, ME_ERR_CUDA, ME_ERR_NO_DEVICE, ME_ERR_RUNTIME = range(6)


class MeConfig(C.Structure):
    _fields_ = [
        ("algo", C.c_int32),
        ("search_range", C.c_int32),
        ("block_size", C.c_int32),
        ("ref_distance", C.c_int32),
        ("halfpel", C.c_int32),
        ("max_iterations", C.c_int32),
        ("step", C.c_int32),
        ("boundary_temporal", C.c_int32),
        ("epsilon", C.c_double),
        ("theta", C.c_double),
    ]


class MeBlockRec(C.Structure):
    _fields_ = [
        ("dx", C.c_int16),
        ("dy", C.c_int16),
        ("cost_q4", C.c_uint32),
        ("comparisons", C.c_uint16),
        ("dpd_steps", C.c_uint16),
        ("iterations", C.c_uint8),
        ("type", C.c_uint8),
        ("reserved", C.c_uint16),
    ]


class MePairStats(C.Structure):
    _fields_ = [
        ("block_comparisons", C.c_int64),
        ("dpd_refinement_steps", C.c_int64),
        ("blocks_opaque", C.c_int64),
        ("blocks_boundary", C.c_int64),
        ("blocks_transparent", C.c_int64),
        ("sse", C.c_int64),
    ]


class MeTuning(C.Structure):
    """me_tuning (include/me_b200.h): kernel-schedule knobs of a context; zeros = defaults."""

    _fields_ = [(n, C.c_int32) for n in (
        "pa_schedule", "pa_wide_blocks", "pa_fast_ctas", "pa_quad_ctas", "pa_duo_threads", "pa_duo_ctas", "pa_poll_ns",
        "pa_static_claim", "pa_no_pdl", "pa_no_smem_pair", "pa_fast_patches", "pa_key_a", "pa_key_s", "sort_no_pdl", "fill_rows",
        "fill_rows_per_cta", "h2d_chunks", "mask_pack", "ring_ctas", "host_threads")] + [("pa_trace_path", C.c_char_p), ("pa_key_plain", C.c_int32)]


PA_SCHEDULES = {"auto": 0, "warp": 1, "generic": 1, "fast": 2, "duo": 3, "duo-hybrid": 4, "hybrid": 5, "quad": 5}


class MeSynthParams(C.Structure):
    _fields_ = [
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("frames", C.c_int32),
        ("seed", C.c_uint64),
        ("blur_sigma_q8", C.c_int32),
        ("bg_jitter", C.c_int32),
        ("bg_drift_q8", C.c_int32 * 2),
        ("n_objects", C.c_int32),
        ("obj_min", C.c_int32),
        ("obj_max", C.c_int32),
        ("obj_w", C.c_int32 * 4),
        ("obj_h", C.c_int32 * 4),
        ("obj_v", (C.c_int32 * 2) * 4),
        ("vel_fixed", C.c_int32),
        ("vmax", C.c_int32),
        ("shapes", C.c_int32),
        ("noise_sigma_q8", C.c_int32),
    ]


# numpy dtype of me_block_rec (16 bytes)
def rec_dtype():
    import numpy as np

    return np.dtype(
        [
            ("dx", "<i2"),
            ("dy", "<i2"),
            ("cost_q4", "<u4"),
            ("comparisons", "<u2"),
            ("dpd_steps", "<u2"),
            ("iterations", "u1"),
            ("type", "u1"),
            ("reserved", "<u2"),
        ]
    )


def stats_dtype():
    import numpy as np

    return np.dtype(
        [
            ("block_comparisons", "<i8"),
            ("dpd_refinement_steps", "<i8"),
            ("blocks_opaque", "<i8"),
            ("blocks_boundary", "<i8"),
            ("blocks_transparent", "<i8"),
            ("sse", "<i8"),
        ]
    )


P = C.c_void_p
I = C.c_int
I32P = C.POINTER(C.c_int32)
I64P = C.POINTER(C.c_int64)
U32P = C.POINTER(C.c_uint32)
U8P = C.POINTER(C.c_uint8)

# name -> (restype, argtypes); every symbol include/me_b200.h declares
SIGNATURES = {
    "me_b200_version": (C.c_char_p, []),
    "me_b200_last_error": (C.c_char_p, []),
    "me_b200_device_count": (I, []),
    "me_b200_ctx_create": (I, [I, C.POINTER(P)]),
    "me_b200_ctx_destroy": (None, [P]),
    "me_b200_ctx_stream": (P, [P]),
    "me_b200_validate_config": (I, [C.POINTER(MeConfig)]),
    "me_b200_ctx_set_profiling": (I, [P, I]),
    "me_b200_ctx_stage_ms": (I, [P, C.POINTER(C.c_float), I]),
    "me_b200_ctx_transfer_bytes": (I, [P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "me_b200_ctx_launches": (I, [P, C.POINTER(C.c_int64)]),
    "me_b200_pack_mask": (I, [P, C.c_size_t, P, C.c_size_t, C.POINTER(C.c_size_t)]),
    "me_b200_run_sequences_dev": (I, [P, C.POINTER(MeConfig), I, I, I, I, P, P, P, P, P, P]),
    "me_b200_run_sequences": (I, [P, C.POINTER(MeConfig), I, I, I, I, P, P, P, P, P]),
    "me_b200_run_sequences_bits_dev": (I, [P, C.POINTER(MeConfig), I, I, I, I, P, P, P, P, P, P]),
    "me_b200_pack_mask_dev": (I, [P, P, C.c_size_t, P, C.POINTER(C.c_int), P]),
    "me_b200_run_sequence_prev_dev": (I, [P, C.POINTER(MeConfig), I, I, I, P, P, P, I, P, P, P]),
    "me_b200_run_band_dev": (I, [P, C.POINTER(MeConfig), I, I, I, I, P, P, I, I, P, P, P]),
    "me_b200_run_sequences_multi": (I, [C.POINTER(MeConfig), I, I, I, I, P, P, P, P, I]),
    "me_b200_estimate_field": (I, [P, C.POINTER(MeConfig), I, I, P, P, P, P, P, I, I, P, P]),
    "me_b200_block_search": (I, [P, I, I, I, P, P, I, I, I, I, I32P, I64P, U32P]),
    "me_b200_brs_select": (I, [P, I, I, P, P, P, P, I, I, I, I, I32P, I, I, I32P, U8P, U32P]),
    "me_b200_prs_refine": (I, [P, I, I, P, P, I, I, I, I32P, I, C.c_double, C.c_double, I, I, I32P, I64P, U32P, C.POINTER(I)]),
    "me_b200_prs_update": (I, [P, I, I, P, P, I, I, I32P, C.c_double, C.c_double, C.POINTER(C.c_double)]),
    "me_b200_sad_texture": (I, [P, I, I, P, P, I, I, I, I, I, U32P]),
    "me_b200_sad_shape": (I, [P, I, I, P, P, I, I, I, I, I, I64P]),
    "me_b200_classify_blocks": (I, [P, I, I, P, I, P]),
    "me_b200_binarize": (I, [P, I, I, P, I, P]),
    "me_b200_predict_frame": (I, [P, I, I, P, P, P, I, P, P, I64P]),
    "me_b200_sse": (I, [P, I, I, P, P, I64P]),
    "me_b200_probe_int_peak": (I, [P, C.POINTER(C.c_double)]),
    "me_b200_ctx_set_tuning": (I, [P, C.POINTER(MeTuning)]),
    "me_b200_ctx_get_tuning": (I, [P, C.POINTER(MeTuning)]),
    "me_b200_synth_preset": (I, [I, C.c_uint64, C.POINTER(MeSynthParams)]),
    "me_b200_synth": (I, [C.POINTER(MeSynthParams), P, P]),
    "me_b200_synth_dev": (I, [P, C.POINTER(MeSynthParams), I, P, P, P]),
}

_lib = None
_lock = threading.Lock()


def lib():
    """Loads libme_b200.so (raises ImportError when it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                    "(there is no CPU fallback)"
                )
            L = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def check(status: int):
    """Maps an me_status to the reference's exception types."""
    if status == ME_OK:
        return
    msg = lib().me_b200_last_error().decode(errors="replace")
    if status == ME_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)  # std::invalid_argument
    if status == ME_ERR_OUT_OF_RANGE:
        raise IndexError(msg)  # std::out_of_range
    raise RuntimeError(f"me_b200 error {status}: {msg}")


_tls = threading.local()


def ctx(device: int = 0):
    """Per-thread, per-device context (me_ctx*)."""
    cache = getattr(_tls, "ctxs", None)
    if cache is None:
        cache = _tls.ctxs = {}
    if device not in cache:
        h = P()
        check(lib().me_b200_ctx_create(device, C.byref(h)))
        cache[device] = h
    return cache[device]


def set_tuning(device: int = 0, **fields):
    """Sets this thread's context tuning (me_b200_ctx_set_tuning); unnamed
    fields take their defaults.  `pa_schedule` may be a name (PA_SCHEDULES).
    Returns the previous tuning (pass it back to restore)."""
    prev = MeTuning()
    check(lib().me_b200_ctx_get_tuning(ctx(device), C.byref(prev)))
    t = MeTuning()
    for k, v in fields.items():
        if k == "pa_schedule" and isinstance(v, str):
            v = PA_SCHEDULES[v]
        if k == "pa_trace_path" and isinstance(v, str):
            v = v.encode()
        setattr(t, k, v)
    check(lib().me_b200_ctx_set_tuning(ctx(device), C.byref(t)))
    return prev


def restore_tuning(prev, device: int = 0):
    check(lib().me_b200_ctx_set_tuning(ctx(device), C.byref(prev)))
