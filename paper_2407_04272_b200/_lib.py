"""ctypes binding of the C ABI in include/embc_cuda.h (libembc_cuda.so).

The shared library is built in-tree (``make -C paper_2407_04272_b200/csrc``)
and loaded from this package directory.  There is no fallback: if the library
is missing or a call fails, an exception is raised.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EMBC_LIB") or os.path.join(HERE, "libembc_cuda.so")  # EMBC_LIB: A/B builds
CSRC = os.path.join(HERE, "csrc")

# ---- status / reason codes (embc_cuda.h) ----------------------------------
OK, ERR_VALUE, ERR_FORMAT, ERR_CONFIG, ERR_CUDA, ERR_CAPACITY, ERR_ARGUMENT, ERR_UNSUPPORTED, ERR_NCCL = range(9)
CODEC_RAW, CODEC_VLZ, CODEC_HUFFMAN = 0, 1, 2
LAYOUT_CHUNKS, LAYOUT_PACKED, LAYOUT_PAYLOAD = 0, 1, 2
SRC_F32, SRC_I32 = 0, 1
OUT_F32, OUT_F64, OUT_I32 = 0, 1, 2

REASONS = {
    0: "none", 1: "nonfinite", 2: "overflow", 3: "eb_too_small", 4: "bad_window", 5: "truncated",
    6: "varint_long", 7: "vlz_dim0", 8: "vlz_bad_offset", 9: "vlz_bad_tag", 10: "vlz_trailing",
    11: "huf_empty", 12: "huf_len_cap", 13: "huf_empty_book", 14: "huf_len_range", 15: "huf_kraft",
    16: "huf_prefix", 17: "huf_dup", 18: "huf_exhausted", 19: "huf_bad_code", 20: "bad_magic",
    21: "bad_version", 22: "bad_codec", 23: "paylen", 24: "bad_eb", 25: "raw_size", 26: "huf_count",
    27: "dim0", 28: "pack_offset", 29: "pack_overrun", 30: "pack_trailing", 31: "capacity",
    32: "meta_mismatch", 33: "range",
}


class EmbcError(RuntimeError):
    """Base of all codec failures (embc::Error, errors.hpp:24-27)."""

    def __init__(self, msg: str, status: int = 0, reason: int = 0, job: int = 0, index: int = 0):
        super().__init__(msg)
        self.status = status
        self.reason = reason
        self.reason_name = REASONS.get(reason, str(reason))
        self.job = job
        self.index = index


class CodecValueError(EmbcError, ValueError):
    """embc::ValueError (errors.hpp:30-33)."""


class CodecFormatError(EmbcError):
    """embc::FormatError (errors.hpp:36-39)."""


class CodecConfigError(EmbcError):
    """embc::ConfigError (errors.hpp:42-45)."""


class CodecUnsupported(EmbcError):
    """Input outside the GPU path's envelope (EMBC_ERR_UNSUPPORTED)."""


_STATUS_EXC = {ERR_VALUE: CodecValueError, ERR_FORMAT: CodecFormatError,
               ERR_CONFIG: CodecConfigError, ERR_UNSUPPORTED: CodecUnsupported}


class EmbcErrorRec(C.Structure):
    _fields_ = [("status", C.c_int32), ("reason", C.c_int32), ("job", C.c_uint32), ("pad", C.c_uint32),
                ("index", C.c_uint64), ("a", C.c_uint64), ("b", C.c_uint64), ("message", C.c_char * 320)]


class Job(C.Structure):
    _fields_ = [("src", C.c_void_p), ("dim", C.c_uint32), ("n", C.c_uint32), ("eb", C.c_double),
                ("window", C.c_uint32), ("codec", C.c_uint8), ("src_kind", C.c_uint8),
                ("pad", C.c_uint8 * 2)]


class ExchangeStats(C.Structure):
    _fields_ = [("uncompressed_bytes", C.c_uint64), ("payload_bytes", C.c_uint64), ("metadata_bytes", C.c_uint64),
                ("sent_values", C.c_uint64), ("sent_bytes", C.c_uint64), ("recv_values", C.c_uint64),
                ("recv_bytes", C.c_uint64)]


class SimTable(C.Structure):
    _fields_ = [("rows", C.c_uint32), ("dim", C.c_uint32), ("dist", C.c_int32), ("pad", C.c_uint32),
                ("mu", C.c_double), ("sigma", C.c_double), ("lo", C.c_double), ("hi", C.c_double),
                ("zipf_s", C.c_double)]


class SimConfig(C.Structure):
    _fields_ = [("ranks", C.c_uint32), ("batch", C.c_uint32), ("iterations", C.c_uint32),
                ("compression", C.c_uint32), ("seed", C.c_uint64), ("global_eb", C.c_double),
                ("decay_fn", C.c_int32), ("decay_steps", C.c_uint32), ("decay_start_scale", C.c_double),
                ("decay_end", C.c_uint64)]


class SimIteration(C.Structure):
    _fields_ = [("iteration", C.c_uint64), ("eb_max", C.c_double), ("uncompressed_bytes", C.c_uint64),
                ("payload_bytes", C.c_uint64), ("metadata_bytes", C.c_uint64), ("wire_bytes", C.c_uint64),
                ("comp_time", C.c_double), ("decomp_time", C.c_double), ("max_abs_error", C.c_double),
                ("delivery_conserved", C.c_uint64), ("delivered_digest", C.c_uint64)]


class ChunkRef(C.Structure):
    _fields_ = [("offset", C.c_uint64), ("length", C.c_uint64), ("out", C.c_void_p),
                ("dim", C.c_uint32), ("count", C.c_uint32), ("eb", C.c_double), ("codec", C.c_uint8),
                ("pad", C.c_uint8 * 7)]


# every symbol include/embc_cuda.h declares (checked by the CPU test suite)
EXPORTS = [
    "embc_ctx_create", "embc_ctx_destroy", "embc_reserve", "embc_sync", "embc_get_error",
    "embc_version", "embc_encode_bound", "embc_encode", "embc_decode", "embc_quantize",
    "embc_dequantize", "embc_match_stats", "embc_pattern_counts", "embc_decay_multiplier",
    "embc_classify_table", "embc_estimate_speedup", "embc_gen_table", "embc_gen_lookup_indices",
    "embc_mix_seed", "embc_gather_rows", "embc_reserve_capture", "embc_capture_reset",
    "embc_timing_enable", "embc_timing_collect", "embc_decode_fallbacks",
    "embc_exchange_unique_id", "embc_exchange_create", "embc_exchange_destroy", "embc_exchange_get_error",
    "embc_exchange_fwd", "embc_exchange_bwd", "embc_exchange_baseline_fwd", "embc_exchange_baseline_bwd",
    "embc_unpack", "embc_exchange_timing_enable", "embc_exchange_timing_collect", "embc_simulate", "embc_decode_dev",
    "embc_exchange_set_mode", "embc_exchange_sync", "embc_exchange_reserve_capture",
]

_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile libembc_cuda.so for sm_100a (nvcc cross-compiles without a GPU)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-j8", "-C", CSRC], check=True)
    return LIB_PATH


def lib() -> C.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                build()
            L = C.CDLL(LIB_PATH)
            vp, u32, u64, i32, dbl = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int, C.c_double
            sig = {
                "embc_ctx_create": (i32, [i32, C.POINTER(vp)]),
                "embc_ctx_destroy": (None, [vp]),
                "embc_reserve": (i32, [vp, u32, u64, u64]),
                "embc_sync": (i32, [vp, vp]),
                "embc_get_error": (i32, [vp, C.POINTER(EmbcErrorRec)]),
                "embc_version": (C.c_char_p, []),
                "embc_encode_bound": (u64, [C.POINTER(Job), u32, i32]),
                "embc_encode": (i32, [vp, C.POINTER(Job), u32, i32, vp, u64, vp, vp, vp, vp, vp]),
                "embc_decode": (i32, [vp, vp, C.POINTER(ChunkRef), u32, i32, i32, vp]),
                "embc_decode_dev": (i32, [vp, vp, C.POINTER(ChunkRef), u32, vp, vp, i32, i32, vp]),
                "embc_quantize": (i32, [vp, vp, i32, u64, dbl, vp, vp]),
                "embc_dequantize": (i32, [vp, vp, u64, dbl, vp, i32, vp]),
                "embc_match_stats": (i32, [vp, vp, u32, u32, u32, C.POINTER(u64), C.POINTER(u64), vp]),
                "embc_pattern_counts": (i32, [vp, vp, u32, u32, dbl, C.POINTER(u64), C.POINTER(u64), vp]),
                "embc_decay_multiplier": (i32, [u64, i32, dbl, u64, u32, C.POINTER(dbl)]),
                "embc_classify_table": (i32, [dbl, dbl, dbl, dbl, dbl, dbl, C.POINTER(i32), C.POINTER(dbl)]),
                "embc_estimate_speedup": (i32, [dbl, dbl, dbl, dbl, C.POINTER(dbl)]),
                "embc_gen_table": (i32, [u32, u32, i32, dbl, dbl, dbl, dbl, u64, vp]),
                "embc_gen_lookup_indices": (i32, [u32, dbl, u64, u32, u64, vp]),
                "embc_mix_seed": (u64, [u64, u64]),
                "embc_gather_rows": (i32, [vp, u32, vp, u32, vp, vp]),
                "embc_reserve_capture": (i32, [vp, u64]),
                "embc_capture_reset": (i32, [vp]),
                "embc_timing_enable": (i32, [vp, i32]),
                "embc_timing_collect": (i32, [vp, vp, C.c_char_p, C.c_size_t, C.POINTER(C.c_float), i32]),
                "embc_decode_fallbacks": (i32, [vp, C.POINTER(u32)]),
                "embc_exchange_unique_id": (i32, [vp]),
                "embc_exchange_create": (i32, [i32, i32, i32, vp, u32, C.POINTER(vp)]),
                "embc_exchange_destroy": (None, [vp]),
                "embc_exchange_get_error": (i32, [vp, C.POINTER(EmbcErrorRec)]),
                "embc_exchange_fwd": (i32, [vp, u32, u32, u32, vp, vp, vp, u32, vp, C.POINTER(ExchangeStats), vp]),
                "embc_exchange_bwd": (i32, [vp, u32, u32, u32, vp, vp, vp, u32, vp, C.POINTER(ExchangeStats), vp]),
                "embc_exchange_baseline_fwd": (i32, [vp, u32, u32, u32, vp, vp, vp]),
                "embc_exchange_baseline_bwd": (i32, [vp, u32, u32, u32, vp, vp, vp]),
                "embc_exchange_timing_enable": (i32, [vp, i32]),
                "embc_exchange_set_mode": (i32, [vp, i32]),
                "embc_exchange_sync": (i32, [vp]),
                "embc_exchange_reserve_capture": (i32, [vp, u64]),
                "embc_exchange_timing_collect": (i32, [vp, C.c_char_p, C.c_size_t, C.POINTER(C.c_float), i32]),
                "embc_unpack": (i32, [vp, u64, vp, vp, u32, C.POINTER(u32), C.POINTER(EmbcErrorRec)]),
                "embc_simulate": (i32, [i32, C.POINTER(SimConfig), C.POINTER(SimTable), u32, vp, vp,
                                        C.POINTER(SimIteration), C.POINTER(u64), C.POINTER(EmbcErrorRec)]),
            }
            for name, (res, args) in sig.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
        return _lib


def raise_for(status: int, msg: str, reason: int = 0, job: int = 0, index: int = 0):
    if status == OK:
        return
    exc = _STATUS_EXC.get(status, EmbcError)
    raise exc(msg, status=status, reason=reason, job=job, index=index)


def host_check(status: int, what: str):
    """Status of a host-only entry point (no context)."""
    if status != OK:
        raise_for(status, f"{what} failed with status {status}")
