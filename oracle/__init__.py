"""Test-only CPU checkers for the codec path.

  Oracle -- oracle/liboracle.so, the plain-C restatement of the reference
            algorithm (embc_oracle.c), each function citing reference file:line.
  Ref    -- oracle/_ref/libembc_ref.so, the reference headers themselves
            (/root/reference/proj/include) compiled unmodified behind a thin
            C shim (ref_shim.cpp).  Built here; the prebuilt .so travels to the
            GPU box.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
legs may import this package.  The product library never links or calls it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libembc_ref.so")


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class OracleError(Exception):
    """A failure reported by a checker: kind 'value' or 'format' + detail."""

    def __init__(self, kind: str, msg: str = "", sub: int = 0, index: int = 0, a: int = 0, b: int = 0):
        super().__init__(f"{kind}: {msg or sub}")
        self.kind, self.msg, self.sub, self.index, self.a, self.b = kind, msg, sub, index, a, b


_KIND = {1: "value", 2: "format", 3: "error", 4: "std"}


class _OErr(C.Structure):
    _fields_ = [("kind", C.c_int), ("sub", C.c_int), ("index", C.c_uint64), ("a", C.c_uint64),
                ("b", C.c_uint64)]


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None and a.size else None


class Oracle:
    """The C restatement (embc_oracle.c)."""

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            build()
        self.L = C.CDLL(ORACLE_SO)
        L = self.L
        vp, u32, u64, i32, dbl = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int, C.c_double
        pe = C.POINTER(_OErr)
        for name, res, args in [
            ("orc_quantize_f64", i32, [vp, u64, dbl, vp, pe]),
            ("orc_quantize_f32", i32, [vp, u64, dbl, vp, pe]),
            ("orc_dequantize_f64", None, [vp, u64, dbl, vp]),
            ("orc_match_stats", i32, [vp, u32, u32, u32, C.POINTER(u64), C.POINTER(u64), pe]),
            ("orc_vlz_encode", i32, [vp, u32, u32, u32, vp, u64, C.POINTER(u64), pe]),
            ("orc_vlz_decode", i32, [vp, u64, u32, u32, vp, pe]),
            ("orc_huff_codebook", i32, [vp, u64, vp, vp, vp, C.POINTER(u32), pe]),
            ("orc_huff_from_histogram", i32, [vp, vp, u32, vp, vp, pe]),
            ("orc_huff_encode", i32, [vp, u64, vp, u64, C.POINTER(u64), pe]),
            ("orc_huff_decode", i32, [vp, u64, vp, u64, C.POINTER(u64), pe]),
            ("orc_encode_chunk", i32, [vp, u32, u32, dbl, i32, u32, vp, u64, C.POINTER(u64), pe]),
            ("orc_decode_chunk", i32, [vp, u64, vp, u64, C.POINTER(u32), C.POINTER(u32), pe]),
            ("orc_metadata", None, [vp, u64, vp]),
            ("orc_pack", i32, [C.POINTER(vp), vp, u32, vp, u64, C.POINTER(u64), pe]),
            ("orc_unpack", i32, [vp, u64, vp, vp, u32, C.POINTER(u32), pe]),
            ("orc_decay_multiplier", dbl, [u64, i32, dbl, u64, u32]),
            ("orc_classify", i32, [dbl, dbl, dbl]),
            ("orc_estimate_speedup", dbl, [dbl, dbl, dbl, dbl]),
            ("orc_unique_rows_f64", u64, [vp, u32, u32]),
            ("orc_unique_rows_i32", u64, [vp, u32, u32]),
        ]:
            f = getattr(L, name)
            f.restype, f.argtypes = res, args

    @staticmethod
    def _raise(rc, e: _OErr):
        if rc:
            raise OracleError(_KIND.get(rc, "error"), "", e.sub, e.index, e.a, e.b)

    def quantize(self, x: np.ndarray, eb: float) -> np.ndarray:
        out = np.zeros(x.size, np.int32)
        e = _OErr()
        if x.dtype == np.float32:
            rc = self.L.orc_quantize_f32(_p(x), x.size, eb, _p(out), C.byref(e))
        else:
            x = np.ascontiguousarray(x, np.float64)
            rc = self.L.orc_quantize_f64(_p(x), x.size, eb, _p(out), C.byref(e))
        self._raise(rc, e)
        return out

    def dequantize(self, codes: np.ndarray, eb: float) -> np.ndarray:
        out = np.zeros(codes.size, np.float64)
        self.L.orc_dequantize_f64(_p(np.ascontiguousarray(codes, np.int32)), codes.size, eb, _p(out))
        return out

    def match_stats(self, codes: np.ndarray, dim: int, window: int = 255):
        c = np.ascontiguousarray(codes, np.int32)
        lit, ref, e = C.c_uint64(), C.c_uint64(), _OErr()
        rc = self.L.orc_match_stats(_p(c), dim, c.size // dim if dim else 0, window, C.byref(lit), C.byref(ref),
                                    C.byref(e))
        self._raise(rc, e)
        return lit.value, ref.value

    def vlz_encode(self, codes: np.ndarray, dim: int, window: int = 255) -> bytes:
        c = np.ascontiguousarray(codes, np.int32)
        n = c.size // dim if dim else 0
        cap = n * max(6, 1 + 5 * dim) + 16
        out = np.zeros(cap, np.uint8)
        ln, e = C.c_uint64(), _OErr()
        rc = self.L.orc_vlz_encode(_p(c), dim, n, window, _p(out), cap, C.byref(ln), C.byref(e))
        self._raise(rc, e)
        return out[:ln.value].tobytes()

    def vlz_decode(self, tokens: bytes, dim: int, n: int) -> np.ndarray:
        t = np.frombuffer(tokens, np.uint8).copy()
        out = np.zeros(dim * n, np.int32)
        e = _OErr()
        rc = self.L.orc_vlz_decode(_p(t), t.size, dim, n, _p(out), C.byref(e))
        self._raise(rc, e)
        return out

    def huff_codebook(self, codes: np.ndarray):
        c = np.ascontiguousarray(codes, np.int32)
        k = max(1, len(np.unique(c)))
        syms, lens, cws = np.zeros(k, np.int32), np.zeros(k, np.uint8), np.zeros(k, np.uint32)
        n, e = C.c_uint32(), _OErr()
        rc = self.L.orc_huff_codebook(_p(c), c.size, _p(syms), _p(lens), _p(cws), C.byref(n), C.byref(e))
        self._raise(rc, e)
        return syms, lens, cws

    def huff_from_histogram(self, sym, cnt):
        s = np.ascontiguousarray(sym, np.int32)
        c = np.ascontiguousarray(cnt, np.uint64)
        os_, ol = np.zeros(len(s), np.int32), np.zeros(len(s), np.uint8)
        e = _OErr()
        rc = self.L.orc_huff_from_histogram(_p(s), _p(c), len(s), _p(os_), _p(ol), C.byref(e))
        self._raise(rc, e)
        return os_, ol

    def huff_encode(self, codes: np.ndarray) -> bytes:
        c = np.ascontiguousarray(codes, np.int32)
        cap = 12 + 9 * c.size + 16
        out = np.zeros(cap, np.uint8)
        ln, e = C.c_uint64(), _OErr()
        rc = self.L.orc_huff_encode(_p(c), c.size, _p(out), cap, C.byref(ln), C.byref(e))
        self._raise(rc, e)
        return out[:ln.value].tobytes()

    def huff_decode(self, data: bytes, cap: int | None = None) -> np.ndarray:
        t = np.frombuffer(data, np.uint8).copy()
        cap = cap if cap is not None else 8 * t.size + 1
        out = np.zeros(max(cap, 1), np.int32)
        cnt, e = C.c_uint64(), _OErr()
        rc = self.L.orc_huff_decode(_p(t), t.size, _p(out), cap, C.byref(cnt), C.byref(e))
        self._raise(rc, e)
        return out[:cnt.value]

    def encode_chunk(self, x: np.ndarray, dim: int, eb: float, codec: int, window: int = 255) -> bytes:
        v = np.ascontiguousarray(x, np.float64)
        n = v.size // dim if dim else 0
        cap = 30 + 12 + 9 * v.size + n * (1 + 5 * dim) + 64
        out = np.zeros(cap, np.uint8)
        ln, e = C.c_uint64(), _OErr()
        rc = self.L.orc_encode_chunk(_p(v), dim, n, eb, codec, window, _p(out), cap, C.byref(ln), C.byref(e))
        self._raise(rc, e)
        return out[:ln.value].tobytes()

    def decode_chunk(self, data: bytes):
        t = np.frombuffer(data, np.uint8).copy()
        dim = count = 0
        if len(data) >= 30:
            dim = int.from_bytes(data[14:18], "little")
            count = int.from_bytes(data[18:22], "little")
        cap = dim * count
        out = np.zeros(max(cap, 1), np.float64)
        d, n, e = C.c_uint32(), C.c_uint32(), _OErr()
        rc = self.L.orc_decode_chunk(_p(t), t.size, _p(out), cap, C.byref(d), C.byref(n), C.byref(e))
        self._raise(rc, e)
        return out[:d.value * n.value].reshape(n.value, d.value)

    def metadata(self, chunk: bytes) -> bytes:
        t = np.frombuffer(chunk, np.uint8).copy()
        out = np.zeros(25, np.uint8)
        self.L.orc_metadata(_p(t), t.size, _p(out))
        return out.tobytes()

    def pack(self, chunks) -> bytes:
        arrs = [np.frombuffer(c, np.uint8).copy() if len(c) else np.zeros(1, np.uint8) for c in chunks]
        ptrs = (C.c_void_p * max(len(arrs), 1))(*[a.ctypes.data for a in arrs])
        lens = np.array([len(c) for c in chunks] or [0], np.uint64)
        cap = 4 + 16 * len(chunks) + sum(len(c) for c in chunks)
        out = np.zeros(cap, np.uint8)
        ln, e = C.c_uint64(), _OErr()
        rc = self.L.orc_pack(ptrs, _p(lens), len(chunks), _p(out), cap, C.byref(ln), C.byref(e))
        self._raise(rc, e)
        return out[:ln.value].tobytes()

    def unpack(self, buf: bytes):
        t = np.frombuffer(buf, np.uint8).copy()
        mx = max(1, len(buf) // 16 + 1)
        offs, lens = np.zeros(mx, np.uint64), np.zeros(mx, np.uint64)
        k, e = C.c_uint32(), _OErr()
        rc = self.L.orc_unpack(_p(t), t.size, _p(offs), _p(lens), mx, C.byref(k), C.byref(e))
        self._raise(rc, e)
        return [(int(offs[i]), int(lens[i])) for i in range(k.value)]

    def decay_multiplier(self, it, fn=0, start=1.0, end=0, steps=4):
        return self.L.orc_decay_multiplier(it, fn, start, end, steps)

    def classify(self, survival, large_thr=0.70, small_thr=0.95):
        return self.L.orc_classify(survival, large_thr, small_thr)

    def estimate_speedup(self, ratio, bw, comp, decomp):
        return self.L.orc_estimate_speedup(ratio, bw, comp, decomp)

    def unique_rows(self, x: np.ndarray, dim: int) -> int:
        if x.dtype == np.int32:
            return int(self.L.orc_unique_rows_i32(_p(np.ascontiguousarray(x)), dim, x.size // dim))
        v = np.ascontiguousarray(x, np.float64)
        return int(self.L.orc_unique_rows_f64(_p(v), dim, v.size // dim))


class Ref:
    """The reference headers compiled unmodified (oracle/_ref/libembc_ref.so)."""

    available = os.path.exists(REF_SO)

    def __init__(self):
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        self.L = C.CDLL(REF_SO)
        L = self.L
        vp, u32, u64, i32, dbl, sz = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int, C.c_double, C.c_size_t
        pp = C.POINTER(C.c_void_p)
        for name, res, args in [
            ("ref_free", None, [vp]),
            ("ref_quantize", i32, [vp, u64, u32, dbl, vp, C.c_char_p, sz]),
            ("ref_dequantize", i32, [vp, u64, u32, dbl, vp, C.c_char_p, sz]),
            ("ref_encode_chunk", i32, [vp, u32, u32, dbl, i32, u32, pp, C.POINTER(u64), C.c_char_p, sz]),
            ("ref_decode_chunk", i32, [vp, u64, pp, C.POINTER(u64), C.POINTER(u32), C.POINTER(u32), C.c_char_p, sz]),
            ("ref_vlz_encode", i32, [vp, u32, u32, u32, pp, C.POINTER(u64), C.c_char_p, sz]),
            ("ref_vlz_decode", i32, [vp, u64, u32, u32, vp, C.c_char_p, sz]),
            ("ref_match_stats", i32, [vp, u32, u32, u32, C.POINTER(u64), C.POINTER(u64), C.c_char_p, sz]),
            ("ref_huff_encode", i32, [vp, u64, pp, C.POINTER(u64), C.c_char_p, sz]),
            ("ref_huff_decode", i32, [vp, u64, pp, C.POINTER(u64), C.c_char_p, sz]),
            ("ref_huff_codebook", i32, [vp, u64, vp, vp, vp, C.POINTER(u32), C.c_char_p, sz]),
            ("ref_huff_from_histogram", i32, [vp, vp, u32, vp, vp, C.c_char_p, sz]),
            ("ref_pack", i32, [pp, vp, u32, pp, C.POINTER(u64), C.c_char_p, sz]),
            ("ref_unpack", i32, [vp, u64, pp, pp, C.POINTER(u32), C.c_char_p, sz]),
            ("ref_metadata", i32, [vp, u64, vp, C.c_char_p, sz]),
            ("ref_gen_table", i32, [i32, u32, u32, i32, dbl, dbl, dbl, dbl, dbl, u64, vp, C.c_char_p, sz]),
            ("ref_lookup_indices", i32, [i32, u32, u32, i32, dbl, dbl, dbl, dbl, dbl, u64, u32, u64, vp,
                                         C.c_char_p, sz]),
            ("ref_mix_seed", u64, [u64, u64]),
            ("ref_pattern_counts", i32, [vp, u32, u32, dbl, C.POINTER(u64), C.POINTER(u64), C.c_char_p, sz]),
            ("ref_decay_multiplier", dbl, [u64, i32, dbl, u64, u32]),
            ("ref_classify", i32, [dbl, dbl, dbl, dbl, dbl, dbl, C.POINTER(i32), C.POINTER(dbl), C.c_char_p, sz]),
            ("ref_estimate_speedup", dbl, [dbl, dbl, dbl, dbl]),
            ("ref_codec_timed", i32, [vp, vp, vp, vp, vp, vp, u32, C.c_uint, i32, C.POINTER(dbl), C.POINTER(dbl),
                                      C.POINTER(u64), C.c_char_p, sz]),
            ("ref_load_preset", i32, [C.c_char_p, u32, C.POINTER(u32), vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                      C.POINTER(i32), C.POINTER(dbl), C.POINTER(u64), C.POINTER(u32),
                                      C.POINTER(u32), C.POINTER(u32), C.c_char_p, sz]),
            ("ref_offline_analysis", i32, [vp, vp, vp, vp, vp, u32, dbl, dbl, dbl, dbl, dbl, dbl, u32, C.c_char_p,
                                           C.c_char_p, sz]),
            ("ref_read_profiles", i32, [C.c_char_p, u32, C.POINTER(u32), vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                        C.c_char_p, sz]),
            ("ref_encode_pack", i32, [vp, vp, vp, vp, vp, vp, u32, u32, C.c_uint, pp, C.POINTER(u64), C.c_char_p,
                                      sz]),
            ("ref_format_double", None, [dbl, C.c_char_p, sz]),
            ("ref_simulate", i32, [u32, u32, u32, u64, i32, dbl, dbl, u64, u32, vp, vp, vp, vp, vp, vp, vp, vp,
                                   u32, vp, vp, vp, vp, vp, vp, vp, C.POINTER(u64), C.c_char_p, sz]),
        ]:
            f = getattr(L, name)
            f.restype, f.argtypes = res, args

    def _call(self, fn, *args):
        err = C.create_string_buffer(512)
        rc = fn(*args, err, 512)
        if rc:
            raise OracleError(_KIND.get(rc, "error"), err.value.decode())

    def _take(self, ptr: C.c_void_p, n: int, dtype) -> np.ndarray:
        if not ptr.value:
            return np.zeros(0, dtype)
        buf = (C.c_char * (n * np.dtype(dtype).itemsize)).from_address(ptr.value)
        out = np.frombuffer(bytes(buf), dtype).copy()
        self.L.ref_free(ptr)
        return out

    def quantize(self, x: np.ndarray, eb: float, dim: int = 1) -> np.ndarray:
        v = np.ascontiguousarray(x, np.float64)
        out = np.zeros(v.size, np.int32)
        self._call(self.L.ref_quantize, _p(v), v.size, dim, eb, _p(out))
        return out

    def dequantize(self, codes: np.ndarray, eb: float, dim: int = 1) -> np.ndarray:
        c = np.ascontiguousarray(codes, np.int32)
        out = np.zeros(c.size, np.float64)
        self._call(self.L.ref_dequantize, _p(c), c.size, dim, eb, _p(out))
        return out

    def encode_chunk(self, x: np.ndarray, dim: int, eb: float, codec: int, window: int = 255) -> bytes:
        v = np.ascontiguousarray(x, np.float64)
        p, ln = C.c_void_p(), C.c_uint64()
        self._call(self.L.ref_encode_chunk, _p(v), dim, v.size // dim if dim else 0, eb, codec, window,
                   C.byref(p), C.byref(ln))
        return self._take(p, ln.value, np.uint8).tobytes()

    def decode_chunk(self, data: bytes) -> np.ndarray:
        t = np.frombuffer(data, np.uint8).copy() if len(data) else np.zeros(0, np.uint8)
        p, n, d, k = C.c_void_p(), C.c_uint64(), C.c_uint32(), C.c_uint32()
        self._call(self.L.ref_decode_chunk, _p(t), len(data), C.byref(p), C.byref(n), C.byref(d), C.byref(k))
        return self._take(p, n.value, np.float64).reshape(k.value, d.value)

    def vlz_encode(self, codes: np.ndarray, dim: int, window: int = 255) -> bytes:
        c = np.ascontiguousarray(codes, np.int32)
        p, ln = C.c_void_p(), C.c_uint64()
        self._call(self.L.ref_vlz_encode, _p(c), dim, c.size // dim if dim else 0, window, C.byref(p), C.byref(ln))
        return self._take(p, ln.value, np.uint8).tobytes()

    def vlz_decode(self, tokens: bytes, dim: int, n: int) -> np.ndarray:
        t = np.frombuffer(tokens, np.uint8).copy() if tokens else np.zeros(0, np.uint8)
        out = np.zeros(dim * n, np.int32)
        self._call(self.L.ref_vlz_decode, _p(t), len(tokens), dim, n, _p(out))
        return out

    def match_stats(self, codes: np.ndarray, dim: int, window: int = 255):
        c = np.ascontiguousarray(codes, np.int32)
        lit, ref = C.c_uint64(), C.c_uint64()
        self._call(self.L.ref_match_stats, _p(c), dim, c.size // dim if dim else 0, window, C.byref(lit),
                   C.byref(ref))
        return lit.value, ref.value

    def huff_encode(self, codes: np.ndarray) -> bytes:
        c = np.ascontiguousarray(codes, np.int32)
        p, ln = C.c_void_p(), C.c_uint64()
        self._call(self.L.ref_huff_encode, _p(c), c.size, C.byref(p), C.byref(ln))
        return self._take(p, ln.value, np.uint8).tobytes()

    def huff_decode(self, data: bytes) -> np.ndarray:
        t = np.frombuffer(data, np.uint8).copy() if data else np.zeros(0, np.uint8)
        p, n = C.c_void_p(), C.c_uint64()
        self._call(self.L.ref_huff_decode, _p(t), len(data), C.byref(p), C.byref(n))
        return self._take(p, n.value, np.int32)

    def huff_codebook(self, codes: np.ndarray):
        c = np.ascontiguousarray(codes, np.int32)
        k = max(1, len(np.unique(c)))
        syms, lens, cws = np.zeros(k, np.int32), np.zeros(k, np.uint8), np.zeros(k, np.uint32)
        n = C.c_uint32()
        self._call(self.L.ref_huff_codebook, _p(c), c.size, _p(syms), _p(lens), _p(cws), C.byref(n))
        return syms, lens, cws

    def huff_from_histogram(self, sym, cnt):
        s = np.ascontiguousarray(sym, np.int32)
        c = np.ascontiguousarray(cnt, np.uint64)
        os_, ol = np.zeros(len(s), np.int32), np.zeros(len(s), np.uint8)
        self._call(self.L.ref_huff_from_histogram, _p(s), _p(c), len(s), _p(os_), _p(ol))
        return os_, ol

    def pack(self, chunks) -> bytes:
        arrs = [np.frombuffer(c, np.uint8).copy() for c in chunks]
        ptrs = (C.c_void_p * max(len(arrs), 1))(*[a.ctypes.data for a in arrs])
        lens = np.array([len(c) for c in chunks] or [0], np.uint64)
        p, ln = C.c_void_p(), C.c_uint64()
        self._call(self.L.ref_pack, ptrs, _p(lens), len(chunks), C.byref(p), C.byref(ln))
        return self._take(p, ln.value, np.uint8).tobytes()

    def unpack(self, buf: bytes):
        t = np.frombuffer(buf, np.uint8).copy()
        p, pl, k = C.c_void_p(), C.c_void_p(), C.c_uint32()
        self._call(self.L.ref_unpack, _p(t), len(buf), C.byref(p), C.byref(pl), C.byref(k))
        lens = self._take(pl, k.value, np.uint64)
        body = self._take(p, int(lens.sum()), np.uint8).tobytes()
        out, o = [], 0
        for ln in lens:
            out.append(body[o:o + int(ln)])
            o += int(ln)
        return out

    def metadata(self, chunk: bytes) -> bytes:
        t = np.frombuffer(chunk, np.uint8).copy()
        out = np.zeros(25, np.uint8)
        self._call(self.L.ref_metadata, _p(t), len(chunk), _p(out))
        return out.tobytes()

    def gen_table(self, rows, dim, dist=0, mu=0.0, sigma=0.1, lo=0.0, hi=1.0, zipf=0.0, seed=1, table_id=0):
        out = np.zeros(rows * dim, np.float64)
        self._call(self.L.ref_gen_table, table_id, rows, dim, dist, mu, sigma, lo, hi, zipf, seed, _p(out))
        return out.reshape(rows, dim)

    def lookup_indices(self, rows, dim, zipf, seed, batch, stream, dist=0, mu=0.0, sigma=0.1, lo=0.0, hi=1.0):
        out = np.zeros(batch, np.uint32)
        self._call(self.L.ref_lookup_indices, 0, rows, dim, dist, mu, sigma, lo, hi, zipf, seed, batch, stream,
                   _p(out))
        return out

    def mix_seed(self, seed, salt):
        return int(self.L.ref_mix_seed(seed, salt))

    def pattern_counts(self, x: np.ndarray, dim: int, eb: float):
        v = np.ascontiguousarray(x, np.float64)
        o, q = C.c_uint64(), C.c_uint64()
        self._call(self.L.ref_pattern_counts, _p(v), dim, v.size // dim, eb, C.byref(o), C.byref(q))
        return o.value, q.value

    def decay_multiplier(self, it, fn=0, start=1.0, end=0, steps=4):
        return self.L.ref_decay_multiplier(it, fn, start, end, steps)

    def classify(self, survival, global_eb=0.02, alpha=5 / 3, beta=3.0, l_thr=0.70, s_thr=0.95):
        cls, eb = C.c_int(), C.c_double()
        self._call(self.L.ref_classify, survival, global_eb, alpha, beta, l_thr, s_thr, C.byref(cls), C.byref(eb))
        return cls.value, eb.value

    def estimate_speedup(self, ratio, bw, comp, decomp):
        return self.L.ref_estimate_speedup(ratio, bw, comp, decomp)

    def codec_timed(self, batches, ebs, codecs, workers: int, reps: int = 3):
        """encode_chunks+pack then unpack+parallel decode_chunk on `workers` threads;
        returns (best compress s, best decompress s, packed length)."""
        vals = np.concatenate([np.ascontiguousarray(b, np.float64).ravel() for b in batches])
        offs = np.cumsum([0] + [b.size for b in batches[:-1]]).astype(np.uint64)
        dims = np.array([b.shape[1] for b in batches], np.uint32)
        ns = np.array([b.shape[0] for b in batches], np.uint32)
        ebs = np.ascontiguousarray(ebs, np.float64)
        cods = np.ascontiguousarray(codecs, np.uint8)
        cs, ds, pl = C.c_double(), C.c_double(), C.c_uint64()
        self._call(self.L.ref_codec_timed, _p(vals), _p(offs), _p(dims), _p(ns), _p(ebs), _p(cods), len(batches),
                   workers, reps, C.byref(cs), C.byref(ds), C.byref(pl))
        return cs.value, ds.value, pl.value

    @staticmethod
    def _jobs(batches):
        vals = np.concatenate([np.ascontiguousarray(b, np.float64).ravel() for b in batches]) if batches else \
            np.zeros(1, np.float64)
        offs = np.cumsum([0] + [b.size for b in batches[:-1]]).astype(np.uint64)
        dims = np.array([b.shape[1] for b in batches], np.uint32)
        ns = np.array([b.shape[0] for b in batches], np.uint32)
        return vals, offs, dims, ns

    def encode_pack(self, batches, ebs, codecs, workers: int = 1, window: int = 255) -> bytes:
        """pack(encode_chunks(jobs, workers)) (container.hpp:242-256, :304-311)."""
        vals, offs, dims, ns = self._jobs(batches)
        e = np.ascontiguousarray(ebs, np.float64)
        c = np.ascontiguousarray(codecs, np.uint8)
        p, ln = C.c_void_p(), C.c_uint64()
        self._call(self.L.ref_encode_pack, _p(vals), _p(offs), _p(dims), _p(ns), _p(e), _p(c), len(batches), window,
                   workers, C.byref(p), C.byref(ln))
        return self._take(p, ln.value, np.uint8).tobytes()

    def load_preset(self, path: str) -> dict:
        """load_tables + load_policy (config.hpp:184-228) of a preset .cfg file."""
        cap = 4096
        arrs = {k: np.zeros(cap, t) for k, t in [("rows", np.uint32), ("dim", np.uint32), ("dist", np.int32),
                                                  ("mu", np.float64), ("sigma", np.float64), ("lo", np.float64),
                                                  ("hi", np.float64), ("zipf", np.float64), ("seed", np.uint64)]}
        pol = np.zeros(5, np.float64)
        cnt, fn, st, end, steps, batch, ranks = (C.c_uint32(), C.c_int(), C.c_double(), C.c_uint64(), C.c_uint32(),
                                                 C.c_uint32(), C.c_uint32())
        self._call(self.L.ref_load_preset, path.encode(), cap, C.byref(cnt), *[_p(arrs[k]) for k in
                   ("rows", "dim", "dist", "mu", "sigma", "lo", "hi", "zipf", "seed")], _p(pol), C.byref(fn),
                   C.byref(st), C.byref(end), C.byref(steps), C.byref(batch), C.byref(ranks))
        n = cnt.value
        tables = [[int(arrs["rows"][i]), int(arrs["dist"][i]), float(arrs["mu"][i]), float(arrs["sigma"][i]),
                   float(arrs["lo"][i]), float(arrs["hi"][i]), float(arrs["zipf"][i])] for i in range(n)]
        return {"tables": tables, "dims": [int(d) for d in arrs["dim"][:n]],
                "policy": {"global_eb": pol[0], "alpha": pol[1], "beta": pol[2], "large_threshold": pol[3],
                           "small_threshold": pol[4], "decay_fn": fn.value, "decay_start": st.value,
                           "decay_end": end.value, "decay_steps": steps.value},
                "batch": batch.value, "ranks": ranks.value}

    def offline_analysis(self, samples, table_ids, path: str, global_eb=0.02, alpha=5 / 3, beta=3.0,
                         l_thr=0.70, s_thr=0.95, bandwidth=1e-300, window: int = 255) -> None:
        """offline_analysis (policy.hpp:278-302), written with write_profiles (config.hpp:247-271)."""
        vals, offs, dims, ns = self._jobs(samples)
        ids = np.ascontiguousarray(table_ids, np.int32)
        self._call(self.L.ref_offline_analysis, _p(vals), _p(offs), _p(dims), _p(ns), _p(ids), len(samples),
                   global_eb, alpha, beta, l_thr, s_thr, bandwidth, window, path.encode())

    def read_profiles(self, path: str) -> dict:
        """read_profiles (config.hpp:273-303) -> {table_id: {...}}."""
        cap = 4096
        tid = np.zeros(cap, np.int32)
        no, nq = np.zeros(cap, np.uint64), np.zeros(cap, np.uint64)
        surv, eb, rv, rh = (np.zeros(cap, np.float64) for _ in range(4))
        cls, cod = np.zeros(cap, np.int32), np.zeros(cap, np.int32)
        cnt = C.c_uint32()
        self._call(self.L.ref_read_profiles, path.encode(), cap, C.byref(cnt), _p(tid), _p(no), _p(nq), _p(surv),
                   _p(cls), _p(cod), _p(eb), _p(rv), _p(rh))
        return {int(tid[i]): {"n_original": int(no[i]), "n_quantized": int(nq[i]), "survival": float(surv[i]),
                              "cls": int(cls[i]), "codec": int(cod[i]), "eb": float(eb[i]),
                              "ratio_vlz": float(rv[i]), "ratio_huffman": float(rh[i])} for i in range(cnt.value)}

    def format_double(self, v: float) -> str:
        buf = C.create_string_buffer(64)
        self.L.ref_format_double(v, buf, 64)
        return buf.value.decode()
