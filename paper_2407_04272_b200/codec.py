"""Python mirror of the reference codec API (namespace ``embc``), backed by the
sm_100a kernels of libembc_cuda.so through the C ABI.

Reference -> this module:
  encode_chunk + serialize_chunk   (container.hpp:119-142, :74-85) -> encode_chunk()
  parse_chunk + decode_chunk       (container.hpp:89-115, :146-181) -> decode_chunk()
  encode_chunks + pack             (container.hpp:304-311, :242-256) -> encode_chunks(), pack_encode()
  unpack                           (container.hpp:258-292)          -> unpack_table()
  quantize / dequantize            (quantizer.hpp:83-102)           -> quantize(), dequantize()
  vlz_encode / vlz_decode          (vlz.hpp:111-158)                -> vlz_encode(), vlz_decode()
  match_stats                      (vlz.hpp:162-168)                -> match_stats()
  huff_encode_codes / huff_decode  (huffman.hpp:228-291)            -> huff_encode(), huff_decode()
  metadata_for + serialize_metadata (container.hpp:196-209)         -> encode_chunks(meta=True)
  detail::pattern_counts           (policy.hpp:167-173)             -> pattern_counts()

Inputs are CUDA tensors (fp32 values, or int32 codes for the codec-stage
entry points).  Errors raise the classes in ``_lib`` with the reference's
exception text.
"""
from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass
from typing import Optional, Sequence

import torch

from . import _lib
from ._lib import (CODEC_HUFFMAN, CODEC_RAW, CODEC_VLZ, LAYOUT_CHUNKS, LAYOUT_PACKED, LAYOUT_PAYLOAD,
                   OUT_F32, OUT_F64, OUT_I32, SRC_F32, SRC_I32)

HEADER_SIZE = 30  # CompressedChunk::kHeaderSize (container.hpp:67)
META_SIZE = 25  # ChunkMetadata::kWireSize (container.hpp:193)
CODEC_NAMES = {CODEC_RAW: "raw", CODEC_VLZ: "vlz", CODEC_HUFFMAN: "huffman"}
CODEC_IDS = {v: k for k, v in CODEC_NAMES.items()}


def _codec_id(c) -> int:
    return CODEC_IDS[c] if isinstance(c, str) else int(c)


def _stream_ptr(stream: Optional[torch.cuda.Stream]) -> Optional[int]:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream or None


class Context:
    """One embc_ctx per (device, host thread): owns scratch + the failure record."""

    _by_device: dict = {}

    def __init__(self, device: int = 0):
        self.device = device
        self._L = _lib.lib()
        h = C.c_void_p()
        with torch.cuda.device(device):
            st = self._L.embc_ctx_create(device, C.byref(h))
        if st != _lib.OK:
            raise _lib.EmbcError(f"embc_ctx_create failed with status {st}", status=st)
        self.handle = h

    @classmethod
    def default(cls, device: Optional[int] = None) -> "Context":
        d = torch.cuda.current_device() if device is None else device
        ctx = cls._by_device.get(d)
        if ctx is None:
            ctx = cls._by_device[d] = cls(d)
        return ctx

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self._L.embc_ctx_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    # -- failures -------------------------------------------------------------
    def last_error(self) -> _lib.EmbcErrorRec:
        rec = _lib.EmbcErrorRec()
        self._L.embc_get_error(self.handle, C.byref(rec))
        return rec

    def check(self, status: int) -> None:
        if status == _lib.OK:
            return
        rec = self.last_error()
        _lib.raise_for(status, rec.message.decode(errors="replace"), rec.reason, rec.job, rec.index)

    def sync(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        self.check(self._L.embc_sync(self.handle, _stream_ptr(stream)))

    def reserve(self, max_jobs: int, max_values: int, max_payload: int = 0) -> None:
        self.check(self._L.embc_reserve(self.handle, max_jobs, max_values, max_payload))

    def reserve_capture(self, nbytes: int) -> None:
        self.check(self._L.embc_reserve_capture(self.handle, nbytes))

    def timing(self, on: bool) -> None:
        self.check(self._L.embc_timing_enable(self.handle, 1 if on else 0))

    def timing_collect(self, stream=None):
        """[(kernel name, ms)] for every launch since timing(True), after a stream sync."""
        names = C.create_string_buffer(1 << 20)
        ms = (C.c_float * 65536)()
        n = self._L.embc_timing_collect(self.handle, _stream_ptr(stream), names, 1 << 20, ms, 65536)
        if n < 0:
            raise _lib.EmbcError("embc_timing_collect failed")
        out = names.raw.split(b"\0")
        return [(out[i].decode(), float(ms[i])) for i in range(n)]

    # -- compression ------------------------------------------------------------
    def encode_raw(self, jobs, layout: int, out: torch.Tensor, offsets=None, lengths=None, meta=None,
                   total=None, stream=None) -> None:
        """embc_encode with prepared ctypes Job array (async)."""
        arr = (_lib.Job * len(jobs))(*jobs)
        st = self._L.embc_encode(self.handle, arr, len(jobs), layout, out.data_ptr() if out is not None else None,
                                 out.numel() if out is not None else 0,
                                 offsets.data_ptr() if offsets is not None else None,
                                 lengths.data_ptr() if lengths is not None else None,
                                 meta.data_ptr() if meta is not None else None,
                                 total.data_ptr() if total is not None else None, _stream_ptr(stream))
        self.check(st)

    def decode_raw(self, buf: torch.Tensor, refs, out_kind: int, payload_only: bool, stream=None) -> None:
        arr = (_lib.ChunkRef * len(refs))(*refs)
        st = self._L.embc_decode(self.handle, buf.data_ptr(), arr, len(refs), out_kind,
                                 1 if payload_only else 0, _stream_ptr(stream))
        self.check(st)

    def decode_dev_raw(self, buf: torch.Tensor, refs, d_off, d_len: torch.Tensor, out_kind: int,
                       payload_only: bool = False, stream=None) -> None:
        """embc_decode_dev: refs carry (base offset, capacity); the received
        relative offsets / lengths are device int64 tensors (async, capturable)."""
        arr = (_lib.ChunkRef * len(refs))(*refs)
        st = self._L.embc_decode_dev(self.handle, buf.data_ptr(), arr, len(refs),
                                     d_off.data_ptr() if d_off is not None else None, d_len.data_ptr(), out_kind,
                                     1 if payload_only else 0, _stream_ptr(stream))
        self.check(st)


@dataclass
class EncodeJob:
    """embc::EncodeJob (container.hpp:295-300): batch is an [n, dim] CUDA tensor."""

    batch: torch.Tensor
    eb: float
    codec: int = CODEC_RAW
    window: int = 255

    def to_c(self) -> _lib.Job:
        b = self.batch
        if b.dim() != 2:
            raise ValueError("batch must be a 2-D [n, dim] tensor")
        if not b.is_cuda:
            raise ValueError("batch must be a CUDA tensor")
        if b.dtype == torch.float32:
            kind = SRC_F32
        elif b.dtype == torch.int32:
            kind = SRC_I32
        else:
            raise ValueError("batch must be float32 values or int32 codes")
        if not b.is_contiguous():
            raise ValueError("batch must be contiguous")
        j = _lib.Job()
        j.src = b.data_ptr() if b.numel() else None
        j.n, j.dim = int(b.shape[0]), int(b.shape[1])
        j.eb = float(self.eb)
        j.window = int(self.window)
        j.codec = _codec_id(self.codec)
        j.src_kind = kind
        return j


@dataclass
class EncodeResult:
    buffer: torch.Tensor  # uint8, device (trimmed to total)
    offsets: torch.Tensor  # int64 (uint64 bits), device
    lengths: torch.Tensor
    meta: Optional[torch.Tensor]  # uint8 [njobs, 25], device
    total: int


def encode_chunks(jobs: Sequence[EncodeJob], layout: int = LAYOUT_CHUNKS, meta: bool = False,
                  ctx: Optional[Context] = None, stream=None) -> EncodeResult:
    """encode_chunks + serialize_chunk/pack on the GPU; synchronises to size the result."""
    ctx = ctx or Context.default()
    cj = [j.to_c() for j in jobs]
    arr = (_lib.Job * len(cj))(*cj)
    bound = int(ctx._L.embc_encode_bound(arr, len(cj), layout))
    dev = jobs[0].batch.device if jobs else torch.device("cuda", ctx.device)
    out = torch.empty(max(bound, 1), dtype=torch.uint8, device=dev)
    n = max(len(cj), 1)
    offs = torch.zeros(n, dtype=torch.int64, device=dev)
    lens = torch.zeros(n, dtype=torch.int64, device=dev)
    tot = torch.zeros(1, dtype=torch.int64, device=dev)
    md = torch.zeros((n, META_SIZE), dtype=torch.uint8, device=dev) if meta else None
    ctx.encode_raw(cj, layout, out, offs, lens, md, tot, stream=stream)
    ctx.sync(stream)
    total = int(tot.item())
    return EncodeResult(out[:total], offs[:len(cj)], lens[:len(cj)], md[:len(cj)] if md is not None else None,
                        total)


def encode_chunk(batch: torch.Tensor, eb: float, codec=CODEC_RAW, window: int = 255,
                 ctx: Optional[Context] = None) -> bytes:
    """serialize_chunk(encode_chunk(batch, eb, codec, VlzConfig{window})) as bytes."""
    r = encode_chunks([EncodeJob(batch, eb, codec, window)], LAYOUT_CHUNKS, ctx=ctx)
    return bytes(r.buffer.cpu().numpy().tobytes())


def pack_encode(jobs: Sequence[EncodeJob], ctx: Optional[Context] = None) -> bytes:
    """pack(encode_chunks(jobs)) bytes (container.hpp:242-256)."""
    r = encode_chunks(jobs, LAYOUT_PACKED, ctx=ctx)
    return bytes(r.buffer.cpu().numpy().tobytes())


def parse_header(chunk: bytes):
    """Host view of the 30-byte chunk header (container.hpp:47-70): codec, eb, dim, count, paylen.
    Used only to size outputs; the device re-validates every field."""
    if len(chunk) < HEADER_SIZE:
        return None
    codec, = struct.unpack_from("<B", chunk, 5)
    eb, dim, count, paylen = struct.unpack_from("<dIIQ", chunk, 6)
    return codec, eb, dim, count, paylen


def _as_device_bytes(data, device) -> torch.Tensor:
    if isinstance(data, torch.Tensor):
        return data if data.is_cuda else data.to(device)
    t = torch.frombuffer(bytearray(data), dtype=torch.uint8) if len(data) else torch.zeros(1, dtype=torch.uint8)
    return t.to(device)


_OUT_DTYPE = {OUT_F32: torch.float32, OUT_F64: torch.float64, OUT_I32: torch.int32}


def decode_chunks(buf, refs: Sequence[tuple], out_kind: int = OUT_F32, payload_only: bool = False,
                  ctx: Optional[Context] = None, stream=None, device=None):
    """Decode chunks at (offset, length, codec, dim, count[, eb]) of buf; returns [count, dim] tensors."""
    ctx = ctx or Context.default()
    device = device or torch.device("cuda", ctx.device)
    dbuf = _as_device_bytes(buf, device)
    outs, crefs = [], []
    for r in refs:
        off, length, codec, dim, count = r[:5]
        eb = r[5] if len(r) > 5 else 0.0
        o = torch.empty((count, dim), dtype=_OUT_DTYPE[out_kind], device=device)
        cr = _lib.ChunkRef()
        cr.offset, cr.length = off, length
        cr.out = o.data_ptr() if o.numel() else None
        cr.dim, cr.count, cr.eb, cr.codec = dim, count, eb, codec
        outs.append(o)
        crefs.append(cr)
    ctx.decode_raw(dbuf, crefs, out_kind, payload_only, stream=stream)
    ctx.sync(stream)
    return outs


def decode_chunk(chunk, out_kind: int = OUT_F32, ctx: Optional[Context] = None) -> torch.Tensor:
    """decode_chunk(parse_chunk(bytes)) -> [count, dim] tensor (float32 = float(reference double))."""
    raw = bytes(chunk.cpu().numpy().tobytes()) if isinstance(chunk, torch.Tensor) else bytes(chunk)
    h = parse_header(raw)
    if h is None or h[0] > 2:
        codec, dim, count = CODEC_RAW, 0, 0
    else:
        codec, _, dim, count, _ = h
    return decode_chunks(raw, [(0, len(raw), codec, dim, count)], out_kind, ctx=ctx)[0]


# ---- codec-stage entry points on int32 codes ----------------------------------

def vlz_encode(codes: torch.Tensor, window: int = 255, ctx: Optional[Context] = None) -> bytes:
    """vlz_encode(QuantizedBatch, VlzConfig{window}).tokens (vlz.hpp:111-125)."""
    r = encode_chunks([EncodeJob(codes, 0.01, CODEC_VLZ, window)], LAYOUT_PAYLOAD, ctx=ctx)
    return bytes(r.buffer.cpu().numpy().tobytes())


def vlz_decode(tokens: bytes, dim: int, count: int, ctx: Optional[Context] = None) -> torch.Tensor:
    """vlz_decode(VlzStream{dim, count, tokens}) codes (vlz.hpp:129-158)."""
    return decode_chunks(tokens, [(0, len(tokens), CODEC_VLZ, dim, count, 0.01)], OUT_I32, payload_only=True,
                         ctx=ctx)[0]


def huff_encode(codes: torch.Tensor, ctx: Optional[Context] = None) -> bytes:
    """huff_encode_codes(codes).bytes (huffman.hpp:228-248)."""
    c2 = codes.reshape(-1, 1) if codes.dim() == 1 else codes
    r = encode_chunks([EncodeJob(c2, 0.01, CODEC_HUFFMAN)], LAYOUT_PAYLOAD, ctx=ctx)
    return bytes(r.buffer.cpu().numpy().tobytes())


def huff_decode(stream_bytes: bytes, count: int, ctx: Optional[Context] = None) -> torch.Tensor:
    """huff_decode(HuffStream) (huffman.hpp:254-291), expecting `count` symbols."""
    return decode_chunks(stream_bytes, [(0, len(stream_bytes), CODEC_HUFFMAN, 1, count, 0.01)], OUT_I32,
                         payload_only=True, ctx=ctx)[0].reshape(-1)


def quantize(x: torch.Tensor, eb: float, ctx: Optional[Context] = None) -> torch.Tensor:
    """quantize() (quantizer.hpp:83-91) of a float32 or float64 CUDA tensor."""
    ctx = ctx or Context.default()
    x = x.contiguous()
    out = torch.empty(x.shape, dtype=torch.int32, device=x.device)
    st = ctx._L.embc_quantize(ctx.handle, x.data_ptr() if x.numel() else None,
                              1 if x.dtype == torch.float64 else 0, x.numel(), float(eb),
                              out.data_ptr() if x.numel() else None, _stream_ptr(None))
    ctx.check(st)
    ctx.sync()
    return out


def dequantize(codes: torch.Tensor, eb: float, dtype=torch.float64, ctx: Optional[Context] = None) -> torch.Tensor:
    """dequantize() (quantizer.hpp:95-102) to float64 (reference bits) or float32."""
    ctx = ctx or Context.default()
    codes = codes.contiguous()
    out = torch.empty(codes.shape, dtype=dtype, device=codes.device)
    st = ctx._L.embc_dequantize(ctx.handle, codes.data_ptr() if codes.numel() else None, codes.numel(),
                                float(eb), out.data_ptr() if codes.numel() else None,
                                1 if dtype == torch.float64 else 0, _stream_ptr(None))
    ctx.check(st)
    ctx.sync()
    return out


def match_stats(codes: torch.Tensor, window: int = 255, ctx: Optional[Context] = None):
    """match_stats() (vlz.hpp:162-168) -> (literal_count, reference_count)."""
    ctx = ctx or Context.default()
    codes = codes.contiguous()
    lit, ref = C.c_uint64(), C.c_uint64()
    st = ctx._L.embc_match_stats(ctx.handle, codes.data_ptr() if codes.numel() else None, int(codes.shape[1]),
                                 int(codes.shape[0]), int(window), C.byref(lit), C.byref(ref),
                                 _stream_ptr(None))
    ctx.check(st)
    return lit.value, ref.value


def pattern_counts(x: torch.Tensor, eb: float, ctx: Optional[Context] = None):
    """detail::pattern_counts (policy.hpp:167-173) -> (original, quantized) distinct rows."""
    ctx = ctx or Context.default()
    x = x.contiguous()
    o, q = C.c_uint64(), C.c_uint64()
    st = ctx._L.embc_pattern_counts(ctx.handle, x.data_ptr() if x.numel() else None, int(x.shape[1]),
                                    int(x.shape[0]), float(eb), C.byref(o), C.byref(q), _stream_ptr(None))
    ctx.check(st)
    return o.value, q.value


def unpack_table(buf: bytes):
    """unpack()'s offset-table validation (container.hpp:258-284) through the C
    ABI (embc_unpack) -> [(offset, length)]; chunk bodies decode on the GPU."""
    L = _lib.lib()
    raw = (C.c_uint8 * max(len(buf), 1)).from_buffer_copy(bytes(buf) or b"\0")
    cap = len(buf) // 16 + 1
    offs, lens = (C.c_uint64 * cap)(), (C.c_uint64 * cap)()
    n, err = C.c_uint32(), _lib.EmbcErrorRec()
    st = L.embc_unpack(raw, len(buf), offs, lens, cap, C.byref(n), C.byref(err))
    if st != _lib.OK:
        _lib.raise_for(st, err.message.decode(errors="replace"), err.reason, err.job, err.index)
    return [(offs[i], lens[i]) for i in range(n.value)]


def decode_packed(buf: bytes, out_kind: int = OUT_F32, ctx: Optional[Context] = None):
    """unpack() + decode_chunk() of every chunk of a PackedSendBuffer, decoded on the GPU."""
    table = unpack_table(buf)
    refs = []
    for (o, ln) in table:
        h = parse_header(buf[o:o + ln])
        codec, dim, count = (CODEC_RAW, 0, 0) if h is None or h[0] > 2 else (h[0], h[2], h[3])
        refs.append((o, ln, codec, dim, count))
    return decode_chunks(buf, refs, out_kind, ctx=ctx)


def decode_fallbacks(ctx: Optional[Context] = None) -> int:
    """Chunks of the last decode that needed the exact sequential walker (0 for
    valid streams inside the parallel envelope)."""
    ctx = ctx or Context.default()
    n = C.c_uint32()
    ctx.check(ctx._L.embc_decode_fallbacks(ctx.handle, C.byref(n)))
    return n.value
