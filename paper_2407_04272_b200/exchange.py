"""Compressed hybrid-parallel embedding all-to-all over torch.distributed
(NCCL over NVLink on the B200 box; gloo in the CPU tests).

Replaces the reference's in-process simulation (Simulator::rank_body,
commsim.hpp:286-435) with a real exchange.  Layout:
table t is owned by rank t mod R; in the forward pass the owner's lookup
output [R*B, dim] is split into R slices of [B, dim], one per destination rank;
every (destination, table) slice is one chunk.  Each rank:

  stage 1  compresses its chunks in (destination, table) order into one send
           buffer (one encode launch sequence, deterministic offsets);
  stage 2  exchanges the 25-byte ChunkMetadata records (commsim.hpp:321-330,
           the reference's two-round protocol) with a fixed-size
           all-to-all, then reads the byte counts to the host (the one
           synchronisation point per exchange);
  stage 3  exchanges the variable-size payloads with all_to_all_single;
  stage 4  decodes every received chunk straight into the consumer tensors,
           verifying the metadata against each chunk header
           (commsim.hpp:371-376).

The backward pass sends each rank's [B, dim] gradient slice of every table to
its owner through the same stages (a capability the reference only
describes).  `uncompressed()` is the C3 baseline: raw fp32
all-to-all of the same tensors.

The codec backend is pluggable so the exchange logic can be tested on CPU:
the product backend is GpuCodec (libembc_cuda.so); tests inject a CPU checker.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import torch
import torch.distributed as dist

from . import codec as K
from . import policy as P

META = K.META_SIZE


class GpuCodec:
    """The product backend: sm_100a kernels through the C ABI.  Encode and
    decode own separate contexts (scratch + staging), so a pipelined exchange
    can run them concurrently on different streams."""

    def __init__(self, ctx: Optional[K.Context] = None, dec_ctx: Optional[K.Context] = None):
        self.ctx = ctx or K.Context.default()
        self.dec_ctx = dec_ctx or K.Context(self.ctx.device)

    def encode(self, jobs: Sequence[K.EncodeJob], out: Optional[torch.Tensor] = None, stream=None):
        """-> (device uint8 buffer, device lengths int64 [njobs], device metadata uint8 [njobs, 25])."""
        cj = [j.to_c() for j in jobs]
        arr = (K._lib.Job * len(cj))(*cj)
        bound = int(self.ctx._L.embc_encode_bound(arr, len(cj), K.LAYOUT_CHUNKS))
        dev = jobs[0].batch.device if jobs else torch.device("cuda", self.ctx.device)
        if out is None or out.numel() < bound:
            out = torch.empty(max(bound, 1), dtype=torch.uint8, device=dev)
        lens = torch.empty(len(cj), dtype=torch.int64, device=dev)
        meta = torch.empty((len(cj), META), dtype=torch.uint8, device=dev)
        self.ctx.encode_raw(cj, K.LAYOUT_CHUNKS, out, None, lens, meta, None, stream=stream)
        return out, lens, meta

    def decode(self, buf: torch.Tensor, refs: Sequence[tuple], outs: Sequence[torch.Tensor], stream=None) -> None:
        crefs = []
        for (off, length, codec, dim, count), o in zip(refs, outs):
            r = K._lib.ChunkRef()
            r.offset, r.length, r.out = off, length, o.data_ptr() if o.numel() else None
            r.dim, r.count, r.codec = dim, count, codec
            crefs.append(r)
        if crefs:
            kind = K.OUT_F64 if outs[0].dtype == torch.float64 else K.OUT_F32
            self.dec_ctx.decode_raw(buf, crefs, kind, False, stream=stream)

    def check(self) -> None:
        self.ctx.sync()
        self.dec_ctx.sync()


@dataclass
class ExchangeStats:
    """Per-rank accounting with the reference's definitions (commsim.hpp:68-83,
    :322-353): bytes sent to other ranks only; plus the codec's totals (own
    rank included) for throughput accounting."""
    uncompressed_bytes: int = 0
    payload_bytes: int = 0
    metadata_bytes: int = 0
    times_ms: Dict[str, float] = field(default_factory=dict)
    sent_values: int = 0
    sent_bytes: int = 0
    recv_values: int = 0
    recv_bytes: int = 0

    @property
    def wire_bytes(self) -> int:
        return self.payload_bytes + self.metadata_bytes

    @property
    def ratio(self) -> float:
        return self.uncompressed_bytes / self.payload_bytes if self.payload_bytes else 1.0


def _parse_meta(rec: bytes):
    """parse_metadata (container.hpp:211-221)."""
    clen, codec = struct.unpack_from("<QB", rec, 0)
    eb, dim, count = struct.unpack_from("<dII", rec, 9)
    return clen, codec, eb, dim, count


class CompressedAllToAll:
    def __init__(self, ntables: int, dim: int, batch: int, profiles: Dict[int, P.TableProfile],
                 cfg: P.PolicyConfig, backend=None, group=None, device=None, window: int = 255,
                 grad_profiles: Optional[Dict[int, P.TableProfile]] = None,
                 grad_cfg: Optional[P.PolicyConfig] = None, timing: bool = False,
                 out_dtype: torch.dtype = torch.float32, groups: int = 1):
        self.group = group
        self.R = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.T, self.dim, self.B = ntables, dim, batch
        self.profiles, self.cfg = profiles, cfg
        self.grad_profiles = grad_profiles if grad_profiles is not None else profiles
        self.grad_cfg = grad_cfg if grad_cfg is not None else cfg
        self.backend = backend or GpuCodec()
        self.device = device or (torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available()
                                 else torch.device("cpu"))
        self.window = window
        self.timing = timing and self.device.type == "cuda"
        self.out_dtype = out_dtype  # float64 reproduces the reference's delivered doubles bit for bit
        self.stats = ExchangeStats()
        self._send_buf: Optional[torch.Tensor] = None
        # > 1: the exchange runs as a pipeline of table groups: group g+1
        # compresses while group g is on the wire and group g-1 decompresses
        self.groups = max(1, groups)
        cuda = self.device.type == "cuda"
        self._s_enc = torch.cuda.Stream(self.device) if cuda and self.groups > 1 else None
        self._s_dec = torch.cuda.Stream(self.device) if cuda and self.groups > 1 else None

    def owner(self, t: int) -> int:
        return t % self.R

    def owned(self, r: int) -> List[int]:
        return [t for t in range(self.T) if t % self.R == r]

    def _codec(self, profiles, t: int) -> int:
        return profiles[t].codec if t in profiles else K.CODEC_RAW

    # -- the four stages, shared by forward and backward ----------------------------
    def _exchange(self, jobs: List[K.EncodeJob], job_dst: List[int], recv_plan: List[List[tuple]],
                  outs: List[List[torch.Tensor]]) -> ExchangeStats:
        """jobs are in (destination, table) order; recv_plan[src] lists the
        (count, dim) of the chunks src sends here, in its job order; outs[src]
        are the tensors they decode into."""
        R = self.R
        st = ExchangeStats()
        ev = {}

        def mark(name):
            if self.timing:
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                ev[name] = e

        mark("start")
        buf, lens, meta = self.backend.encode(jobs, self._send_buf)
        self._send_buf = buf
        mark("compressed")
        # stage 2: metadata round (fixed 25 B per chunk)
        send_cnt = [sum(1 for d in job_dst if d == r) for r in range(R)]
        recv_cnt = [len(recv_plan[s]) for s in range(R)]
        meta_recv = torch.empty((sum(recv_cnt), META), dtype=torch.uint8, device=meta.device)
        if R > 1:
            dist.all_to_all_single(meta_recv.view(-1), meta.view(-1), [c * META for c in recv_cnt],
                                   [c * META for c in send_cnt], group=self.group)
        else:
            meta_recv.copy_(meta)
        mark("metadata")
        # the host needs the byte counts: one device -> host read per exchange
        host = torch.cat([lens.view(-1).to(torch.int64), meta_recv.view(-1).to(torch.int64)]).cpu()
        lens_h = host[:len(jobs)].tolist()
        meta_h = bytes(host[len(jobs):].to(torch.uint8).numpy().tobytes())
        send_bytes = [0] * R
        for l, d in zip(lens_h, job_dst):
            send_bytes[d] += l
        recs = [_parse_meta(meta_h[i * META:(i + 1) * META]) for i in range(sum(recv_cnt))]
        recv_bytes = [0] * R
        k = 0
        for s in range(R):
            for _ in range(recv_cnt[s]):
                recv_bytes[s] += recs[k][0]
                k += 1
        total_send = sum(send_bytes)
        recv = torch.empty(max(sum(recv_bytes), 1), dtype=torch.uint8, device=buf.device)
        if R > 1:
            dist.all_to_all_single(recv[:sum(recv_bytes)], buf[:total_send], recv_bytes, send_bytes,
                                   group=self.group)
        else:
            recv[:total_send].copy_(buf[:total_send])
        mark("payload")
        # stage 4: decode into the consumer tensors; headers are checked
        # against the metadata records on the device
        refs, dst_tensors = [], []
        off, k = 0, 0
        for s in range(R):
            for j, (count, dim) in enumerate(recv_plan[s]):
                clen, codec, _eb, mdim, mcount = recs[k]
                refs.append((off, clen, codec, mdim, mcount))
                dst_tensors.append(outs[s][j])
                if (mdim, mcount) != (dim, count):
                    from ._lib import CodecFormatError
                    raise CodecFormatError(f"rank {self.rank} decompress stage (from rank {s}): metadata from rank "
                                           f"{s} disagrees with its chunk", status=2, reason=32)
                off += clen
                k += 1
        self.backend.decode(recv, refs, dst_tensors)
        mark("decompressed")
        self.backend.check()
        # accounting (reference definitions: d != src only)
        for l, d, j in zip(lens_h, job_dst, jobs):
            st.sent_values += j.batch.numel()
            st.sent_bytes += l
            if d != self.rank:
                st.payload_bytes += l
                st.metadata_bytes += META
                st.uncompressed_bytes += j.batch.numel() * 4
        for r in refs:
            st.recv_values += r[3] * r[4]
            st.recv_bytes += r[1]
        if self.timing:
            names = list(ev)
            for a, b in zip(names, names[1:]):
                st.times_ms[b] = ev[a].elapsed_time(ev[b])
            st.times_ms["total"] = ev[names[0]].elapsed_time(ev[names[-1]])
        self.stats = st
        return st

    def _exchange_pipelined(self, jobs_by: List[List[K.EncodeJob]], dst_by: List[List[int]],
                            plan_by: List[List[List[tuple]]], outs_by: List[List[List[torch.Tensor]]]) -> ExchangeStats:
        """The same four stages per table group, overlapped: every group's
        compression is queued on the encode stream up front; each group's
        metadata and payload rounds go out as soon as its compression is done,
        and its decompression runs on the decode stream while the next group
        is on the wire.  Byte-for-byte the same chunks as one big exchange."""
        import contextlib
        cuda = self._s_enc is not None
        cur = torch.cuda.current_stream(self.device) if cuda else None
        enc_ctx = (lambda: torch.cuda.stream(self._s_enc)) if cuda else contextlib.nullcontext
        dec_ctx = (lambda: torch.cuda.stream(self._s_dec)) if cuda else contextlib.nullcontext
        st = ExchangeStats()
        t0 = t1 = None
        if self.timing:
            t0 = torch.cuda.Event(enable_timing=True)
            t0.record(cur)
        if cuda:
            self._s_enc.wait_stream(cur)  # the inputs were produced on the caller's stream
        encoded = []
        for jobs in jobs_by:
            if not jobs:
                encoded.append(None)
                continue
            with enc_ctx():
                if cuda:
                    buf, lens, meta = self.backend.encode(jobs, None, stream=self._s_enc)
                else:
                    buf, lens, meta = self.backend.encode(jobs, None)
                ev = None
                if cuda:
                    ev = torch.cuda.Event()
                    ev.record(self._s_enc)
            encoded.append((buf, lens, meta, ev))
        R = self.R
        for g, jobs in enumerate(jobs_by):
            recv_plan, outs, job_dst = plan_by[g], outs_by[g], dst_by[g]
            send_cnt = [sum(1 for d in job_dst if d == r) for r in range(R)]
            recv_cnt = [len(recv_plan[s]) for s in range(R)]
            if encoded[g] is None:
                buf = torch.zeros(1, dtype=torch.uint8, device=self.device)
                lens = torch.zeros(0, dtype=torch.int64, device=self.device)
                meta = torch.zeros((0, META), dtype=torch.uint8, device=self.device)
            else:
                buf, lens, meta, ev = encoded[g]
                if ev is not None:
                    cur.wait_event(ev)
            meta_recv = torch.empty((sum(recv_cnt), META), dtype=torch.uint8, device=self.device)
            if R > 1:
                dist.all_to_all_single(meta_recv.view(-1), meta.reshape(-1), [c * META for c in recv_cnt],
                                       [c * META for c in send_cnt], group=self.group)
            else:
                meta_recv.copy_(meta)
            host = torch.cat([lens.view(-1), meta_recv.view(-1).to(torch.int64)]).cpu()
            lens_h = host[:len(jobs)].tolist()
            meta_h = bytes(host[len(jobs):].to(torch.uint8).numpy().tobytes())
            send_bytes = [0] * R
            for l, d in zip(lens_h, job_dst):
                send_bytes[d] += l
            recs = [_parse_meta(meta_h[i * META:(i + 1) * META]) for i in range(sum(recv_cnt))]
            recv_bytes = [0] * R
            k = 0
            for src in range(R):
                for _ in range(recv_cnt[src]):
                    recv_bytes[src] += recs[k][0]
                    k += 1
            total_send = sum(send_bytes)
            recv = torch.empty(max(sum(recv_bytes), 1), dtype=torch.uint8, device=self.device)
            if R > 1:
                dist.all_to_all_single(recv[:sum(recv_bytes)], buf[:total_send], recv_bytes, send_bytes,
                                       group=self.group)
            else:
                recv[:total_send].copy_(buf[:total_send])
            refs, dst_tensors = [], []
            off, k = 0, 0
            for src in range(R):
                for j, (count, dim) in enumerate(recv_plan[src]):
                    clen, codec, _eb, mdim, mcount = recs[k]
                    refs.append((off, clen, codec, mdim, mcount))
                    dst_tensors.append(outs[src][j])
                    if (mdim, mcount) != (dim, count):
                        from ._lib import CodecFormatError
                        raise CodecFormatError(f"rank {self.rank} decompress stage (from rank {src}): metadata from "
                                               f"rank {src} disagrees with its chunk", status=2, reason=32)
                    off += clen
                    k += 1
            if cuda:
                self._s_dec.wait_stream(cur)
                with dec_ctx():
                    self.backend.decode(recv, refs, dst_tensors, stream=self._s_dec)
                    recv.record_stream(self._s_dec)
            else:
                self.backend.decode(recv, refs, dst_tensors)
            for l, d, j in zip(lens_h, job_dst, jobs):
                st.sent_values += j.batch.numel()
                st.sent_bytes += l
                if d != self.rank:
                    st.payload_bytes += l
                    st.metadata_bytes += META
                    st.uncompressed_bytes += j.batch.numel() * 4
            for r in refs:
                st.recv_values += r[3] * r[4]
                st.recv_bytes += r[1]
        if cuda:
            cur.wait_stream(self._s_dec)  # outputs are ready on the caller's stream
        if self.timing:
            t1 = torch.cuda.Event(enable_timing=True)
            t1.record(cur)
            t1.synchronize()
            st.times_ms["total"] = t0.elapsed_time(t1)
        self.backend.check()
        self.stats = st
        return st

    def forward(self, iteration: int, lookups: Dict[int, torch.Tensor],
                out: Optional[Dict[int, torch.Tensor]] = None) -> Dict[int, torch.Tensor]:
        """lookups[t] for owned t: [R*B, dim] with rows d*B..(d+1)*B destined to
        rank d.  Returns {t: [B, dim]} for every table (rank's data-parallel
        slice), decoded into `out` when given (contiguous [B, dim] per table)."""
        R, B = self.R, self.B
        own = self.owned(self.rank)
        jobs, job_dst = [], []
        for d in range(R):
            for t in own:
                eb = P.eb_at(t, iteration, self.profiles, self.cfg)
                jobs.append(K.EncodeJob(lookups[t][d * B:(d + 1) * B], eb, self._codec(self.profiles, t),
                                        self.window))
                job_dst.append(d)
        if out is None:
            out = {t: torch.empty((B, self.dim), dtype=self.out_dtype, device=self.device) for t in range(self.T)}
        if self.groups > 1:  # group k = the k-th run of every rank's owned tables
            jobs_by, dst_by, plan_by, outs_by = [], [], [], []
            G = min(self.groups, max(len(self.owned(r)) for r in range(R)))  # identical on every rank
            mine = [self._split_of(len(own), G, k) for k in range(G)]
            for k in range(G):
                jg, dg = [], []
                for d in range(R):
                    for i in mine[k]:
                        t = own[i]
                        eb = P.eb_at(t, iteration, self.profiles, self.cfg)
                        jg.append(K.EncodeJob(lookups[t][d * B:(d + 1) * B], eb, self._codec(self.profiles, t),
                                              self.window))
                        dg.append(d)
                plan, og = [], []
                for src in range(R):
                    theirs = self.owned(src)
                    part = self._split_of(len(theirs), G, k)
                    plan.append([(B, self.dim) for _ in part])
                    og.append([out[theirs[i]] for i in part])
                jobs_by.append(jg)
                dst_by.append(dg)
                plan_by.append(plan)
                outs_by.append(og)
            self._exchange_pipelined(jobs_by, dst_by, plan_by, outs_by)
            return out
        recv_plan = [[(B, self.dim) for _ in self.owned(s)] for s in range(R)]
        outs = [[out[t] for t in self.owned(s)] for s in range(R)]
        self._exchange(jobs, job_dst, recv_plan, outs)
        return out

    def _split_of(self, n: int, ngroups: int, k: int) -> List[int]:
        """Positions of group k when n items are cut into ngroups runs (every
        rank uses the same group count so the rounds line up)."""
        return list(range(k * n // ngroups, (k + 1) * n // ngroups))

    def backward(self, iteration: int, grads: Dict[int, torch.Tensor]) -> Dict[int, torch.Tensor]:
        """grads[t] for every table: [B, dim] local gradient slice.  Returns
        {t: [R*B, dim]} for owned tables (rows s*B.. from rank s).  With
        groups > 1 the same pipeline as forward, over the destinations' owned
        tables."""
        R, B = self.R, self.B
        jobs, job_dst = [], []
        for d in range(R):
            for t in self.owned(d):
                eb = P.eb_at(t, iteration, self.grad_profiles, self.grad_cfg)
                jobs.append(K.EncodeJob(grads[t], eb, self._codec(self.grad_profiles, t), self.window))
                job_dst.append(d)
        own = self.owned(self.rank)
        out = {t: torch.empty((R * B, self.dim), dtype=self.out_dtype, device=self.device) for t in own}
        if self.groups > 1:  # group k = the k-th run of every destination's owned tables
            G = min(self.groups, max(len(self.owned(r)) for r in range(R)))  # identical on every rank
            mine = [self._split_of(len(own), G, k) for k in range(G)]
            jobs_by, dst_by, plan_by, outs_by = [], [], [], []
            for k in range(G):
                jg, dg = [], []
                for d in range(R):
                    theirs = self.owned(d)
                    for i in self._split_of(len(theirs), G, k):
                        t = theirs[i]
                        eb = P.eb_at(t, iteration, self.grad_profiles, self.grad_cfg)
                        jg.append(K.EncodeJob(grads[t], eb, self._codec(self.grad_profiles, t), self.window))
                        dg.append(d)
                jobs_by.append(jg)
                dst_by.append(dg)
                plan_by.append([[(B, self.dim) for _ in mine[k]] for s in range(R)])
                outs_by.append([[out[own[i]][s * B:(s + 1) * B] for i in mine[k]] for s in range(R)])
            self._exchange_pipelined(jobs_by, dst_by, plan_by, outs_by)
            return out
        recv_plan = [[(B, self.dim) for _ in own] for s in range(R)]
        outs = [[out[t][s * B:(s + 1) * B] for t in own] for s in range(R)]
        self._exchange(jobs, job_dst, recv_plan, outs)
        return out

    def uncompressed(self, lookups: Dict[int, torch.Tensor]) -> Dict[int, torch.Tensor]:
        """C3 baseline: the same forward exchange as raw fp32 all_to_all_single."""
        R, B, D = self.R, self.B, self.dim
        own = self.owned(self.rank)
        send = torch.cat([lookups[t][d * B:(d + 1) * B] for d in range(R) for t in own]) if own else \
            torch.zeros((0, D), device=self.device)
        recv_counts = [len(self.owned(s)) * B * D for s in range(R)]
        recv = torch.empty(sum(recv_counts), dtype=torch.float32, device=self.device)
        if R > 1:
            dist.all_to_all_single(recv, send.reshape(-1), recv_counts, [len(own) * B * D] * R, group=self.group)
        else:
            recv.copy_(send.reshape(-1))
        out, off = {}, 0
        for s in range(R):
            for t in self.owned(s):
                out[t] = recv[off:off + B * D].view(B, D)
                off += B * D
        return out

    def uncompressed_backward(self, grads: Dict[int, torch.Tensor]) -> Dict[int, torch.Tensor]:
        """C3 baseline of the backward direction: every table's [B, dim]
        gradient slice to its owner as raw fp32 all_to_all_single."""
        R, B, D = self.R, self.B, self.dim
        own = self.owned(self.rank)
        parts = [grads[t] for d in range(R) for t in self.owned(d)]
        send = torch.cat(parts) if parts else torch.zeros((0, D), device=self.device)
        send_counts = [len(self.owned(d)) * B * D for d in range(R)]
        recv = torch.empty(len(own) * R * B * D, dtype=torch.float32, device=self.device)
        if R > 1:
            dist.all_to_all_single(recv, send.reshape(-1), [len(own) * B * D] * R, send_counts, group=self.group)
        else:
            recv.copy_(send.reshape(-1))
        out = {t: torch.empty((R * B, D), dtype=torch.float32, device=self.device) for t in own}
        off = 0
        for s in range(R):
            for t in own:
                out[t][s * B:(s + 1) * B] = recv[off:off + B * D].view(B, D)
                off += B * D
        return out


class NcclExchange:
    """The product exchange on GPUs: embc_exchange_* (exchange.cpp, C++ over
    NCCL grouped send/recv, codec through the C ABI on encode / decode streams),
    with the same interface and semantics as CompressedAllToAll.  One instance
    per process; its NCCL communicator spans the ranks of `group` (the unique id
    travels over torch.distributed)."""

    def __init__(self, ntables: int, dim: int, batch: int, profiles: Dict[int, P.TableProfile],
                 cfg: P.PolicyConfig, group=None, device=None, window: int = 255,
                 grad_profiles: Optional[Dict[int, P.TableProfile]] = None,
                 grad_cfg: Optional[P.PolicyConfig] = None, groups: int = 1, p2p: bool = False):
        """p2p: the peer-to-peer transport (embc_exchange_set_mode 1): chunks
        written straight into the destination's IPC-shared window, flags
        instead of the metadata round, no host synchronisation."""
        import ctypes as C
        from . import _lib
        self._C, self._lib = C, _lib
        self.L = _lib.lib()
        self.group = group
        self.R = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.T, self.dim, self.B = ntables, dim, batch
        self.profiles, self.cfg = profiles, cfg
        self.grad_profiles = grad_profiles if grad_profiles is not None else profiles
        self.grad_cfg = grad_cfg if grad_cfg is not None else cfg
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.window = window
        self.stats = ExchangeStats()
        uid = (C.c_uint8 * 128)()
        if self.rank == 0:
            st = self.L.embc_exchange_unique_id(uid)
            if st != _lib.OK:
                raise _lib.EmbcError(f"embc_exchange_unique_id failed with status {st}", status=st)
        if self.R > 1:
            box = [bytes(uid)]
            dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                       group=group)
            C.memmove(uid, box[0], 128)
        h = C.c_void_p()
        st = self.L.embc_exchange_create(self.device.index or 0, self.rank, self.R, uid, max(1, groups), C.byref(h))
        if st != _lib.OK:
            raise _lib.EmbcError(f"embc_exchange_create failed with status {st}", status=st)
        self.handle = h
        self.p2p = p2p
        if p2p:
            self._check(self.L.embc_exchange_set_mode(h, 1))

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self.L.embc_exchange_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    def owner(self, t: int) -> int:
        return t % self.R

    def owned(self, r: int) -> List[int]:
        return [t for t in range(self.T) if t % self.R == r]

    def _check(self, st: int) -> None:
        if st == self._lib.OK:
            return
        rec = self._lib.EmbcErrorRec()
        self.L.embc_exchange_get_error(self.handle, self._C.byref(rec))
        self._lib.raise_for(st, rec.message.decode(errors="replace"), rec.reason, rec.job, rec.index)

    def _ptrs(self, tensors: Dict[int, torch.Tensor]):
        C = self._C
        arr = (C.c_void_p * self.T)()
        for t, v in tensors.items():
            if not (v.is_cuda and v.dtype == torch.float32 and v.is_contiguous()):
                raise ValueError("exchange tensors must be contiguous float32 CUDA tensors")
            arr[t] = v.data_ptr()
        return arr

    def _policy(self, iteration: int, profiles, cfg):
        C = self._C
        ebs = (C.c_double * self.T)(*[P.eb_at(t, iteration, profiles, cfg) for t in range(self.T)])
        codecs = (C.c_uint8 * self.T)(*[profiles[t].codec if t in profiles else K.CODEC_RAW for t in range(self.T)])
        return ebs, codecs

    def _stats(self, s) -> ExchangeStats:
        return ExchangeStats(s.uncompressed_bytes, s.payload_bytes, s.metadata_bytes, {}, s.sent_values, s.sent_bytes,
                             s.recv_values, s.recv_bytes)

    def forward(self, iteration: int, lookups: Dict[int, torch.Tensor],
                out: Optional[Dict[int, torch.Tensor]] = None, stats: bool = True) -> Dict[int, torch.Tensor]:
        """lookups[t] for owned t: [R*B, dim].  Returns {t: [B, dim]} for every
        table, decoded into `out` when given."""
        if out is None:
            out = {t: torch.empty((self.B, self.dim), dtype=torch.float32, device=self.device) for t in range(self.T)}
        ebs, codecs = self._policy(iteration, self.profiles, self.cfg)
        st = self._lib.ExchangeStats()
        # p2p without stats: asynchronous and graph-capturable (failures at sync())
        sp = self._C.byref(st) if (stats or not self.p2p) else None
        self._check(self.L.embc_exchange_fwd(self.handle, self.T, self.dim, self.B, self._ptrs(lookups), ebs, codecs,
                                             self.window, self._ptrs(out), sp,
                                             torch.cuda.current_stream(self.device).cuda_stream))
        if sp is not None:
            self.stats = self._stats(st)
        return out

    def sync(self) -> None:
        """Waits for the exchange; raises a codec failure or a silent peer."""
        self._check(self.L.embc_exchange_sync(self.handle))

    def reserve_capture(self, nbytes: int) -> None:
        """Descriptor staging for CUDA-graph capture of the exchange's codec calls."""
        self._check(self.L.embc_exchange_reserve_capture(self.handle, nbytes))

    def backward(self, iteration: int, grads: Dict[int, torch.Tensor], stats: bool = True) -> Dict[int, torch.Tensor]:
        """grads[t] for every table: [B, dim].  Returns {t: [R*B, dim]} for owned tables."""
        own = self.owned(self.rank)
        out = {t: torch.empty((self.R * self.B, self.dim), dtype=torch.float32, device=self.device) for t in own}
        ebs, codecs = self._policy(iteration, self.grad_profiles, self.grad_cfg)
        st = self._lib.ExchangeStats()
        sp = self._C.byref(st) if (stats or not self.p2p) else None
        self._check(self.L.embc_exchange_bwd(self.handle, self.T, self.dim, self.B, self._ptrs(grads), ebs, codecs,
                                             self.window, self._ptrs(out), sp,
                                             torch.cuda.current_stream(self.device).cuda_stream))
        if sp is not None:
            self.stats = self._stats(st)
        return out

    def uncompressed(self, lookups: Dict[int, torch.Tensor]) -> Dict[int, torch.Tensor]:
        out = {t: torch.empty((self.B, self.dim), dtype=torch.float32, device=self.device) for t in range(self.T)}
        self._check(self.L.embc_exchange_baseline_fwd(self.handle, self.T, self.dim, self.B, self._ptrs(lookups),
                                                      self._ptrs(out),
                                                      torch.cuda.current_stream(self.device).cuda_stream))
        return out

    def uncompressed_backward(self, grads: Dict[int, torch.Tensor]) -> Dict[int, torch.Tensor]:
        own = self.owned(self.rank)
        out = {t: torch.empty((self.R * self.B, self.dim), dtype=torch.float32, device=self.device) for t in own}
        self._check(self.L.embc_exchange_baseline_bwd(self.handle, self.T, self.dim, self.B, self._ptrs(grads),
                                                      self._ptrs(out),
                                                      torch.cuda.current_stream(self.device).cuda_stream))
        return out

    def timing(self, on: bool) -> None:
        self._check(self.L.embc_exchange_timing_enable(self.handle, 1 if on else 0))

    def timing_collect(self):
        """[(kernel name, ms)] of the codec launches since timing(True)."""
        C = self._C
        names = C.create_string_buffer(1 << 20)
        ms = (C.c_float * 65536)()
        n = self.L.embc_exchange_timing_collect(self.handle, names, 1 << 20, ms, 65536)
        if n < 0:
            raise self._lib.EmbcError("embc_exchange_timing_collect failed")
        out = names.raw.split(b"\0")
        return [(out[i].decode(), float(ms[i])) for i in range(n)]
