"""CPU, world_size 2 (gloo): the compressed all-to-all exchange logic
(metadata round, variable-size payload all-to-all, decode placement, backward
direction, accounting) with the oracle as the codec backend, checked against
locally computed expectations and against the reference Simulator's
per-iteration accounting and delivered-value digest (commsim.hpp:146-163)."""
import os
import socket
import struct

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class OracleCodec:
    """Test-only backend: CPU restatement of the codec (oracle/embc_oracle.c)."""

    def __init__(self, out_dtype=torch.float32):
        from oracle import Oracle
        self.o = Oracle()
        self.out_dtype = out_dtype

    def encode(self, jobs, out=None):
        chunks = [self.o.encode_chunk(j.batch.double().numpy().ravel(), j.batch.shape[1], j.eb, j.codec, j.window)
                  for j in jobs]
        buf = torch.frombuffer(bytearray(b"".join(chunks) or b"\0"), dtype=torch.uint8)
        lens = torch.tensor([len(c) for c in chunks], dtype=torch.int64)
        meta = torch.frombuffer(bytearray(b"".join(self.o.metadata(c) for c in chunks) or b"\0" * 25),
                                dtype=torch.uint8).view(-1, 25)[:len(chunks)]
        return buf, lens, meta

    def decode(self, buf, refs, outs):
        raw = bytes(buf.numpy().tobytes())
        for (off, length, codec, dim, count), o in zip(refs, outs):
            vals = self.o.decode_chunk(raw[off:off + length])
            o.copy_(torch.from_numpy(vals).to(o.dtype))

    def check(self):
        pass


def fnv1a(data: bytes, h: int = 0xCBF29CE484222325) -> int:
    for b in data:
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, mode):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2407_04272_b200 import codec as K
        from paper_2407_04272_b200 import exchange as X
        from paper_2407_04272_b200 import policy as P
        from paper_2407_04272_b200 import workload as W
        if mode == "general":
            T, dim, B = 5, 8, 64
            specs = W.preset_tables(W.KAGGLE_TABLES, T, dim)
            tabs = {t: W.gen_table(specs[t]) for t in range(T)}
            profiles = {t: P.TableProfile(t, codec=t % 3, eb=0.01 + 0.01 * (t % 2)) for t in range(T)}
            cfg = P.PolicyConfig(global_eb=0.01, decay=P.DecayConfig("stepwise", 2.0, 4, 2))
            ex = X.CompressedAllToAll(T, dim, B, profiles, cfg, backend=OracleCodec(), device=torch.device("cpu"))
            res = {"fwd_ok": True, "bwd_ok": True}
            for it in range(3):
                look = {}
                for t in ex.owned(rank):
                    look[t] = torch.cat([torch.from_numpy(tabs[t][W.lookup_indices(specs[t], B,
                                                                                  W.lookup_stream(it, t, d, world))])
                                         for d in range(world)])
                out = ex.forward(it, look)
                # expected: owner's slice for this rank, through the oracle codec at eb_at
                from oracle import Oracle
                o = Oracle()
                for t in range(T):
                    x = tabs[t][W.lookup_indices(specs[t], B, W.lookup_stream(it, t, rank, world))]
                    eb = P.eb_at(t, it, profiles, cfg)
                    want = o.decode_chunk(o.encode_chunk(x.astype(np.float64).ravel(), dim, eb, profiles[t].codec))
                    if not np.array_equal(out[t].numpy(), want.astype(np.float32)):
                        res["fwd_ok"] = False
                st = ex.stats
                own = ex.owned(rank)
                res.setdefault("unc", []).append(st.uncompressed_bytes)
                res.setdefault("meta", []).append(st.metadata_bytes)
                exp_unc = len(own) * (world - 1) * B * dim * 4
                if st.uncompressed_bytes != exp_unc or st.metadata_bytes != 25 * len(own) * (world - 1):
                    res["fwd_ok"] = False
                # backward: gradients of every table -> owner
                grads = {t: torch.full((B, dim), 0.001 * (rank + 1) * (t + 1), dtype=torch.float32) for t in range(T)}
                gout = ex.backward(it, grads)
                for t in own:
                    for s in range(world):
                        g = np.full(B * dim, 0.001 * (s + 1) * (t + 1), np.float32).astype(np.float64)
                        eb = P.eb_at(t, it, profiles, cfg)
                        want = o.decode_chunk(o.encode_chunk(g, dim, eb, profiles[t].codec))
                        if not np.array_equal(gout[t][s * B:(s + 1) * B].numpy(), want.astype(np.float32)):
                            res["bwd_ok"] = False
                base = ex.uncompressed(look)
                for t in range(T):
                    x = tabs[t][W.lookup_indices(specs[t], B, W.lookup_stream(it, t, rank, world))]
                    if not np.array_equal(base[t].numpy(), x):
                        res["fwd_ok"] = False
            q.put((rank, res))
        elif mode == "pipelined":  # table groups overlapped == one exchange, byte for byte
            T, dim, B = 7, 8, 48
            specs = W.preset_tables(W.KAGGLE_TABLES, T, dim)
            tabs = {t: W.gen_table(specs[t]) for t in range(T)}
            profiles = {t: P.TableProfile(t, codec=t % 3, eb=0.01 + 0.01 * (t % 2)) for t in range(T)}
            cfg = P.PolicyConfig(global_eb=0.01)
            res = {"ok": True}
            ex1 = X.CompressedAllToAll(T, dim, B, profiles, cfg, backend=OracleCodec(), device=torch.device("cpu"))
            for G in (2, 3, 8):
                exg = X.CompressedAllToAll(T, dim, B, profiles, cfg, backend=OracleCodec(), device=torch.device("cpu"),
                                           groups=G)
                for it in range(2):
                    look = {t: torch.cat([torch.from_numpy(tabs[t][W.lookup_indices(specs[t], B,
                                                                                   W.lookup_stream(it, t, d, world))])
                                          for d in range(world)]) for t in ex1.owned(rank)}
                    a1 = ex1.forward(it, look)
                    s1 = ex1.stats
                    ag = exg.forward(it, look)
                    sg = exg.stats
                    for t in range(T):
                        if not torch.equal(a1[t], ag[t]):
                            res["ok"] = False
                    if (s1.payload_bytes, s1.metadata_bytes, s1.uncompressed_bytes) != \
                            (sg.payload_bytes, sg.metadata_bytes, sg.uncompressed_bytes):
                        res["ok"] = False
                    # backward through the same pipeline: gradients of every table -> owner
                    grads = {t: (a1[t] * 0.5 + 0.01 * (t + 1)).contiguous() for t in range(T)}
                    b1 = ex1.backward(it, grads)
                    bg = exg.backward(it, grads)
                    for t in ex1.owned(rank):
                        if not torch.equal(b1[t], bg[t]):
                            res["ok"] = False
                    if ex1.stats.payload_bytes != exg.stats.payload_bytes:
                        res["ok"] = False
            q.put((rank, res))
        elif mode == "few_tables":  # T < R: a rank that owns no table still receives
            T, dim, B = 2, 4, 32
            specs = W.preset_tables(W.KAGGLE_TABLES, T, dim)
            tabs = {t: W.gen_table(specs[t]) for t in range(T)}
            profiles = {t: P.TableProfile(t, codec=1 + t % 2, eb=0.02) for t in range(T)}
            cfg = P.PolicyConfig(global_eb=0.02)
            from oracle import Oracle
            o = Oracle()
            res = {"ok": True}
            for G in (1, 2):
                ex = X.CompressedAllToAll(T, dim, B, profiles, cfg, backend=OracleCodec(), device=torch.device("cpu"),
                                          groups=G)
                look = {t: torch.cat([torch.from_numpy(tabs[t][W.lookup_indices(specs[t], B,
                                                                               W.lookup_stream(0, t, d, world))])
                                      for d in range(world)]) for t in ex.owned(rank)}
                out = ex.forward(0, look)
                for t in range(T):
                    x = tabs[t][W.lookup_indices(specs[t], B, W.lookup_stream(0, t, rank, world))]
                    want = o.decode_chunk(o.encode_chunk(x.astype(np.float64).ravel(), dim, 0.02, profiles[t].codec))
                    if not np.array_equal(out[t].numpy(), want.astype(np.float32)):
                        res["ok"] = False
                if not ex.owned(rank) and ex.stats.payload_bytes != 0:
                    res["ok"] = False
                grads = {t: torch.full((B, dim), 0.01 * (t + 1), dtype=torch.float32) for t in range(T)}
                gout = ex.backward(0, grads)
                if sorted(gout) != ex.owned(rank):
                    res["ok"] = False
            q.put((rank, res))
        else:  # simulator parity: one table per rank, reference seeding
            from oracle import Ref
            ref_specs = [(64, 0, 0.0, 0.05, 0, 1, 1.1), (256, 1, 0.0, 0.1, -0.2, 0.3, 0.6)]
            dim, B, seed, iters = 8, 128, 7, 4
            T = world
            specs = [W.TableSpec.preset(ref_specs, t, dim, run_seed=seed) for t in range(T)]
            tabs = {t: W.gen_table(specs[t]) for t in range(T)}
            codecs, ebs = [1, 2], [0.02, 0.01]
            profiles = {t: P.TableProfile(t, codec=codecs[t], eb=ebs[t]) for t in range(T)}
            cfg = P.PolicyConfig(global_eb=0.02, decay=P.DecayConfig("stepwise", 2.0, decay_end=4, step_count=3))
            ex = X.CompressedAllToAll(T, dim, B, profiles, cfg, backend=OracleCodec(torch.float64),
                                      device=torch.device("cpu"), out_dtype=torch.float64)
            digests, pay, unc, meta = [], [], [], []
            for it in range(iters):
                look = {t: torch.cat([torch.from_numpy(tabs[t][W.lookup_indices(specs[t], B,
                                                                                W.lookup_stream(it, t, d, world))])
                                      for d in range(world)]) for t in ex.owned(rank)}
                # delivered values in source order, as doubles (commsim.hpp:409-426)
                ex_out = {}
                ex.device = torch.device("cpu")
                out = ex.forward(it, look)
                h = 0xCBF29CE484222325
                for s in range(world):
                    h = fnv1a(out[s].to(torch.float64).numpy().tobytes(), h)
                digests.append(h)
                pay.append(ex.stats.payload_bytes)
                unc.append(ex.stats.uncompressed_bytes)
                meta.append(ex.stats.metadata_bytes)
                del ex_out
            q.put((rank, {"digests": digests, "pay": pay, "unc": unc, "meta": meta, "specs": ref_specs,
                          "dim": dim, "B": B, "seed": seed, "iters": iters, "codecs": codecs, "ebs": ebs}))
    finally:
        dist.destroy_process_group()


def _run(mode, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, mode)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    return out


def test_exchange_forward_backward_gloo():
    out = _run("general")
    for r in (0, 1):
        assert out[r]["fwd_ok"], r
        assert out[r]["bwd_ok"], r


def test_exchange_pipelined_groups_gloo():
    """groups > 1 (compression / transfer / decompression overlapped per table
    group) delivers the same values and accounting as one exchange, forward
    and backward."""
    out = _run("pipelined")
    for r in (0, 1):
        assert out[r]["ok"], r


def test_exchange_rank_without_tables_gloo():
    """T < R (3 ranks, 2 tables): the rank that owns no table sends nothing and
    still decodes what its peers send, with one exchange or table groups."""
    out = _run("few_tables", world=3)
    for r in range(3):
        assert out[r]["ok"], r


def test_exchange_matches_reference_simulator(ref):
    """One table per rank: per-iteration payload/metadata/uncompressed bytes and
    the delivered-value digest equal the reference Simulator's."""
    out = _run("sim")
    a = out[0]
    R, iters = 2, a["iters"]
    # the reference's per-iteration digest folds the per-rank digests in rank order
    import ctypes as C
    n = iters
    u64 = np.zeros(n, np.uint64)
    arrs = {k: np.zeros(n, np.uint64) for k in ("unc", "pay", "meta", "dig")}
    maxerr = np.zeros(n, np.float64)
    rep = C.c_uint64()
    specs = a["specs"]
    rows = np.array([s[0] for s in specs], np.uint32)
    dims = np.array([a["dim"]] * len(specs), np.uint32)
    dist_ = np.array([s[1] for s in specs], np.int32)
    mu = np.array([s[2] for s in specs], np.float64)
    sig = np.array([s[3] for s in specs], np.float64)
    lo = np.array([s[4] for s in specs], np.float64)
    hi = np.array([s[5] for s in specs], np.float64)
    zf = np.array([s[6] for s in specs], np.float64)
    pc = np.array(a["codecs"], np.uint8)
    pe = np.array(a["ebs"], np.float64)
    err = C.create_string_buffer(512)
    p = lambda x: x.ctypes.data_as(C.c_void_p)  # noqa: E731
    rc = ref.L.ref_simulate(R, a["B"], iters, a["seed"], 1, 0.02, 2.0, 4, 3, p(rows), p(dims), p(dist_), p(mu),
                            p(sig), p(lo), p(hi), p(zf), len(specs), p(pc), p(pe), p(arrs["unc"]), p(arrs["pay"]),
                            p(arrs["meta"]), p(maxerr), p(arrs["dig"]), C.byref(rep), err, 512)
    assert rc == 0, err.value
    del u64
    for it in range(iters):
        assert sum(out[r]["unc"][it] for r in range(R)) == arrs["unc"][it]
        assert sum(out[r]["pay"][it] for r in range(R)) == arrs["pay"][it]
        assert sum(out[r]["meta"][it] for r in range(R)) == arrs["meta"][it]
        h = 0xCBF29CE484222325
        for r in range(R):
            h = fnv1a(struct.pack("<Q", out[r]["digests"][it]), h)
        assert h == int(arrs["dig"][it]), it
