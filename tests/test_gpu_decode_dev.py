"""GPU: embc_decode_dev -- the decode planned on the device from received
lengths (the receiving side of a peer-to-peer exchange) -- against the
host-planned embc_decode on the same chunks (bit-identical fp64 and fp32
values), inside a CUDA graph whose replays see different lengths, and the
capacity check."""
import numpy as np
import pytest
import torch

from paper_2407_04272_b200 import _lib
from paper_2407_04272_b200 import codec as K
from paper_2407_04272_b200 import workload as W

pytestmark = pytest.mark.gpu


def _jobs(name, it, T=None, codec=None):
    w = W.WORKLOADS[name]
    prof = W.workload_profiles(name)
    specs = W.workload_specs(name)
    T = T or w["tables"]
    dim, B = w["dim"], w["batch"](1)
    dev = torch.device("cuda", 0)
    x = torch.empty((T, B, dim), dtype=torch.float32, device=dev)
    for t in range(T):
        x[t] = W.Table(specs[t], dev).lookup_batch(B, W.lookup_stream(it, t, 0, 1))
    codecs = [codec if codec is not None else prof[t].codec for t in range(T)]
    return x, [K.EncodeJob(x[t], prof[t].eb, codecs[t]) for t in range(T)]


def _bounds(jobs):
    out = []
    for j in jobs:
        arr = (_lib.Job * 1)(j.to_c())
        out.append(int(_lib.lib().embc_encode_bound(arr, 1, K.LAYOUT_CHUNKS)))
    return out


def _refs(jobs, outs, offsets, lengths):
    refs = []
    for j, o, off, ln in zip(jobs, outs, offsets, lengths):
        r = _lib.ChunkRef()
        r.offset, r.length, r.out = off, ln, o.data_ptr()
        r.dim, r.count, r.codec = j.batch.shape[1], j.batch.shape[0], j.codec
        refs.append(r)
    return refs


@pytest.mark.parametrize("name,T,codec", [("kg", None, None), ("tb", 8, None), ("tb", 6, 2), ("kg", 12, 0),
                                          ("cfg1", None, 1)])
def test_decode_dev_equals_host_planned(ctx, name, T, codec):
    x, jobs = _jobs(name, 0, T, codec)
    n = len(jobs)
    caps = _bounds(jobs)
    base = np.concatenate([[0], np.cumsum(caps)[:-1]]).astype(np.uint64)
    # every chunk in its own slot of capacity `cap` (as a sender writes into a peer window)
    buf = torch.zeros(int(sum(caps)) + 64, dtype=torch.uint8, device="cuda")
    d_len = torch.empty(n, dtype=torch.int64, device="cuda")
    d_rel = torch.zeros(n, dtype=torch.int64, device="cuda")
    for k, j in enumerate(jobs):
        r = K.encode_chunks([j], K.LAYOUT_CHUNKS)
        L = int(r.total)
        buf[int(base[k]):int(base[k]) + L] = r.buffer[:L]
        d_len[k] = L
    lens = d_len.cpu().numpy()
    for kind, dt in ((K.OUT_F64, torch.float64), (K.OUT_F32, torch.float32)):
        want = [torch.empty(j.batch.shape, dtype=dt, device="cuda") for j in jobs]
        got = [torch.full(j.batch.shape, float("nan"), dtype=dt, device="cuda") for j in jobs]
        ctx.decode_raw(buf, _refs(jobs, want, base, lens), kind, False)
        ctx.decode_dev_raw(buf, _refs(jobs, got, base, caps), d_rel, d_len, kind)
        ctx.sync()
        for k in range(n):
            assert torch.equal(got[k].view(torch.int64 if dt == torch.float64 else torch.int32),
                               want[k].view(torch.int64 if dt == torch.float64 else torch.int32)), (name, k, kind)


def test_decode_dev_in_cuda_graph(ctx):
    """Encode (chunk placement on the device) + device-planned decode captured
    once; replays with other iterations' inputs (other lengths) decode exactly
    what the eager host-planned path decodes."""
    x, jobs = _jobs("kg", 0)
    n = len(jobs)
    caps = _bounds(jobs)
    cj = [j.to_c() for j in jobs]
    buf = torch.zeros(int(sum(caps)) + 64, dtype=torch.uint8, device="cuda")
    d_off = torch.empty(n, dtype=torch.int64, device="cuda")
    d_len = torch.empty(n, dtype=torch.int64, device="cuda")
    y = torch.empty_like(x)
    refs = _refs(jobs, list(y), [0] * n, [int(sum(caps))] * n)  # one slot: the whole buffer
    ctx.reserve_capture(64 << 20)
    s = torch.cuda.Stream()
    # warm up (scratch sized) then capture
    with torch.cuda.stream(s):
        ctx.encode_raw(cj, K.LAYOUT_CHUNKS, buf, d_off, d_len, stream=s)
        ctx.decode_dev_raw(buf, refs, d_off, d_len, K.OUT_F32, stream=s)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        ctx.encode_raw(cj, K.LAYOUT_CHUNKS, buf, d_off, d_len, stream=s)
        ctx.decode_dev_raw(buf, refs, d_off, d_len, K.OUT_F32, stream=s)
    for it in (1, 2, 3):
        x2, jobs2 = _jobs("kg", it)
        x.copy_(x2)
        g.replay()
        torch.cuda.synchronize()
        ctx.sync()
        r = K.encode_chunks(jobs2, K.LAYOUT_CHUNKS)
        want = torch.empty_like(x)
        table_off = d_off.cpu().tolist()
        table_len = d_len.cpu().tolist()
        assert table_len == [int(v) for v in r.lengths.cpu().tolist()]
        ctx.decode_raw(r.buffer, _refs(jobs2, list(want), r.offsets.cpu().tolist(), table_len), K.OUT_F32, False)
        ctx.sync()
        assert torch.equal(y.view(torch.int32), want.view(torch.int32)), it
        del table_off


def test_decode_dev_length_over_capacity(ctx):
    x, jobs = _jobs("kg", 0, 4)
    r = K.encode_chunks(jobs, K.LAYOUT_CHUNKS)
    offs = r.offsets.to(torch.int64)
    lens = r.lengths.to(torch.int64)
    outs = [torch.empty_like(j.batch) for j in jobs]
    caps = lens.cpu().tolist()
    caps[2] -= 1  # chunk 2 arrives one byte longer than its slot
    ctx.decode_dev_raw(r.buffer, _refs(jobs, outs, [0] * 4, caps), offs, lens, K.OUT_F32)
    with pytest.raises(_lib.CodecFormatError) as e:
        ctx.sync()
    assert e.value.reason == 31 and e.value.job == 2
