"""GPU: compress + decompress captured in CUDA graphs (descriptors uploaded
once at capture time into the device mirror of the capture arena) replay
byte-identical to eager calls, in any order."""
import pytest
import torch

from paper_2407_04272_b200 import _lib
from paper_2407_04272_b200 import codec as K
from paper_2407_04272_b200 import workload as W

pytestmark = pytest.mark.gpu


def _sets(dev, nsets, T=7, dim=16, B=1024):
    specs = W.preset_tables(W.KAGGLE_TABLES, T, dim)
    tables = [W.Table(s, dev) for s in specs]
    out = []
    for it in range(nsets):
        x = torch.stack([tables[t].lookup_batch(B, W.lookup_stream(it, t, 0, 1)) for t in range(T)])
        jobs = [K.EncodeJob(x[t], 0.01 + 0.02 * (t % 2), t % 3) for t in range(T)]
        r = K.encode_chunks(jobs, K.LAYOUT_PACKED)
        want = r.buffer[: r.total].clone()
        table = K.unpack_table(bytes(want.cpu().numpy().tobytes()))
        out.append({"x": x, "jobs": jobs, "cj": [j.to_c() for j in jobs], "want": want, "table": table,
                    "buf": torch.zeros(r.total + 256, dtype=torch.uint8, device=dev),
                    "y": torch.empty_like(x)})
    return out


def _crefs(s, dim, B):
    refs = []
    for t, (o, ln) in enumerate(s["table"]):
        cr = _lib.ChunkRef()
        cr.offset, cr.length, cr.out, cr.dim, cr.count, cr.codec = o, ln, s["y"][t].data_ptr(), dim, B, s["jobs"][t].codec
        refs.append(cr)
    return refs


def test_graph_replay_matches_eager():
    dev = torch.device("cuda", 0)
    ctx = K.Context(0)  # own context: own scratch and capture arena
    ctx.reserve_capture(8 << 20)
    sets = _sets(dev, 3)
    T, B, dim = sets[0]["x"].shape
    for s in sets:  # eager: sizes scratch, checks the buffer path against encode_chunks
        s["crefs"] = _crefs(s, dim, B)
        ctx.encode_raw(s["cj"], K.LAYOUT_PACKED, s["buf"])
        ctx.decode_raw(s["buf"], s["crefs"], K.OUT_F32, False)
    ctx.sync()
    eager_y = [s["y"].clone() for s in sets]
    for s in sets:
        assert torch.equal(s["buf"][: s["want"].numel()], s["want"])
    cap = torch.cuda.Stream()
    graphs = []
    for s in sets:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap):
            ctx.encode_raw(s["cj"], K.LAYOUT_PACKED, s["buf"], stream=cap)
            ctx.decode_raw(s["buf"], s["crefs"], K.OUT_F32, False, stream=cap)
        graphs.append(g)
    torch.cuda.synchronize()
    for order in ([2, 0, 1], [1, 1, 2, 0]):
        for k in order:
            sets[k]["buf"].zero_()
            sets[k]["y"].fill_(float("nan"))
            graphs[k].replay()
            torch.cuda.synchronize()
            ctx.sync()
            assert torch.equal(sets[k]["buf"][: sets[k]["want"].numel()], sets[k]["want"]), k
            assert torch.equal(sets[k]["y"], eager_y[k]), k
