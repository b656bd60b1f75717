"""Graph replay time of the Kaggle-shaped step split into its calls: encode-only,
decode-only and both graphs, plus an empty-kernel graph, to size the gaps
between launches.  usage: python tools/probe_graph.py [kg|tb]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2407_04272_b200 import _lib
from paper_2407_04272_b200 import codec as K
from paper_2407_04272_b200 import workload as W

wl = sys.argv[1] if len(sys.argv) > 1 else "kg"
dev = torch.device("cuda", 0)
preset, T, dim, B, geb = bench.workload_spec(wl)
specs = [W.TableSpec.preset(preset, t, dim) for t in range(T)]
tables = [W.Table(s, dev) for s in specs]
samples = {t: tables[t].lookup_batch(B, 0) for t in range(T)}
profiles, _ = bench.build_profiles(preset, samples, geb)
ctx = K.Context.default(0)
ctx.reserve_capture(64 << 20)
P = 8
sets = []
for it in range(P):
    x = torch.stack([tables[t].lookup_batch(B, W.lookup_stream(it, t, 0, 1)) for t in range(T)])
    jobs = [K.EncodeJob(x[t], profiles[t].eb, profiles[t].codec) for t in range(T)]
    r = K.encode_chunks(jobs, K.LAYOUT_PACKED)
    table = K.unpack_table(bytes(r.buffer.cpu().numpy().tobytes()))
    y = torch.empty_like(x)
    refs = []
    for t, (o, ln) in enumerate(table):
        cr = _lib.ChunkRef()
        cr.offset, cr.length, cr.out, cr.dim, cr.count, cr.codec = o, ln, y[t].data_ptr(), dim, B, jobs[t].codec
        refs.append(cr)
    sets.append({"x": x, "y": y, "cj": [j.to_c() for j in jobs], "refs": refs,
                 "out": torch.empty(r.total + 256, dtype=torch.uint8, device=dev)})
for s in sets:
    ctx.encode_raw(s["cj"], K.LAYOUT_PACKED, s["out"])
    ctx.decode_raw(s["out"], s["refs"], K.OUT_F32, False)
ctx.sync()
cap = torch.cuda.Stream()
def graphs(enc, dec):
    gs = []
    for s in sets:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap):
            if enc:
                ctx.encode_raw(s["cj"], K.LAYOUT_PACKED, s["out"], stream=cap)
            if dec:
                ctx.decode_raw(s["out"], s["refs"], K.OUT_F32, False, stream=cap)
        gs.append(g)
    return gs
def timeit(gs, reps=200):
    for k in range(10):
        gs[k % len(gs)].replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(reps):
        gs[k % len(gs)].replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3
both, enc, dec = graphs(True, True), graphs(True, False), graphs(False, True)
print(f"{wl}: both {timeit(both):.1f} us, encode only {timeit(enc):.1f} us, decode only {timeit(dec):.1f} us")
g = torch.cuda.CUDAGraph()
z = torch.zeros(1, device=dev)
with torch.cuda.graph(g, stream=cap):
    z.add_(1)
print(f"empty graph (one tiny kernel): {timeit([g]):.1f} us")
