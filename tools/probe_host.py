"""Host-side cost of one eager encode+decode call pair on the KG workload."""
import time, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2407_04272_b200 import codec as K, workload as W, _lib
preset, T, dim, B, geb = bench.workload_spec(sys.argv[1] if len(sys.argv) > 1 else "kg")
dev = torch.device("cuda", 0)
specs = [W.TableSpec.preset(preset, t, dim) for t in range(T)]
tables = [W.Table(s, dev) for s in specs]
x = torch.stack([tables[t].lookup_batch(B, 1) for t in range(T)])
profiles, cfg = bench.build_profiles(preset, {t: x[t] for t in range(T)}, geb)
jobs = [K.EncodeJob(x[t], profiles[t].eb, profiles[t].codec) for t in range(T)]
r = K.encode_chunks(jobs, K.LAYOUT_PACKED)
table = K.unpack_table(bytes(r.buffer.cpu().numpy().tobytes()))
out = torch.empty(r.total + 256, dtype=torch.uint8, device=dev)
y = torch.empty_like(x)
cj = [j.to_c() for j in jobs]
crefs = []
for t, (o, ln) in enumerate(table):
    c = _lib.ChunkRef(); c.offset, c.length, c.out, c.dim, c.count, c.codec = o, ln, y[t].data_ptr(), dim, B, jobs[t].codec
    crefs.append(c)
ctx = K.Context.default(0)
for _ in range(5):
    ctx.encode_raw(cj, K.LAYOUT_PACKED, out); ctx.decode_raw(out, crefs, K.OUT_F32, False)
torch.cuda.synchronize()
te = td = 0.0
n = 50
for _ in range(n):
    t0 = time.perf_counter(); ctx.encode_raw(cj, K.LAYOUT_PACKED, out); t1 = time.perf_counter()
    ctx.decode_raw(out, crefs, K.OUT_F32, False); t2 = time.perf_counter()
    torch.cuda.synchronize()
    te += t1 - t0; td += t2 - t1
print(f"host enqueue per call: encode {te / n * 1e6:.1f} us, decode {td / n * 1e6:.1f} us")
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
for _ in range(n):
    ctx.encode_raw(cj, K.LAYOUT_PACKED, out); ctx.decode_raw(out, crefs, K.OUT_F32, False)
ev1.record(); torch.cuda.synchronize()
print(f"eager back-to-back step: {ev0.elapsed_time(ev1) / n * 1e3:.1f} us")
