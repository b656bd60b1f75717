"""Per-kernel timing probe (CUDA events via embc_timing_*) for the BASELINE
workload shapes.  Usage: python tools/probe.py [kg|tb|cfg1] [codec-override]"""
import os
import sys
import time
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2407_04272_b200 import codec as K  # noqa: E402
from paper_2407_04272_b200 import workload as W  # noqa: E402


def jobs_for(name, codec_override=None, it=0):
    if name == "kg":
        specs = W.preset_tables(W.KAGGLE_TABLES, 26, 16)
        batch, ebs = 2048, [0.03] * 26
    elif name == "tb":  # rank 0 of 8: tables 0, 8, 16, 24 x 8 destinations
        specs = [TS for TS in W.preset_tables(W.TERABYTE_TABLES, 26, 64)][0:26:8]
        batch, ebs = 8192, [0.03] * 4
    else:
        specs = [W.TableSpec(100000, 64, 0, 0.0, 0.1, 0, 1, 1.1, 20260810)]
        batch, ebs = 2048, [1e-3]
    tabs = [W.Table(s, "cuda") for s in specs]
    jobs = []
    dsts = 8 if name == "tb" else 1
    for t, tab in enumerate(tabs):
        for d in range(dsts):
            c = codec_override if codec_override is not None else (1 if t % 2 == 0 else 2)
            jobs.append(K.EncodeJob(tab.lookup_batch(batch, W.lookup_stream(it, t, d, dsts)), ebs[t], c))
    return jobs


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "kg"
    ov = int(sys.argv[2]) if len(sys.argv) > 2 else None
    ctx = K.Context.default(0)
    jobs = jobs_for(name, ov)
    nbytes = sum(j.batch.numel() * 4 for j in jobs)
    r = K.encode_chunks(jobs, K.LAYOUT_PACKED)
    buf = r.buffer
    table = K.unpack_table(bytes(buf.cpu().numpy().tobytes()))
    refs = [(o, ln, j.codec, j.batch.shape[1], j.batch.shape[0]) for (o, ln), j in zip(table, jobs)]
    print(f"{name}: {len(jobs)} chunks, {nbytes / 2**20:.2f} MiB in, {r.total / 2**20:.3f} MiB packed, CR {nbytes / r.total:.2f}")
    cj = [j.to_c() for j in jobs]
    out = torch.empty(int(r.total) + 64, dtype=torch.uint8, device="cuda")
    outs = [torch.empty_like(j.batch) for j in jobs]
    crefs = []
    for (o, ln, c, dim, n), ot in zip(refs, outs):
        cr = K._lib.ChunkRef()
        cr.offset, cr.length, cr.out, cr.dim, cr.count, cr.codec = o, ln, ot.data_ptr(), dim, n, c
        crefs.append(cr)
    for _ in range(3):
        ctx.encode_raw(cj, K.LAYOUT_PACKED, out)
        ctx.decode_raw(buf, crefs, K.OUT_F32, False)
    ctx.sync()
    reps = 20
    ctx.timing(True)
    t0 = time.perf_counter()
    for _ in range(reps):
        ctx.encode_raw(cj, K.LAYOUT_PACKED, out)
        ctx.decode_raw(buf, crefs, K.OUT_F32, False)
    ctx.sync()
    t1 = time.perf_counter()
    tm = ctx.timing_collect()
    ctx.timing(False)
    agg = defaultdict(float)
    for n_, ms in tm:
        agg[n_] += ms / reps
    tot = sum(agg.values())
    for n_, ms in sorted(agg.items(), key=lambda kv: -kv[1]):
        print(f"  {n_:18s} {ms * 1e3:9.1f} us  {100 * ms / tot:5.1f}%")
    print(f"  kernel sum {tot * 1e3:.1f} us/step; wall {1e6 * (t1 - t0) / reps:.1f} us/step; "
          f"codec GB/s (kernel sum) {nbytes / (tot * 1e-3) / 1e9:.1f}")
    for o, j in zip(outs, jobs):
        assert (o.double() - j.batch.double()).abs().max().item() <= j.eb * 1.0000001 + 1e-7


if __name__ == "__main__":
    main()
