"""Per-codec throughput probe: the workload's tables (profile bounds) with every
chunk forced to one codec, or the profile's codecs ("prof").  Encode and
decode are timed separately (CUDA events via embc_timing_*).

  python tools/probe_codec.py WORKLOAD [prof|raw|vlz|huffman ...] [--tables K] [--batch B]
"""
import argparse
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2407_04272_b200 import _lib  # noqa: E402
from paper_2407_04272_b200 import codec as K  # noqa: E402
from paper_2407_04272_b200 import workload as W  # noqa: E402

NAMES = {"raw": 0, "vlz": 1, "huffman": 2}


def run(name, mode, ntab, batch, reps=10):
    w = W.WORKLOADS[name]
    T = ntab or w["tables"]
    dim, B = w["dim"], batch or w["batch"](1)
    prof = W.workload_profiles(name)
    specs = W.workload_specs(name)[:T]
    ebs = [prof[t].eb for t in range(T)]
    codecs = [prof[t].codec for t in range(T)] if mode == "prof" else [NAMES[mode]] * T
    dev = torch.device("cuda", 0)
    ctx = K.Context.default(0)
    x = torch.empty((T, B, dim), dtype=torch.float32, device=dev)
    for t in range(T):
        x[t] = W.Table(specs[t], dev).lookup_batch(B, W.lookup_stream(0, t, 0, 1))
    jobs = [K.EncodeJob(x[t], ebs[t], codecs[t]) for t in range(T)]
    r = K.encode_chunks(jobs, K.LAYOUT_PACKED)
    table = K.unpack_table(bytes(r.buffer.cpu().numpy().tobytes()))
    cj = [j.to_c() for j in jobs]
    out = torch.empty(int(r.total) + 256, dtype=torch.uint8, device=dev)
    y = torch.empty_like(x)
    crefs = []
    for t, (o, ln) in enumerate(table):
        cr = _lib.ChunkRef()
        cr.offset, cr.length, cr.out, cr.dim, cr.count, cr.codec = o, ln, y[t].data_ptr(), dim, B, codecs[t]
        crefs.append(cr)
    for _ in range(3):
        ctx.encode_raw(cj, K.LAYOUT_PACKED, out)
        ctx.decode_raw(out, crefs, K.OUT_F32, False)
    ctx.sync()
    ctx.timing(True)
    for _ in range(reps):
        ctx.encode_raw(cj, K.LAYOUT_PACKED, out)
        ctx.decode_raw(out, crefs, K.OUT_F32, False)
    ctx.sync()
    tm = ctx.timing_collect()
    ctx.timing(False)
    fb = K.decode_fallbacks(ctx)
    agg = defaultdict(float)
    for n_, ms in tm:
        agg[n_] += ms / reps
    nbytes = x.numel() * 4
    enc = sum(v for k, v in agg.items() if k != "k_dec_main")
    dec = agg.get("k_dec_main", 0.0)
    assert torch.equal(out[:r.total], r.buffer[:r.total])
    err = max((y[t].double() - x[t].double()).abs().max().item() / ebs[t] for t in range(T))
    assert err <= 1.0000001
    ks = " ".join(f"{k}={v * 1e3:.1f}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1]))
    print(f"{name:4s} {mode:7s} T={T} B={B} dim={dim} in={nbytes / 2**20:.1f}MiB CR={nbytes / r.total:6.2f} "
          f"fb={fb} enc {enc * 1e3:8.1f}us {nbytes / enc / 1e6:7.1f}GB/s  dec {dec * 1e3:8.1f}us {nbytes / dec / 1e6:7.1f}GB/s  [{ks}]",
          flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload")
    ap.add_argument("modes", nargs="*", default=["prof", "raw", "vlz", "huffman"])
    ap.add_argument("--tables", type=int, default=0)
    ap.add_argument("--batch", type=int, default=0)
    a = ap.parse_args()
    for m in a.modes:
        run(a.workload, m, a.tables, a.batch)


if __name__ == "__main__":
    main()
