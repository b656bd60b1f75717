"""Encode-only kernel times (CUDA events via embc_timing_*) for a workload with
the profile's codecs; used to A/B library variants (EMBC_LIB) whose decode
may be deliberately broken.   python tools/probe_enc.py WORKLOAD [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2407_04272_b200 import codec as K  # noqa: E402
from paper_2407_04272_b200 import workload as W  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "kg"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    w = W.WORKLOADS[name]
    T, dim, B = w["tables"], w["dim"], w["batch"](1)
    prof = W.workload_profiles(name)
    specs = W.workload_specs(name)
    dev = torch.device("cuda", 0)
    ctx = K.Context.default(0)
    xs = []
    for it in range(8):
        x = torch.empty((T, B, dim), dtype=torch.float32, device=dev)
        for t in range(T):
            x[t] = W.Table(specs[t], dev).lookup_batch(B, W.lookup_stream(it, t, 0, 1))
        xs.append(x)
    cjs = [[K.EncodeJob(x[t], prof[t].eb, prof[t].codec).to_c() for t in range(T)] for x in xs]
    out = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
    for k in range(20):
        ctx.encode_raw(cjs[k % 8], K.LAYOUT_PACKED, out)
    torch.cuda.synchronize()
    ctx.timing(True)
    for k in range(reps):
        ctx.encode_raw(cjs[k % 8], K.LAYOUT_PACKED, out)
    tm = ctx.timing_collect()
    ctx.timing(False)
    per = {}
    for n, v in tm:
        per.setdefault(n, []).append(v)
    print(name, {n: round(1000 * sum(v) / len(v), 2) for n, v in per.items()}, "us per launch")


if __name__ == "__main__":
    main()
