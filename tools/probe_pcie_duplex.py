"""PCIe floor of the e2e pipeline: H2D and D2H of one Kaggle-shaped step
(26 x [2048, 16] fp32 = 3.4 MB each way) on two streams, alone and together,
through the same registered host buffers the bench uses.
  python tools/probe_pcie_duplex.py [MB]"""
import ctypes, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402  (host_pinned)

mb = float(sys.argv[1]) if len(sys.argv) > 1 else 3.25
n = int(mb * (1 << 20) / 4)
dev = torch.device("cuda", 0)
hs = [bench.host_pinned((n,)) for _ in range(6)]
d = [torch.empty(n, device=dev) for _ in range(6)]
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
def run(mode, reps=200):
    for _ in range(2):
        for k in range(reps):
            if mode in ("h2d", "both"):
                with torch.cuda.stream(sa): d[k % 3].copy_(hs[k % 3], non_blocking=True)
            if mode in ("d2h", "both"):
                with torch.cuda.stream(sb): hs[3 + k % 3].copy_(d[3 + k % 3], non_blocking=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(sa); sb.wait_event(e0)
        if reps == 0: break
        t0 = e0
    # timed
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    sa.wait_stream(torch.cuda.current_stream()); sb.wait_stream(torch.cuda.current_stream())
    for k in range(reps):
        if mode in ("h2d", "both"):
            with torch.cuda.stream(sa): d[k % 3].copy_(hs[k % 3], non_blocking=True)
        if mode in ("d2h", "both"):
            with torch.cuda.stream(sb): hs[3 + k % 3].copy_(d[3 + k % 3], non_blocking=True)
    torch.cuda.current_stream().wait_stream(sa); torch.cuda.current_stream().wait_stream(sb)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    print(f"{mode:5s} {mb:.2f} MB per step: {us:7.1f} us/step  {n * 4 / us / 1e3:6.1f} GB/s each way")
for m in ("h2d", "d2h", "both"):
    run(m)
