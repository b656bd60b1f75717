"""Pinned H2D / D2H bandwidth by size, torch copy_ vs. a raw cudaMemcpyAsync, vs. an SM copy from mapped host memory."""
import ctypes, glob, os, time
import torch
rt = None
for cand in glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*")) + ["libcudart.so"]:
    try:
        rt = ctypes.CDLL(cand); break
    except OSError:
        pass
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); a = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - a) / reps
for mb in (1, 3.4, 8, 16, 54.5):
    n = int(mb * 2**20 / 4)
    h1 = torch.empty(n, dtype=torch.float32).pin_memory()
    d1 = torch.empty(n, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    h2d = t(lambda: d1.copy_(h1, non_blocking=True))
    raw = None
    if rt is not None:
        raw = t(lambda: rt.cudaMemcpyAsync(ctypes.c_void_p(d1.data_ptr()), ctypes.c_void_p(h1.data_ptr()),
                                           ctypes.c_size_t(n * 4), 1, ctypes.c_void_p(s)))
    print(f"{mb} MB: torch H2D {n*4/h2d/1e9:.1f} GB/s ({h2d*1e6:.0f} us), raw cudaMemcpyAsync "
          f"{(n*4/raw/1e9) if raw else 0:.1f} GB/s")

# H2D split across streams (copy engines), and repeated small H2D
for mb in (3.25, 52):
    n = int(mb * 2**20 / 4)
    h1 = torch.empty(n, dtype=torch.float32).pin_memory()
    d1 = torch.empty(n, dtype=torch.float32, device="cuda")
    for parts in (1, 2, 4, 8):
        ss = [torch.cuda.Stream() for _ in range(parts)]
        step = (n + parts - 1) // parts
        def f():
            cur = torch.cuda.current_stream()
            for i, s in enumerate(ss):
                s.wait_stream(cur)
                with torch.cuda.stream(s):
                    d1[i * step:(i + 1) * step].copy_(h1[i * step:(i + 1) * step], non_blocking=True)
            for s in ss:
                cur.wait_stream(s)
        dt = t(f)
        print(f"{mb} MB H2D in {parts} streams: {n*4/dt/1e9:.1f} GB/s ({dt*1e6:.0f} us)")
