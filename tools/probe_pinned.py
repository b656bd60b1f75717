"""H2D throughput of pinned buffers by allocation method, several fresh buffers each:
torch pin_memory (cudaHostAlloc) vs. 2 MB-aligned anonymous memory with
MADV_HUGEPAGE registered with cudaHostRegister."""
import ctypes, mmap, time
import numpy as np
import torch

NB = int(3.25 * 2**20)
dev = torch.empty(NB // 4, dtype=torch.float32, device="cuda")
cudart = torch.cuda.cudart()
libc = ctypes.CDLL("libc.so.6")

def h2d_us(h, reps=30):
    for _ in range(3):
        dev.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        dev.copy_(h, non_blocking=True)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3

keep = []
res = []
for i in range(8):
    h = torch.empty(NB // 4, dtype=torch.float32).pin_memory()
    h.fill_(1.0)
    keep.append(h)
    res.append(round(h2d_us(h), 1))
print("pin_memory      us per 3.25 MB H2D:", res)
res = []
for i in range(8):
    size = 4 << 20
    m = mmap.mmap(-1, size + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    base = ctypes.addressof(ctypes.c_char.from_buffer(m))
    aligned = (base + (2 << 20) - 1) & ~((2 << 20) - 1)
    libc.madvise(ctypes.c_void_p(aligned), ctypes.c_size_t(size), 14)  # MADV_HUGEPAGE
    arr = np.frombuffer((ctypes.c_char * size).from_address(aligned), dtype=np.float32)
    arr[:] = 1.0
    r = cudart.cudaHostRegister(aligned, size, 0)
    h = torch.from_numpy(arr[: NB // 4])
    keep.append((m, arr, h))
    res.append(round(h2d_us(h), 1))
print("THP + register  us per 3.25 MB H2D:", res)
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
