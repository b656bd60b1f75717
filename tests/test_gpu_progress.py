"""Forward progress of the codec kernels while other work holds most of the GPU.

The kernels assign work by block index and only ever wait on lower indices
(decode roles, encode look-backs, vlz hash windows) or, in the single-launch
encode, on the codebook of the tile's own job (built by that job's last tile).
A test-built "hog" kernel keeps one 100 KB-shared-memory CTA on every SM for
a bounded time (3 s); the Kaggle-shaped compress + decompress on another stream must
finish long before the hog does (it must not need the hog's slots back) and
produce the same bytes and values as without it.
"""
import ctypes
import os
import shutil
import subprocess
import time

import numpy as np
import pytest
import torch

from paper_2407_04272_b200 import _lib
from paper_2407_04272_b200 import codec as K
from paper_2407_04272_b200 import workload as W

pytestmark = pytest.mark.gpu
DEV = "cuda:0"

HOG_SRC = r"""
#include <cuda_runtime.h>
__global__ void k_hog(unsigned long long ns, int* done) {
  extern __shared__ int sm[];
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
  if (threadIdx.x == 0 && sm[0] == 12345) *done = 1;
}
extern "C" int hog_launch(unsigned long long ns, int smem, int ctas, void* stream, int* done) {
  if (cudaFuncSetAttribute(k_hog, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return 1;
  k_hog<<<ctas, 32, smem, (cudaStream_t)stream>>>(ns, done);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
"""


@pytest.fixture(scope="module")
def hog(tmp_path_factory):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    d = tmp_path_factory.mktemp("hog")
    src, lib = d / "hog.cu", d / "libhog.so"
    src.write_text(HOG_SRC)
    subprocess.run([nvcc, "-shared", "-Xcompiler", "-fPIC", "-gencode", "arch=compute_100a,code=sm_100a",
                    "-o", str(lib), str(src)], check=True)
    h = ctypes.CDLL(str(lib))
    h.hog_launch.argtypes = [ctypes.c_ulonglong, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    return h


def kg_step_inputs():
    specs = W.workload_specs("kg")
    prof = W.workload_profiles("kg")
    B = W.WORKLOADS["kg"]["batch"](1)
    xs = [W.Table(specs[t], DEV).lookup_batch(B, W.lookup_stream(0, t, 0, 1)) for t in range(len(specs))]
    return xs, [prof[t].eb for t in range(len(specs))], [prof[t].codec for t in range(len(specs))]


def test_codec_progresses_beside_a_hog(hog):
    xs, ebs, codecs = kg_step_inputs()
    jobs = [K.EncodeJob(x, eb, c) for x, eb, c in zip(xs, ebs, codecs)]
    want = K.encode_chunks(jobs, K.LAYOUT_PACKED)
    torch.cuda.synchronize()
    want_bytes = bytes(want.buffer[: want.total].cpu().numpy().tobytes())
    table = K.unpack_table(want_bytes)
    ctx = K.Context.default(0)
    cj = [j.to_c() for j in jobs]
    out = torch.zeros(int(want.total) + 256, dtype=torch.uint8, device=DEV)
    ys = [torch.empty_like(x) for x in xs]
    refs = []
    for t, (o, ln) in enumerate(table):
        r = _lib.ChunkRef()
        r.offset, r.length, r.out = o, ln, ys[t].data_ptr()
        r.dim, r.count, r.codec = xs[t].shape[1], xs[t].shape[0], codecs[t]
        refs.append(r)
    props = torch.cuda.get_device_properties(0)
    nsm = props.multi_processor_count
    done = torch.zeros(1, dtype=torch.int32, device=DEV)
    s_hog, s_run = torch.cuda.Stream(), torch.cuda.Stream()
    hog_ms = 3000
    # one CTA per SM with 100 KB of shared memory: each SM keeps room for one
    # or two codec CTAs, fewer slots than the step's encode and decode have CTAs
    rc = hog.hog_launch(hog_ms * 1_000_000, 100 * 1024, nsm, ctypes.c_void_p(s_hog.cuda_stream),
                        ctypes.c_void_p(done.data_ptr()))
    assert rc == 0
    time.sleep(0.05)  # the hog is resident
    t0 = time.monotonic()
    ctx.encode_raw(cj, K.LAYOUT_PACKED, out, stream=s_run)
    ctx.decode_raw(out, refs, K.OUT_F32, False, stream=s_run)
    ev = torch.cuda.Event()
    ev.record(s_run)
    while not ev.query():
        assert time.monotonic() - t0 < hog_ms / 1000 * 0.5, "the codec waited on the hog's slots"
        time.sleep(0.001)
    elapsed = time.monotonic() - t0
    torch.cuda.synchronize()
    assert bytes(out[: want.total].cpu().numpy().tobytes()) == want_bytes
    for t in range(len(xs)):
        err = (ys[t].double() - xs[t].double()).abs().max().item()
        assert err <= ebs[t] * (1 + 1e-12), t
    assert elapsed < hog_ms / 1000 * 0.5
