import torch, numpy as np, sys
sys.path.insert(0, '.')
from paper_2407_04272_b200 import codec as K, _lib
from oracle import Ref
ref = Ref()
dev = 'cuda:0'
T, B, dim = 3, 64, 8
for codec in (1, 2, 0):
    look = [torch.zeros((B, dim), device=dev) for _ in range(T)]
    look[1][5, 3] = float('nan')
    jobs = [K.EncodeJob(l, 0.01, codec) for l in look]
    try:
        K.encode_chunks(jobs, K.LAYOUT_CHUNKS, meta=True)
        print("no error?!")
    except Exception as e:
        print("err", e)
    look[1][5, 3] = 0.0
    r = K.encode_chunks(jobs, K.LAYOUT_CHUNKS, meta=True)
    want = b"".join(ref.encode_chunk(l.cpu().numpy().astype(np.float64), dim, 0.01, codec) for l in look)
    got = bytes(r.buffer.cpu().numpy().tobytes())
    print(codec, "bytes equal", got == want, len(got), len(want), r.lengths.cpu().tolist())
