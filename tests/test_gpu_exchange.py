"""GPU: the compressed exchange on one rank (R = 1, the payload round is a
device copy) through the product backend, pipelined over table groups on
separate encode / decode streams, against the unpipelined exchange and the
oracle restatement."""
import numpy as np
import pytest
import torch

from paper_2407_04272_b200 import exchange as X
from paper_2407_04272_b200 import policy as P
from paper_2407_04272_b200 import workload as W

pytestmark = pytest.mark.gpu


def test_pipelined_exchange_single_rank(ctx, oracle):
    dev = torch.device("cuda", 0)
    T, dim, B = 9, 16, 512
    specs = W.preset_tables(W.KAGGLE_TABLES, T, dim)
    tables = [W.Table(s, dev) for s in specs]
    profiles = {t: P.TableProfile(t, codec=t % 3, eb=0.01 + 0.02 * (t % 2)) for t in range(T)}
    cfg = P.PolicyConfig(global_eb=0.01)
    ex1 = X.CompressedAllToAll(T, dim, B, profiles, cfg, device=dev)
    ex4 = X.CompressedAllToAll(T, dim, B, profiles, cfg, device=dev, groups=4)
    for it in range(3):
        look = {t: tables[t].lookup_batch(B, W.lookup_stream(it, t, 0, 1)) for t in range(T)}
        a = ex1.forward(it, look)
        b = ex4.forward(it, look)
        torch.cuda.synchronize()
        assert (ex1.stats.payload_bytes, ex1.stats.uncompressed_bytes) == (ex4.stats.payload_bytes,
                                                                           ex4.stats.uncompressed_bytes)
        for t in range(T):
            assert torch.equal(a[t], b[t]), (it, t)
            x = look[t].cpu().numpy().astype(np.float64)
            want = oracle.decode_chunk(oracle.encode_chunk(x.ravel(), dim, profiles[t].eb, profiles[t].codec))
            assert np.array_equal(b[t].cpu().numpy(), want.astype(np.float32).reshape(B, dim)), (it, t)
        grads = {t: (b[t] * 0.5 + 0.01).contiguous() for t in range(T)}
        g1 = ex1.backward(it, grads)
        g4 = ex4.backward(it, grads)
        torch.cuda.synchronize()
        assert ex1.stats.payload_bytes == ex4.stats.payload_bytes
        for t in range(T):
            assert torch.equal(g1[t], g4[t]), ("bwd", it, t)
