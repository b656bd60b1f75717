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


@pytest.mark.parametrize("groups", [1, 3])
def test_nccl_exchange_single_rank(ctx, ref, groups):
    """The C++ exchange over NCCL (embc_exchange_*, a one-rank communicator:
    the metadata and payload rounds are real ncclSend/ncclRecv to self) delivers
    byte for byte what the reference's encode_chunk + decode_chunk deliver, with
    the same accounting as the torch.distributed exchange, forward and
    backward, with a mid-decay bound; the uncompressed baseline is exact."""
    dev = torch.device("cuda", 0)
    T, dim, B = 7, 16, 768
    specs = W.preset_tables(W.KAGGLE_TABLES, T, dim)
    tables = [W.Table(s, dev) for s in specs]
    profiles = {t: P.TableProfile(t, codec=t % 3, eb=0.01 + 0.02 * (t % 2)) for t in range(T)}
    cfg = P.PolicyConfig(global_eb=0.01, decay=P.DecayConfig("stepwise", 2.0, 4, 4))
    gprof = {t: P.TableProfile(t, codec=2 - t % 2, eb=1e-4) for t in range(T)}
    gcfg = P.PolicyConfig(global_eb=1e-4)
    nx = X.NcclExchange(T, dim, B, profiles, cfg, device=dev, grad_profiles=gprof, grad_cfg=gcfg, groups=groups)
    tx = X.CompressedAllToAll(T, dim, B, profiles, cfg, device=dev, grad_profiles=gprof, grad_cfg=gcfg)
    for it in (0, 2, 5):
        look = {t: tables[t].lookup_batch(B, W.lookup_stream(it, t, 0, 1)) for t in range(T)}
        a = nx.forward(it, look)
        sa = nx.stats
        b = tx.forward(it, look)
        for t in range(T):
            assert torch.equal(a[t], b[t]), (it, t)
            x = look[t].cpu().numpy().astype(np.float64)
            eb = P.eb_at(t, it, profiles, cfg)
            want = ref.decode_chunk(ref.encode_chunk(x, dim, eb, profiles[t].codec))
            assert np.array_equal(a[t].cpu().numpy(), want.astype(np.float32)), (it, t)
        assert (sa.payload_bytes, sa.metadata_bytes, sa.uncompressed_bytes) == (0, 0, 0)  # R = 1: nothing leaves
        assert sa.sent_values == sa.recv_values == T * B * dim and sa.sent_bytes == sa.recv_bytes > 0
        g = {t: (torch.randn((B, dim), device=dev, generator=torch.Generator(dev).manual_seed(it * 31 + t)) * 1e-3)
             for t in range(T)}
        ga = nx.backward(it, g)
        gb = tx.backward(it, g)
        for t in range(T):
            assert torch.equal(ga[t], gb[t]), ("bwd", it, t)
            assert (ga[t] - g[t]).abs().max().item() <= 1e-4 * 1.0000001
        u = nx.uncompressed(look)
        ub = nx.uncompressed_backward(g)
        for t in range(T):
            assert torch.equal(u[t], look[t]) and torch.equal(ub[t], g[t])


def test_nccl_exchange_reports_codec_failure(ctx):
    """A non-finite value in a lookup: the compress stage's ValueError with the
    reference's rank/stage attribution (commsim.hpp:317-319); the exchange
    stays usable."""
    dev = torch.device("cuda", 0)
    T, dim, B = 3, 8, 64
    profiles = {t: P.TableProfile(t, codec=1, eb=0.01) for t in range(T)}
    nx = X.NcclExchange(T, dim, B, profiles, P.PolicyConfig(global_eb=0.01), device=dev)
    look = {t: torch.zeros((B, dim), device=dev) for t in range(T)}
    look[1][5, 3] = float("nan")
    from paper_2407_04272_b200 import _lib
    with pytest.raises(_lib.CodecValueError, match=r"^rank 0 forward compress stage: non-finite value at index 43$"):
        nx.forward(0, look)
    look[1][5, 3] = 0.0
    out = nx.forward(0, look)
    assert all(torch.equal(out[t], look[t]) for t in range(T))


def test_p2p_exchange_single_rank(ctx):
    """The peer-to-peer transport (chunks written into the destination's
    window, flags, device-planned decode) delivers byte for byte what the NCCL
    two-round exchange delivers, with the same accounting, forward and
    backward, over several iterations of a decaying bound (a one-rank loopback:
    the window is this rank's own)."""
    dev = torch.device("cuda", 0)
    T, dim, B = 9, 16, 1024
    specs = W.preset_tables(W.KAGGLE_TABLES, T, dim)
    tables = [W.Table(s, dev) for s in specs]
    profiles = {t: P.TableProfile(t, codec=t % 3, eb=0.01 + 0.02 * (t % 2)) for t in range(T)}
    cfg = P.PolicyConfig(global_eb=0.01, decay=P.DecayConfig("stepwise", 2.0, 4, 4))
    gprof = {t: P.TableProfile(t, codec=2 - t % 2, eb=1e-4) for t in range(T)}
    gcfg = P.PolicyConfig(global_eb=1e-4)
    nx = X.NcclExchange(T, dim, B, profiles, cfg, device=dev, grad_profiles=gprof, grad_cfg=gcfg)
    px = X.NcclExchange(T, dim, B, profiles, cfg, device=dev, grad_profiles=gprof, grad_cfg=gcfg, p2p=True)
    for it in (0, 1, 3, 6):
        look = {t: tables[t].lookup_batch(B, W.lookup_stream(it, t, 0, 1)) for t in range(T)}
        a = nx.forward(it, look)
        b = px.forward(it, look)
        assert vars(nx.stats) == vars(px.stats)
        for t in range(T):
            assert torch.equal(a[t], b[t]), (it, t)
        g = {t: (torch.randn((B, dim), device=dev, generator=torch.Generator(dev).manual_seed(it * 7 + t)) * 1e-3)
             for t in range(T)}
        ga = nx.backward(it, g)
        gb = px.backward(it, g)
        assert vars(nx.stats) == vars(px.stats)
        for t in range(T):
            assert torch.equal(ga[t], gb[t]), ("bwd", it, t)


def test_p2p_exchange_cuda_graph(ctx):
    """The peer-to-peer forward is graph-capturable (no host read of the
    lengths): one capture, replays with other iterations' lookups (other chunk
    lengths) deliver what the eager two-round exchange delivers."""
    dev = torch.device("cuda", 0)
    T, dim, B = 7, 16, 2048
    specs = W.preset_tables(W.KAGGLE_TABLES, T, dim)
    tables = [W.Table(s, dev) for s in specs]
    profiles = {t: P.TableProfile(t, codec=1 + t % 2, eb=0.02) for t in range(T)}
    cfg = P.PolicyConfig(global_eb=0.02)
    nx = X.NcclExchange(T, dim, B, profiles, cfg, device=dev)
    px = X.NcclExchange(T, dim, B, profiles, cfg, device=dev, p2p=True)
    look = {t: tables[t].lookup_batch(B, W.lookup_stream(0, t, 0, 1)).clone() for t in range(T)}
    out = {t: torch.empty((B, dim), device=dev) for t in range(T)}
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        px.forward(0, look, out=out, stats=False)  # warm-up: windows and scratch sized
    s.synchronize()
    px.sync()
    px.reserve_capture(64 << 20)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        px.forward(0, look, out=out, stats=False)
    for it in (1, 2, 3):
        for t in range(T):
            look[t].copy_(tables[t].lookup_batch(B, W.lookup_stream(it, t, 0, 1)))
        g.replay()
        torch.cuda.synchronize()
        px.sync()
        want = nx.forward(0, look)
        for t in range(T):
            assert torch.equal(out[t], want[t]), (it, t)
