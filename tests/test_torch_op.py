"""torch.ops.embc.compressed_all_to_all on CPU, world_size 2 (gloo), with the
oracle as the codec backend: forward delivers every table's slice as the
[B, T, dim] interaction input, autograd's backward runs the compressed
gradient all-to-all and returns each owned table's [R*B, dim] gradient, and
both equal the exchange called directly (the same chunks, byte for byte)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from test_exchange_gloo import OracleCodec
        from paper_2407_04272_b200 import exchange as X
        from paper_2407_04272_b200 import policy as P
        from paper_2407_04272_b200 import torch_ops as O
        T, dim, B = 5, 8, 16
        prof = {t: P.TableProfile(t, codec=t % 3, eb=0.01) for t in range(T)}
        gprof = {t: P.TableProfile(t, codec=(t + 1) % 3, eb=1e-3) for t in range(T)}
        cfg = P.PolicyConfig(global_eb=0.01, decay=P.DecayConfig("stepwise", 2.0, 4, 4))
        gcfg = P.PolicyConfig(global_eb=1e-3)
        ex = X.CompressedAllToAll(T, dim, B, prof, cfg, backend=OracleCodec(), device=torch.device("cpu"),
                                  grad_profiles=gprof, grad_cfg=gcfg)
        mod = O.CompressedEmbeddingExchange(ex)
        own = ex.owned(rank)
        g = torch.Generator().manual_seed(100 + rank)
        res = {}
        for it in range(2):
            look = [(torch.randn((world * B, dim), generator=g) * 0.1).requires_grad_() for _ in own]
            y = mod(look)
            assert tuple(y.shape) == (B, T, dim)
            direct = ex.forward(it, {t: x.detach() for t, x in zip(own, look)})
            fwd_eq = all(torch.equal(y[:, t, :], direct[t]) for t in range(T))
            w = torch.randn((B, T, dim), generator=g) * 0.01
            (y * w).sum().backward()
            want = ex.backward(it, {t: w[:, t, :].contiguous() for t in range(T)})
            bwd_eq = all(torch.equal(x.grad, want[t]) for t, x in zip(own, look))
            # bounded error against the exact gradient: rows s*B.. come from rank s's w
            allw = [torch.empty_like(w) for _ in range(world)]
            dist.all_gather(allw, w)
            bwd_err = max(((x.grad[s * B:(s + 1) * B] - allw[s][:, t, :]).abs().max().item()
                           for t, x in zip(own, look) for s in range(world)), default=0.0)
            res[it] = (fwd_eq, bwd_eq, bwd_err)
            mod.step()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_compressed_all_to_all_op_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    env_pp = os.environ.get("PYTHONPATH", "")
    here = os.path.dirname(os.path.abspath(__file__))
    os.environ["PYTHONPATH"] = os.pathsep.join([here, os.path.dirname(here), env_pp])
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, res in out.items():
        for it, (fwd_eq, bwd_eq, bwd_err) in res.items():
            assert fwd_eq, (rank, it)
            assert bwd_eq, (rank, it)
            assert bwd_err <= 1e-3 * (1 + 1e-9), (rank, it, bwd_err)


def test_op_registered():
    from paper_2407_04272_b200 import torch_ops  # noqa: F401
    assert hasattr(torch.ops.embc, "compressed_all_to_all")
    assert hasattr(torch.ops.embc, "compressed_all_to_all_backward")
    with pytest.raises(ValueError):
        torch.ops.embc.compressed_all_to_all(987654, 0, [torch.zeros(2, 2)])
