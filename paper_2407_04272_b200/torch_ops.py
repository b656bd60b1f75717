"""PyTorch operator for the compressed embedding all-to-all.

    torch.ops.embc.compressed_all_to_all(handle, iteration, lookups) -> Tensor [B, T, dim]

`lookups` are the rank's owned tables' embedding-bag outputs, [R*B, dim] each,
in the order of `exchange.owned(rank)`, with rows d*B..(d+1)*B destined to rank
d (the model-parallel -> data-parallel hand-off of a hybrid-parallel DLRM,
PAPER.md:36).  The result is the data-parallel interaction input [B, T, dim]
(a [T, B, dim]-strided view: every table's slice is decoded straight into its
[B, dim] plane, no extra copy).  Autograd is wired: backward() sends every
table's [B, dim] gradient slice back to its owner through the compressed
backward all-to-all and returns the owned tables' [R*B, dim]
gradients.

`handle` names an exchange registered with `register_exchange` -- the product
`NcclExchange` (embc_exchange_* over NCCL) or the torch.distributed
`CompressedAllToAll`; the error bound of each table per iteration comes from
the exchange's dual-level controller (eb_at, policy.hpp:336-342), the
gradient's from its own profiles.
"""
from __future__ import annotations

import itertools
import threading
from typing import Dict, List

import torch

_REG: Dict[int, object] = {}
_LOCK = threading.Lock()
_NEXT = itertools.count(1)


def register_exchange(ex) -> int:
    """Register an exchange object; returns the integer handle the op takes."""
    with _LOCK:
        h = next(_NEXT)
        _REG[h] = ex
    return h


def unregister_exchange(handle: int) -> None:
    with _LOCK:
        _REG.pop(handle, None)


def _ex(handle: int):
    try:
        return _REG[handle]
    except KeyError:
        raise ValueError(f"embc: no exchange registered under handle {handle}") from None


@torch.library.custom_op("embc::compressed_all_to_all", mutates_args=())
def compressed_all_to_all(handle: int, iteration: int, lookups: List[torch.Tensor]) -> torch.Tensor:
    ex = _ex(handle)
    own = ex.owned(ex.rank)
    if len(lookups) != len(own):
        raise ValueError(f"embc: rank {ex.rank} owns {len(own)} tables, got {len(lookups)} lookup tensors")
    for t, x in zip(own, lookups):
        if tuple(x.shape) != (ex.R * ex.B, ex.dim):
            raise ValueError(f"embc: table {t} lookup must be [{ex.R * ex.B}, {ex.dim}], got {list(x.shape)}")
    planes = torch.empty((ex.T, ex.B, ex.dim), dtype=torch.float32, device=ex.device)
    ex.forward(iteration, {t: x.contiguous() for t, x in zip(own, lookups)},
               out={t: planes[t] for t in range(ex.T)})
    return planes.permute(1, 0, 2)


@compressed_all_to_all.register_fake
def _(handle: int, iteration: int, lookups: List[torch.Tensor]) -> torch.Tensor:
    ex = _ex(handle)
    planes = lookups[0].new_empty((ex.T, ex.B, ex.dim)) if lookups else torch.empty((ex.T, ex.B, ex.dim))
    return planes.permute(1, 0, 2)


@torch.library.custom_op("embc::compressed_all_to_all_backward", mutates_args=())
def compressed_all_to_all_backward(handle: int, iteration: int, grad: torch.Tensor) -> List[torch.Tensor]:
    ex = _ex(handle)
    if tuple(grad.shape) != (ex.B, ex.T, ex.dim):
        raise ValueError(f"embc: gradient must be [{ex.B}, {ex.T}, {ex.dim}], got {list(grad.shape)}")
    planes = grad.permute(1, 0, 2).to(torch.float32).contiguous()  # [T, B, dim]: one contiguous slice per table
    got = ex.backward(iteration, {t: planes[t] for t in range(ex.T)})
    return [got[t] for t in ex.owned(ex.rank)]


@compressed_all_to_all_backward.register_fake
def _(handle: int, iteration: int, grad: torch.Tensor) -> List[torch.Tensor]:
    ex = _ex(handle)
    return [grad.new_empty((ex.R * ex.B, ex.dim)) for _ in ex.owned(ex.rank)]


def _setup_context(ctx, inputs, output):
    ctx.handle, ctx.iteration = inputs[0], inputs[1]
    ctx.n = len(inputs[2])


def _backward(ctx, grad):
    grads = torch.ops.embc.compressed_all_to_all_backward(ctx.handle, ctx.iteration, grad)
    return None, None, list(grads)


torch.library.register_autograd("embc::compressed_all_to_all", _backward, setup_context=_setup_context)


class CompressedEmbeddingExchange(torch.nn.Module):
    """Module form: y = module(lookups) with an iteration counter the controller's
    iteration-wise decay reads (eb_at)."""

    def __init__(self, exchange):
        super().__init__()
        self.exchange = exchange
        self.handle = register_exchange(exchange)
        self.iteration = 0

    def forward(self, lookups: List[torch.Tensor]) -> torch.Tensor:
        y = torch.ops.embc.compressed_all_to_all(self.handle, self.iteration, list(lookups))
        return y

    def step(self) -> None:
        self.iteration += 1

    def __del__(self):
        try:
            unregister_exchange(self.handle)
        except Exception:
            pass
