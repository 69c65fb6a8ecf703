"""Item (1) producer for a real model: autograd writes each worker's gradient straight into its
row of the exchange bucket, and the exchange's fused momentum SGD updates the model in place.

Reference contract: the flattened gradient is every parameter's gradient concatenated in
canonical order -- layers in order, weight before bias, row-major (``nn.loss_and_grad``
flat concat, nn.py:122-124) -- and the optimizer steps the flat parameter vector
(``nn.sgd_momentum_step`` on ``replica.flat``, nn.py:161-172, engine.py:282-283).

``bind(model, ex)`` re-points every parameter of ``model`` (``model.parameters()`` order,
which for torch modules is the canonical layer order with weight before bias) at a view of
``ex.params``, copying the current values in, so ``GradientExchange.step`` updates the model
without a copy.  ``worker_grads(model, ex, j)`` then makes each ``param.grad`` a view of
bucket row ``j`` (zeroed), so the next backward accumulates the gradient in place in the
canonical flat layout: no flatten, no copy, and the Top-k reads it where autograd wrote it.
"""

from __future__ import annotations

import torch


def layout(model: torch.nn.Module) -> list[tuple[torch.nn.Parameter, int, int]]:
    """(parameter, offset, numel) in canonical flat order."""
    out, off = [], 0
    for p in model.parameters():
        out.append((p, off, p.numel()))
        off += p.numel()
    return out


def flat_size(model: torch.nn.Module) -> int:
    return sum(p.numel() for p in model.parameters())


def bind(model: torch.nn.Module, ex) -> None:
    """Make the model's parameters views of ``ex.params`` (values copied in)."""
    lay = layout(model)
    if lay[-1][1] + lay[-1][2] != ex.dim:
        raise ValueError(f"model has {flat_size(model)} parameters, the exchange {ex.dim}")
    with torch.no_grad():
        for p, off, n in lay:
            if p.dtype != ex.params.dtype or p.device != ex.params.device:
                raise ValueError("parameters must match the exchange dtype and device")
            view = ex.params[off:off + n].view_as(p)
            view.copy_(p)
            p.data = view


def worker_grads(model: torch.nn.Module, ex, j: int) -> None:
    """Point every ``param.grad`` at its slice of bucket row ``j`` and zero the row, so the
    next backward pass writes worker j's flattened gradient in place."""
    row = ex.bucket[j]
    row.zero_()
    for p, off, n in layout(model):
        p.grad = row[off:off + n].view_as(p)


def release_grads(model: torch.nn.Module) -> None:
    for p in model.parameters():
        p.grad = None
