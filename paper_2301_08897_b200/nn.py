"""Drop-in for the optimizer part of ``streamsgd.nn`` (reference nn.py:144-190).

``sgd_momentum_step`` runs the fused momentum-SGD kernel: buffer <- momentum*buffer +
(grad + wd*params); params <- params - lr*buffer, in binary64 round-to-nearest for float64
inputs (bit-identical to numpy's in-place ufunc sequence at nn.py:169-171) and binary64
arithmetic on float32 storage for CUDA float32 tensors.  The MLP forward/backward of the
reference is the gradient *producer* and is out of scope; the drop-in helper
forwards those names to the reference module untouched.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import kernels


@dataclass
class OptimizerState:
    """Momentum SGD state; weight decay is folded into the momentum buffer (nn.py:144-158)."""

    momentum: float = 0.9
    weight_decay: float = 0.0
    base_lr: float = 0.1
    schedule: list = field(default_factory=list)
    momentum_buffer: object = None

    def __post_init__(self):
        if not 0.0 <= self.momentum < 1.0:
            raise ValueError("momentum must lie in [0, 1)")
        if self.base_lr <= 0:
            raise ValueError("base_lr must be positive")


def _as_device(x, dtype):
    """``x`` as a CUDA tensor of ``dtype`` (device tensors of another dtype are converted, so
    the kernel never reads a buffer as the wrong element type)."""
    if isinstance(x, torch.Tensor) and x.is_cuda:
        return x if x.dtype == dtype else x.to(dtype)
    kernels.require_cuda()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(
        torch.device("cuda", torch.cuda.current_device()), dtype=dtype
    )


def sgd_momentum_step(state: OptimizerState, params, grad, lr: float):
    """buffer <- momentum*buffer + (grad + wd*params); params <- params - lr*buffer (nn.py:161-172).

    ``params`` is updated in place (numpy arrays are round-tripped through the device and
    written back into the same buffer, like the reference's in-place ufuncs).
    """
    if tuple(params.shape) != tuple(grad.shape):
        raise ValueError("parameter and gradient shapes differ")
    on_dev = isinstance(params, torch.Tensor) and params.is_cuda
    dt = params.dtype if on_dev else torch.float64
    p = params if on_dev else _as_device(params, dt)
    g = _as_device(grad, dt)
    first = state.momentum_buffer is None
    if first:
        buf = torch.empty_like(p)
    elif (isinstance(state.momentum_buffer, torch.Tensor) and state.momentum_buffer.is_cuda
          and state.momentum_buffer.dtype == dt):
        buf = state.momentum_buffer
    else:
        buf = _as_device(state.momentum_buffer, dt)
    kernels.sgd_momentum(p, buf, g, lr, state.momentum, state.weight_decay, first)
    if on_dev:
        state.momentum_buffer = buf
        return params
    state.momentum_buffer = buf.cpu().numpy()
    params[...] = p.cpu().numpy()
    return params


def lr_at_epoch(base_lr: float, schedule, epoch: int) -> float:
    """Step decay: multiply by every milestone factor whose epoch has passed (nn.py:175-181)."""
    lr = base_lr
    for milestone, factor in schedule:
        if epoch >= milestone:
            lr *= factor
    return lr


def scale_lr(base_lr: float, sum_rates: float, base_global_batch: int) -> float:
    """Linear scaling lr * sum(S) / B (nn.py:184-190)."""
    if base_global_batch < 1:
        raise ValueError("base global batch must be >= 1")
    if sum_rates < 1:
        raise ValueError("sum of rates must be >= 1")
    return base_lr * sum_rates / base_global_batch
