"""Route the reference training loop's hot path through this package.

The reference engine looks its collaborators up as module attributes at call time
(``from . import comm, datagen, nn, streams`` at engine.py:18; ``comm.compression_gate`` at
engine.py:253, ``comm.weights_from_rates``/``comm.weighted_aggregate`` at 266-270,
``nn.OptimizerState`` at 133-140 and ``nn.sgd_momentum_step`` at 282-283).  ``install`` swaps
``engine.comm`` for :mod:`paper_2301_08897_b200.comm` and ``engine.nn`` for a proxy whose
optimizer entries come from :mod:`paper_2301_08897_b200.nn` while the gradient producer
(MLP forward/backward, init, evaluate) stays the reference's.  ``uninstall`` restores both.
"""

from __future__ import annotations

import types

from . import comm as _comm
from . import nn as _nn

_OPT_NAMES = ("OptimizerState", "sgd_momentum_step", "lr_at_epoch", "scale_lr")


class _NNProxy(types.ModuleType):
    def __init__(self, base):
        super().__init__(base.__name__)
        self._base = base
        for name in _OPT_NAMES:
            setattr(self, name, getattr(_nn, name))

    def __getattr__(self, name):
        return getattr(self._base, name)


def install(engine_module) -> tuple:
    """Substitute the B200 modules into a ``streamsgd.engine`` module; returns the originals."""
    saved = (engine_module.comm, engine_module.nn)
    engine_module.comm = _comm
    engine_module.nn = _NNProxy(saved[1])
    return saved


def uninstall(engine_module, saved: tuple) -> None:
    engine_module.comm, engine_module.nn = saved
