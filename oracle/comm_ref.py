"""Numpy restatement of the reference hot path (TEST INFRASTRUCTURE ONLY — see oracle/__init__).

Follows /root/reference/pkg/src/streamsgd/comm.py and nn.py; each function cites the lines.
Everything is float64, like the reference.
"""

from __future__ import annotations

import math

import numpy as np

VALUE_BYTES = 4  # comm.py:16
INDEX_BYTES = 4  # comm.py:17


def topk_count(dim: int, cr: float) -> int:
    """comm.py:81-87 — max(1, ceil(cr*dim - 1e-12)), cr in (0, 1]."""
    if not (0.0 < cr <= 1.0):
        raise ValueError("compression ratio must lie in (0, 1]")
    return max(1, math.ceil(cr * dim - 1e-12))


def rate_weights(rates) -> np.ndarray:
    """comm.py:57-64 — r_j = S_j / sum(S) in float64."""
    s = np.asarray(rates, dtype=np.float64)
    if s.size == 0 or np.any(s < 1):
        raise ValueError("rates must be non-empty and >= 1")
    return s / s.sum()


def topk_indices_lexsort(g: np.ndarray, m: int) -> np.ndarray:
    """comm.py:94-95 — primary key -|g| ascending, secondary the index; first m, re-sorted.

    This is the reference's own O(D log D) algorithm (numpy lexsort puts NaN keys last)."""
    g = np.asarray(g, dtype=np.float64)
    order = np.lexsort((np.arange(g.size), -np.abs(g)))
    return np.sort(order[:m])


def topk_indices_threshold(g: np.ndarray, m: int) -> np.ndarray:
    """Same selection as topk_indices_lexsort in O(D): threshold by np.partition.

    a = |g| with NaN mapped below every number; T = the m-th largest a; keep a > T plus the
    lowest-index (m - count(a > T)) entries with a == T.  Validated against the lexsort form
    in tests/test_oracle.py before being used for large D."""
    g = np.asarray(g)
    a = np.abs(g).astype(np.float64)
    a[np.isnan(a)] = -1.0
    D = a.size
    T = np.partition(a, D - m)[D - m]
    above = np.flatnonzero(a > T)
    ties = np.flatnonzero(a == T)[: m - above.size]
    return np.sort(np.concatenate([above, ties]))


def topk(g: np.ndarray, cr: float, method: str = "lexsort"):
    """comm.py:90-96 — (indices int64 ascending, values = g[indices])."""
    g = np.asarray(g, dtype=np.float64)
    m = topk_count(g.size, cr)
    if g.size == 0:
        return np.zeros(0, dtype=np.int64), np.zeros(0)
    pick = topk_indices_lexsort if method == "lexsort" else topk_indices_threshold
    idx = pick(g, m).astype(np.int64)
    return idx, g[idx]


def densify(dim: int, idx, vals) -> np.ndarray:
    """comm.py:45-50 — zeros(dim) with the kept values scattered in."""
    out = np.zeros(dim)
    out[np.asarray(idx, dtype=np.int64)] = vals
    return out


def aggregate(payloads, weights) -> np.ndarray:
    """comm.py:67-78 — acc = 0; acc += w_j * densify(p_j) for j ascending.

    A payload is a dense float64 vector or a (dim, idx, vals) triple."""
    w = np.asarray(weights, dtype=np.float64)
    if len(payloads) != len(w):
        raise ValueError("one weight per gradient required")
    dims = {p[0] if isinstance(p, tuple) else len(p) for p in payloads}
    if len(dims) != 1:
        raise ValueError("gradient dimensions differ")
    acc = np.zeros(dims.pop())
    for wj, p in zip(w, payloads):
        dense = densify(*p) if isinstance(p, tuple) else np.asarray(p, dtype=np.float64)
        acc += wj * dense
    return acc


class GateState:
    """comm.py:99-119 — the per-worker EWMA gate state."""

    def __init__(self, cr, delta, ewma_factor=0.9, raw_gate=False):
        self.cr, self.delta, self.f, self.raw = cr, delta, ewma_factor, raw_gate
        self.ewma_full = 0.0
        self.ewma_topk = 0.0
        self.initialized = False
        self.n_compressed = 0
        self.n_uncompressed = 0


def gate(g: np.ndarray, st: GateState, method: str = "lexsort"):
    """comm.py:129-160 — (compressed, (idx, vals) or g, rho, s_full, s_topk); mutates st."""
    g = np.asarray(g, dtype=np.float64)
    idx, vals = topk(g, st.cr, method)
    s_full = float(g @ g)
    s_topk = float(vals @ vals)
    if st.initialized:
        st.ewma_full = st.f * st.ewma_full + (1.0 - st.f) * s_full
        st.ewma_topk = st.f * st.ewma_topk + (1.0 - st.f) * s_topk
    else:
        st.ewma_full, st.ewma_topk, st.initialized = s_full, s_topk, True
    full, kept = (s_full, s_topk) if st.raw else (st.ewma_full, st.ewma_topk)
    rho = 0.0 if full == 0.0 else abs(full - kept) / full
    if rho <= st.delta:
        st.n_compressed += 1
        return True, (idx, vals), rho, s_full, s_topk
    st.n_uncompressed += 1
    return False, g, rho, s_full, s_topk


def volume(compressed: bool, dim: int, cr: float) -> tuple[int, int]:
    """comm.py:177-197 — (floats, bytes) of one payload."""
    if compressed:
        m = topk_count(dim, cr)
        return m, m * (VALUE_BYTES + INDEX_BYTES)
    return dim, dim * VALUE_BYTES


def sgd_momentum(params: np.ndarray, buf, grad: np.ndarray, lr: float, momentum: float,
                 weight_decay: float):
    """nn.py:161-172 — returns (new params, new buffer); buf None = lazily created zeros."""
    b = np.zeros_like(params) if buf is None else np.array(buf, dtype=np.float64)
    b *= momentum
    b += grad + weight_decay * params
    p = params - lr * b
    return p, b


def step_reference(grads, states, weights, params, buf, lr, momentum, weight_decay,
                   compression=True, method="lexsort"):
    """One synchronous iteration of engine.py:248-286 minus the gradient producer:
    gate every worker, aggregate, momentum step.  Returns (params, buf, aggregate, decisions)."""
    payloads, decisions = [], []
    for g, st in zip(grads, states):
        if compression:
            c, payload, _, _, _ = gate(g, st, method)
            decisions.append(c)
            payloads.append((len(g), *payload) if c else payload)
        else:
            payloads.append(np.asarray(g, dtype=np.float64))
    agg = aggregate(payloads, weights)
    p, b = sgd_momentum(params, buf, agg, lr, momentum, weight_decay)
    return p, b, agg, decisions
