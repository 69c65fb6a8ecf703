"""Drop-in replacement of ``streamsgd.comm`` whose compute runs on the B200 kernels.

Same names, signatures, argument meaning, return types and ``ValueError`` messages as the
reference module (``/root/reference/pkg/src/streamsgd/comm.py``); the reference engine resolves
``comm.<fn>`` at call time (engine.py:18, 253-270), so substituting this module for
``streamsgd.engine.comm`` routes every gate and aggregation through the GPU
(see ``paper_2301_08897_b200.dropin``).

* numpy inputs take the float64 kernels: Top-k indices/values and the aggregate are
  bit-identical to the reference; gate decisions are identical except where |rho - delta|
  is within the last-bits difference of the two dot-product summation orders.
* CUDA float32 tensors take the float32 throughput kernels and stay on the device.

Accounting (``account_volume``, ``payload_bytes``), weights and the link cost model are
integer/scalar host arithmetic in the reference too and are
restated here unchanged in meaning.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _capi, kernels

FLOAT_BYTES = 4  # payloads are counted as single-precision floats (comm.py:16)
INDEX_BYTES = 4  # comm.py:17


def _device() -> torch.device:
    kernels.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


class SparseGradient:
    """Top-k remnant of a dense gradient (comm.py:20-42).

    Holds either host arrays (validated like the reference) or device tensors produced by the
    Top-k kernel (ascending by construction); host views are materialised lazily.
    """

    def __init__(self, dim: int, indices, values):
        self.dim = int(dim)
        self._dev = isinstance(indices, torch.Tensor) and indices.is_cuda
        if self._dev:
            self._idx_t = indices
            self._val_t = values
            self._indices = None
            self._values = None
            return
        self._idx_t = self._val_t = None
        self._indices = np.asarray(indices, dtype=np.int64)
        self._values = np.asarray(values, dtype=np.float64)
        if self._indices.shape != self._values.shape:
            raise ValueError("indices and values must align")
        if len(self._indices) and (
            np.any(np.diff(self._indices) <= 0) or self._indices[0] < 0 or self._indices[-1] >= self.dim
        ):
            raise ValueError("indices must be strictly increasing and < dim")

    @property
    def indices(self) -> np.ndarray:
        if self._indices is None:
            self._indices = self._idx_t.cpu().numpy().astype(np.int64)
        return self._indices

    @indices.setter
    def indices(self, v) -> None:
        self._indices = np.asarray(v, dtype=np.int64)
        self._idx_t = None
        self._dev = False

    @property
    def values(self) -> np.ndarray:
        if self._values is None:
            self._values = self._val_t.cpu().numpy().astype(np.float64)
        return self._values

    @values.setter
    def values(self, v) -> None:
        self._values = np.asarray(v, dtype=np.float64)
        self._val_t = None
        self._dev = False

    @property
    def nnz(self) -> int:
        return int(self._idx_t.numel()) if self._dev else len(self._indices)

    def device_arrays(self, dtype: torch.dtype = torch.float64):
        """(int32 indices, values) on the current CUDA device."""
        if self._dev and self._val_t.dtype == dtype:
            return self._idx_t, self._val_t
        dev = _device()
        idx = torch.from_numpy(self.indices.astype(np.int32)).to(dev)
        val = torch.from_numpy(self.values).to(dev, dtype=dtype)
        return idx, val

    def __repr__(self) -> str:
        return f"SparseGradient(dim={self.dim}, nnz={self.nnz})"


def densify(g) -> np.ndarray:
    """comm.py:45-50: zeros plus a scatter of the kept values (signed zeros preserved)."""
    if isinstance(g, SparseGradient):
        if g.dim == 0:
            return np.zeros(0)
        dev = _device()
        idx, val = g.device_arrays(torch.float64)
        out = torch.zeros(g.dim, dtype=torch.float64, device=dev)
        if g.nnz:
            out.index_copy_(0, idx.long(), val)
        return out.cpu().numpy()
    if isinstance(g, torch.Tensor):
        return g
    return np.asarray(g, dtype=np.float64)


def grad_dim(g) -> int:
    if isinstance(g, SparseGradient):
        return g.dim
    return int(g.shape[-1]) if isinstance(g, torch.Tensor) else len(g)


def weights_from_rates(rates) -> np.ndarray:
    """r = S / sum(S) (comm.py:57-64).  These, never batch sizes, are the aggregation weights."""
    r = np.asarray(rates, dtype=np.float64)
    if r.size == 0:
        raise ValueError("need at least one rate")
    if np.any(r < 1):
        raise ValueError("rates must be >= 1")
    return r / r.sum()


MAX_FOLD = 64  # workers per kernel launch (sg_weighted_aggregate_*); more are folded in chunks


def weighted_aggregate(grads, weights):
    """sum_j w_j * densify(g_j), folded in ascending j (comm.py:67-78), on the GPU.

    numpy / host payloads -> float64 kernel, returns a fresh float64 numpy array (bit-exact).
    CUDA float32 tensors / device payloads -> float32 kernel, returns a CUDA tensor.

    Any number of workers: beyond MAX_FOLD the fold continues chunk by chunk, each chunk
    starting from the previous chunk's float64 accumulator entered as a dense worker of
    weight 1.0 (0 + 1.0*acc == acc exactly, and acc never holds -0.0), so the ascending-j
    operation sequence -- and therefore every bit -- is the reference's.
    """
    w = np.asarray(weights, dtype=np.float64)
    if len(grads) != len(w):
        raise ValueError("one weight per gradient required")
    dims = {grad_dim(g) for g in grads}
    if len(dims) != 1:
        raise ValueError(f"gradient dimensions differ: {sorted(dims)}")
    dim = dims.pop()
    on_device = any(
        (isinstance(g, torch.Tensor) and g.is_cuda and g.dtype == torch.float32)
        or (isinstance(g, SparseGradient) and g._dev and g._val_t.dtype == torch.float32)
        for g in grads
    )
    dt = torch.float32 if on_device else torch.float64
    if dim == 0:
        return torch.zeros(0, dtype=dt, device=_device()) if on_device else np.zeros(0)
    if len(grads) <= MAX_FOLD:
        out = _aggregate(list(grads), w, dim, dt)
    else:
        acc = _aggregate(list(grads[:MAX_FOLD]), w[:MAX_FOLD], dim, torch.float64)
        for i in range(MAX_FOLD, len(grads), MAX_FOLD - 1):
            chunk = [acc] + list(grads[i:i + MAX_FOLD - 1])
            acc = _aggregate(chunk, np.concatenate(([1.0], w[i:i + MAX_FOLD - 1])), dim, torch.float64)
        out = acc.to(dt)
    return out if on_device else out.cpu().numpy()


def _aggregate(grads, w, dim, dt):
    """One kernel launch over <= MAX_FOLD workers; returns a CUDA tensor of dtype dt."""
    dev = _device()
    nw = len(grads)
    comp = np.array([isinstance(g, SparseGradient) for g in grads], dtype=np.uint8)
    dense = None
    if not comp.all():
        dense = torch.zeros((nw, dim), dtype=dt, device=dev)
        for j, g in enumerate(grads):
            if not comp[j]:
                dense[j] = torch.as_tensor(g if isinstance(g, torch.Tensor) else np.asarray(g, dtype=np.float64)).to(dev, dtype=dt)
    idx = val = row_ptr = comp_t = None
    if comp.any():
        parts_i, parts_v, ptr = [], [], [0]
        for j, g in enumerate(grads):
            if comp[j]:
                i_t, v_t = g.device_arrays(dt)
                parts_i.append(i_t)
                parts_v.append(v_t)
                ptr.append(ptr[-1] + g.nnz)
            else:
                ptr.append(ptr[-1])
        idx = torch.cat(parts_i) if parts_i else torch.zeros(0, dtype=torch.int32, device=dev)
        val = torch.cat(parts_v) if parts_v else torch.zeros(0, dtype=dt, device=dev)
        if idx.numel() == 0:  # keep valid pointers for an all-empty sparse set
            idx = torch.zeros(1, dtype=torch.int32, device=dev)
            val = torch.zeros(1, dtype=dt, device=dev)
        row_ptr = torch.tensor(ptr, dtype=torch.int64, device=dev)
        comp_t = torch.from_numpy(comp).to(dev)
    return kernels.weighted_aggregate(
        w, dim, compressed=comp_t, dense=dense, idx=idx, val=val, row_ptr=row_ptr, dtype=dt
    )


def topk_count(dim: int, cr: float) -> int:
    """Entries kept at compression ratio cr: max(1, ceil(cr*dim - 1e-12)) (comm.py:81-87)."""
    if not 0.0 < cr <= 1.0:
        raise ValueError("compression ratio must lie in (0, 1]")
    return max(1, math.ceil(cr * dim - 1e-12))


def topk_sparsify(g, cr: float) -> SparseGradient:
    """Keep the largest-magnitude entries; ties go to the lower index (comm.py:90-96)."""
    if isinstance(g, torch.Tensor) and g.is_cuda:
        gt = g.reshape(-1)
    else:
        gt = None
        g = np.asarray(g, dtype=np.float64)
    D = int(gt.numel()) if gt is not None else len(g)
    m = topk_count(D, cr)
    if D == 0:
        return SparseGradient(0, np.zeros(0, dtype=np.int64), np.zeros(0))
    if gt is None:
        gt = torch.from_numpy(g).to(_device())
    idx, val, _, _, _ = kernels.topk_gate(gt.contiguous(), m)
    return SparseGradient(D, idx[0], val[0])


@dataclass
class CompressionState:
    """Per-device gate state: EWMAs of squared norms plus decision counters (comm.py:99-119)."""

    cr: float
    delta: float
    ewma_factor: float = 0.9
    raw_gate: bool = False
    ewma_full: float = 0.0
    ewma_topk: float = 0.0
    initialized: bool = False
    n_compressed: int = 0
    n_uncompressed: int = 0

    def __post_init__(self):
        if not 0.0 < self.cr <= 1.0:
            raise ValueError("compression ratio must lie in (0, 1]")
        if self.delta < 0:
            raise ValueError("threshold delta must be non-negative")
        if not 0.0 < self.ewma_factor < 1.0:
            raise ValueError("ewma_factor must lie in (0, 1)")

    def to_record(self) -> np.ndarray:
        rec = np.zeros(1, dtype=_capi.GATE_STATE_DTYPE)
        for f in ("cr", "delta", "ewma_factor", "ewma_full", "ewma_topk", "n_compressed", "n_uncompressed"):
            rec[f] = getattr(self, f)
        rec["raw_gate"] = int(bool(self.raw_gate))
        rec["initialized"] = int(bool(self.initialized))
        return rec

    def load_record(self, rec) -> None:
        self.ewma_full = float(rec["ewma_full"])
        self.ewma_topk = float(rec["ewma_topk"])
        self.initialized = bool(rec["initialized"])
        self.n_compressed = int(rec["n_compressed"])
        self.n_uncompressed = int(rec["n_uncompressed"])


@dataclass
class GateDecision:
    compressed: bool
    payload: object
    ratio: float  # smoothed relative squared-norm loss used for the decision


def compression_gate(g, state: CompressionState) -> GateDecision:
    """Send Top-k iff its (smoothed) squared-norm loss stays within delta (comm.py:129-160).

    The Top-k selection, both squared norms and the EWMA/ratio/decision update run on the GPU
    (one fused launch sequence); the state's fields are updated in place from the device
    record, and the uncompressed payload aliases the input like the reference.
    """
    if isinstance(g, torch.Tensor) and g.is_cuda:
        gt = g.reshape(-1).contiguous()
        host = None
    else:
        host = np.asarray(g, dtype=np.float64)
        gt = None
    D = int(gt.numel()) if gt is not None else len(host)
    m = topk_count(D, state.cr)
    if D == 0:
        # empty gradient: both norms are exactly 0.0, the Top-k payload is empty
        rec = state.to_record()
        _gate_empty(rec[0])
        state.load_record(rec[0])
        return GateDecision(True, SparseGradient(0, np.zeros(0, dtype=np.int64), np.zeros(0)), 0.0)
    dev = _device()
    if gt is None:
        gt = torch.from_numpy(host).to(dev)
    st = kernels.gate_states_tensor(state.to_record(), dev)
    idx, val, norms2, decision, rho = kernels.topk_gate(gt, m, st)
    rec = kernels.gate_states_numpy(st)[0]
    compressed = bool(decision.item())
    ratio = float(rho.item())
    state.load_record(rec)
    if compressed:
        return GateDecision(True, SparseGradient(D, idx[0], val[0]), ratio)
    return GateDecision(False, host if host is not None else g, ratio)


def _gate_empty(rec) -> None:
    if not rec["initialized"]:
        rec["ewma_full"] = 0.0
        rec["ewma_topk"] = 0.0
        rec["initialized"] = 1
    else:
        f = float(rec["ewma_factor"])
        rec["ewma_full"] = f * float(rec["ewma_full"]) + (1.0 - f) * 0.0
        rec["ewma_topk"] = f * float(rec["ewma_topk"]) + (1.0 - f) * 0.0
    full = 0.0 if rec["raw_gate"] else float(rec["ewma_full"])
    kept = 0.0 if rec["raw_gate"] else float(rec["ewma_topk"])
    rho = 0.0 if full == 0.0 else abs(full - kept) / full
    if rho <= float(rec["delta"]):
        rec["n_compressed"] += 1
    else:
        rec["n_uncompressed"] += 1


def cnc_ratio(state: CompressionState) -> float:
    """Fraction of recorded decisions that sent the compressed payload (comm.py:163-168)."""
    total = state.n_compressed + state.n_uncompressed
    if total == 0:
        raise ValueError("no gate decisions recorded")
    return state.n_compressed / total


@dataclass
class VolumeStats:
    floats_sent: int = 0
    bytes_sent: int = 0


def account_volume(compressed: bool, dim: int, cr: float, stats: VolumeStats) -> VolumeStats:
    """Dense payloads count dim floats; sparse count m values + 4 B per index (comm.py:177-190)."""
    if compressed:
        m = topk_count(dim, cr)
        stats.floats_sent += m
        stats.bytes_sent += m * (FLOAT_BYTES + INDEX_BYTES)
    else:
        stats.floats_sent += dim
        stats.bytes_sent += dim * FLOAT_BYTES
    return stats


def payload_bytes(compressed: bool, dim: int, cr: float) -> int:
    """Wire size of one gradient payload (comm.py:193-197)."""
    if compressed:
        return topk_count(dim, cr) * (FLOAT_BYTES + INDEX_BYTES)
    return dim * FLOAT_BYTES


@dataclass
class LinkModel:
    latency: float
    bandwidth: float  # bytes per second

    def __post_init__(self):
        if self.latency < 0:
            raise ValueError("latency must be non-negative")
        if self.bandwidth <= 0:
            raise ValueError("bandwidth must be positive")


def comm_time(nbytes: float, link: LinkModel, n_devices: int) -> float:
    """Simulated ring-allreduce time latency + 2(n-1)/n * bytes/bandwidth (comm.py:212-219)."""
    if nbytes < 0:
        raise ValueError("byte count must be non-negative")
    if n_devices < 1:
        raise ValueError("need at least one device")
    ring = 2.0 * (n_devices - 1) / n_devices
    return link.latency + ring * nbytes / link.bandwidth
