"""Torch-tensor wrappers over the C-ABI (device memory and streams come from PyTorch).

Every function here launches the sm_100a kernels of ``libscadles_b200.so`` on the current
torch CUDA stream and returns without synchronising.  Inputs must be CUDA tensors; there is
no CPU path.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _capi

_GATE_BYTES = _capi.GATE_STATE_DTYPE.itemsize

# Kernel launches issued through this module (each C-ABI entry point launches a fixed
# sequence; see csrc/topk.cu and csrc/aggregate.cu).  bench.py reports the count.
LAUNCHES = {"n": 0}
# float32: sample+estimate (one clustered launch; two with SG_SAMPLE_EST=0), main + fallback,
# collect, resolve, write(+gate); float64: sample, estimate, main + fallback, collect, resolve, write
TOPK_LAUNCHES = {torch.float32: (1 if os.environ.get("SG_SAMPLE_EST", "1") != "0" else 2) + 2 + 1 + 1 + 1,
                 torch.float64: 2 + 2 + 1 + 1 + 1}


def _count(n: int) -> None:
    LAUNCHES["n"] += n


def _sparse_merge_launches(sparse_merge: int) -> int:
    """k_merge_ws + k_merge_own (one exits by payload density) unless the caller picked one."""
    return 2 if sparse_merge < 0 else 1


def require_cuda(t: torch.Tensor | None = None) -> None:
    if not torch.cuda.is_available():
        raise RuntimeError("scadles_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    if t is not None and not t.is_cuda:
        raise ValueError("expected a CUDA tensor")


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


class Workspace:
    """Grow-only device scratch buffers owned by the Python caller, one per (device, kind,
    slot).  ``slot`` separates calls that may run concurrently on different streams; ``kind``
    keeps the float32 Top-k workspace (which carries zero-initialised state between calls,
    see sg_topk_workspace_zero_bytes_f32) apart from every other user."""

    _cache: dict[tuple, torch.Tensor] = {}
    _keys: dict[tuple, tuple] = {}

    @classmethod
    def get(cls, nbytes: int, device: torch.device, slot: int = 0, kind: str = "scratch") -> torch.Tensor:
        idx = device.index if device.index is not None else torch.cuda.current_device()
        key = (idx, kind, slot)
        buf = cls._cache.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.zeros(max(int(nbytes), 256), dtype=torch.uint8, device=device)
            cls._cache[key] = buf
            cls._keys.pop(key, None)
        return buf

    @classmethod
    def get_topk(cls, nbytes: int, zero_bytes: int, plan_key: tuple, device: torch.device, slot: int = 0,
                 kind: str = "topk32"):
        """A float32 Top-k workspace: zero-filled when created and whenever the plan
        (k, dim, m) changes; every call leaves its zero-state region as it found it."""
        buf = cls.get(nbytes, device, slot, kind=kind)
        idx = device.index if device.index is not None else torch.cuda.current_device()
        key = (idx, kind, slot)
        if cls._keys.get(key) != plan_key:
            buf[:min(int(zero_bytes), buf.numel())].zero_()
            cls._keys[key] = plan_key
        return buf


def gate_states_tensor(states: np.ndarray, device: torch.device) -> torch.Tensor:
    """Pack a GATE_STATE_DTYPE record array into a device byte tensor."""
    raw = np.ascontiguousarray(states, dtype=_capi.GATE_STATE_DTYPE).view(np.uint8)
    return torch.from_numpy(raw.copy()).to(device)


def gate_states_numpy(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(_capi.GATE_STATE_DTYPE).copy()


MERGE_TILE = 4096


def merge_tiles(dim: int) -> int:
    return (dim + MERGE_TILE - 1) // MERGE_TILE


def topk_workspace_bytes(dtype: torch.dtype, k: int, dim: int, m: int, fused: bool = False) -> int:
    lib = _capi.load()
    if dtype == torch.float32:
        fn = lib.sg_topk_workspace_bytes_fused_f32 if fused else lib.sg_topk_workspace_bytes_f32
    else:
        fn = lib.sg_topk_workspace_bytes_f64
    return int(fn(k, dim, m))


# Launch-chain workspace budget: the chain keeps a candidate slot per element (8 B x k x D, e.g.
# 69 GB at D = 1e9, k = 8); above the budget the persistent variant (a ~2m-entry candidate
# pool, identical results) is taken instead.  Default: a quarter of the device's memory (45 GB
# on a B200); SG_TOPK_WS_BUDGET overrides (bytes).
TOPK_WS_BUDGET = int(os.environ["SG_TOPK_WS_BUDGET"]) if os.environ.get("SG_TOPK_WS_BUDGET") else None


def topk_ws_budget(device: torch.device | None = None) -> int:
    if TOPK_WS_BUDGET is not None:
        return TOPK_WS_BUDGET
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    return torch.cuda.get_device_properties(dev).total_memory // 4


def topk_use_fused(dtype: torch.dtype, k: int, dim: int, m: int, device: torch.device | None = None) -> bool:
    """The Top-k variant `topk_gate(fused=None)` takes: the launch chain (faster at every k
    and cr measured) unless its workspace exceeds the budget (topk_ws_budget)."""
    return dtype == torch.float32 and topk_workspace_bytes(dtype, k, dim, m) > topk_ws_budget(device)


def _topk_ws(dtype, k, dim, m, device, slot, fused):
    """float32 workspaces carry zero-state between calls: zero-filled when created and
    whenever the plan (k, dim, m) changes (sg_topk_workspace_zero_bytes_*)."""
    if dtype == torch.float32:
        lib = _capi.load()
        if fused:
            return Workspace.get_topk(topk_workspace_bytes(dtype, k, dim, m, True),
                                      int(lib.sg_topk_workspace_zero_bytes_fused_f32(k, dim, m)), (k, dim, m), device,
                                      slot, kind="topk32f")
        return Workspace.get_topk(topk_workspace_bytes(dtype, k, dim, m),
                                  int(lib.sg_topk_workspace_zero_bytes_f32(k, dim, m)), (k, dim, m), device, slot,
                                  kind="topk32")
    return Workspace.get(topk_workspace_bytes(dtype, k, dim, m), device, slot, kind="topk64")


def topk_gate(
    g: torch.Tensor,
    m: int,
    states: torch.Tensor | None = None,
    *,
    dim: int | None = None,
    out: tuple | None = None,
    tile_off: torch.Tensor | None = None,
    workspace_slot: int = 0,
    fused: bool | None = None,
):
    """Batched Top-k + norms (+ gate) over the rows of ``g`` ([k, ld] or [D]).

    ``workspace_slot`` selects a separate scratch buffer for calls issued concurrently on
    different streams.  ``fused`` (float32) takes the persistent one-kernel variant
    (sg_topk_gate_fused_f32) instead of the launch chain; the results are identical.  None
    (default): the chain unless its workspace exceeds the budget (topk_use_fused).

    Returns (idx int32 [k, m] (uint32 bits), val [k, m], norms2 f64 [k, 2], decision u8 [k],
    rho f64 [k]); decision/rho are None without ``states``.
    """
    require_cuda(g)
    if g.dtype not in (torch.float32, torch.float64):
        raise ValueError("gradient bucket must be float32 or float64")
    g2 = g.unsqueeze(0) if g.dim() == 1 else g
    if g2.dim() != 2 or g2.stride(1) != 1:
        raise ValueError("bucket must be [k, ld] with unit inner stride")
    k = g2.shape[0]
    ld = g2.stride(0) if k > 1 else g2.shape[1]
    D = int(dim if dim is not None else g2.shape[1])
    dev = g.device
    if out is None:
        idx = torch.empty((k, m), dtype=torch.int32, device=dev)
        val = torch.empty((k, m), dtype=g.dtype, device=dev)
        norms2 = torch.empty((k, 2), dtype=torch.float64, device=dev)
        decision = torch.empty(k, dtype=torch.uint8, device=dev) if states is not None else None
        rho = torch.empty(k, dtype=torch.float64, device=dev) if states is not None else None
    else:
        idx, val, norms2, decision, rho = out
    if states is not None and states.numel() != k * _GATE_BYTES:
        raise ValueError("one gate state per worker required")
    if fused is None:
        fused = topk_use_fused(g.dtype, k, D, m, g.device)
    fused = bool(fused) and g.dtype == torch.float32
    if topk_workspace_bytes(g.dtype, k, D, m, fused) == 0:
        raise ValueError("invalid top-k shape")
    lib = _capi.load()
    ws = _topk_ws(g.dtype, k, D, m, dev, workspace_slot, fused)
    args = [g2.data_ptr(), k, ld, D, m, idx.data_ptr(), val.data_ptr(), norms2.data_ptr(),
            _ptr(states), _ptr(decision), _ptr(rho)]
    if g.dtype == torch.float32:
        fn = lib.sg_topk_gate_fused_f32 if fused else lib.sg_topk_gate_f32
        st = fn(*args, _ptr(tile_off), ws.data_ptr(), ws.numel(), _stream())
    else:
        if tile_off is not None:
            raise ValueError("tile offsets are produced by the float32 path only")
        st = lib.sg_topk_gate_f64(*args, ws.data_ptr(), ws.numel(), _stream())
    _capi.check(st, "sg_topk_gate")
    _count(1 if fused else TOPK_LAUNCHES[g.dtype])
    return idx, val, norms2, decision, rho


def topk_stats(dtype: torch.dtype, k: int, dim: int, m: int, device: torch.device, workspace_slot: int = 0,
               fused: bool = False) -> np.ndarray:
    """Per-worker diagnostics of the last topk_gate call (synchronises): launch chain
    {candidates, boundary, fallback pass, slow resolve}; fused {candidates, boundary, estimate
    undershot, exact fallback}."""
    fused = bool(fused) and dtype == torch.float32
    ws = _topk_ws(dtype, k, dim, m, device, workspace_slot, fused)
    out = torch.zeros((k, 4), dtype=torch.int64, device=device)
    lib = _capi.load()
    if dtype == torch.float32:
        fn = lib.sg_topk_stats_fused_f32 if fused else lib.sg_topk_stats_f32
    else:
        fn = lib.sg_topk_stats_f64
    _capi.check(fn(k, dim, m, ws.data_ptr(), ws.numel(), out.data_ptr(), _stream()), "sg_topk_stats")
    return out.cpu().numpy()


def topk_phases(k: int, dim: int, m: int, device: torch.device, workspace_slot: int = 0) -> np.ndarray:
    """Fused float32 Top-k phase timestamps of the last call (ns, [k, nseg, 16]; synchronises)."""
    lib = _capi.load()
    nseg = int(lib.sg_topk_segments_f32(k, dim, m))
    ws = _topk_ws(torch.float32, k, dim, m, device, workspace_slot, True)
    out = torch.zeros(k * nseg * 16, dtype=torch.int64, device=device)
    _capi.check(lib.sg_topk_phases_f32(k, dim, m, ws.data_ptr(), ws.numel(), out.data_ptr(), out.numel(), _stream()),
                "sg_topk_phases_f32")
    return out.cpu().numpy().reshape(k, nseg, 16)


def gate_update(norms2: torch.Tensor, states: torch.Tensor):
    require_cuda(norms2)
    k = norms2.shape[0]
    decision = torch.empty(k, dtype=torch.uint8, device=norms2.device)
    rho = torch.empty(k, dtype=torch.float64, device=norms2.device)
    st = _capi.load().sg_gate_update(norms2.data_ptr(), k, states.data_ptr(), decision.data_ptr(), rho.data_ptr(), _stream())
    _capi.check(st, "sg_gate_update")
    _count(1)
    return decision, rho


def weighted_aggregate(
    weights,
    dim: int,
    *,
    compressed: torch.Tensor | None = None,
    dense: torch.Tensor | None = None,
    idx: torch.Tensor | None = None,
    val: torch.Tensor | None = None,
    row_ptr: torch.Tensor | None = None,
    tile_off: torch.Tensor | None = None,
    out: torch.Tensor | None = None,
    params: torch.Tensor | None = None,
    momentum_buf: torch.Tensor | None = None,
    lr: float = 0.0,
    momentum: float = 0.0,
    weight_decay: float = 0.0,
    first_step: bool = False,
    dtype: torch.dtype | None = None,
    sparse_merge: int = -1,
):
    """sum_j w_j * densify(payload_j) (+ optional fused momentum-SGD) on the GPU.

    ``sparse_merge``: all-sparse float32 merge kernel (-1 the device picks by density,
    0 k_merge_ws, 1 k_merge_own; identical results)."""
    w, wp = _capi.weights_ptr(np.asarray(weights, dtype=np.float64))
    nw = len(w)
    ref = next(t for t in (dense, val, params, out) if t is not None)
    require_cuda(ref)
    dt = dtype or ref.dtype
    dev = ref.device
    ld = 0
    if dense is not None:
        d2 = dense.unsqueeze(0) if dense.dim() == 1 else dense
        if d2.stride(-1) != 1:
            raise ValueError("dense rows need unit stride")
        ld = d2.stride(0) if d2.shape[0] > 1 else d2.shape[1]
        dense = d2
    if out is None and params is None:
        out = torch.empty(dim, dtype=dt, device=dev)
    ws = None
    nbytes = 0
    if compressed is not None and tile_off is None:
        nbytes = int(_capi.load().sg_aggregate_workspace_bytes(nw, dim))
        ws = Workspace.get(nbytes, dev)
    lib = _capi.load()
    common = (nw, wp, _ptr(compressed), _ptr(dense), ld, _ptr(idx), _ptr(val), _ptr(row_ptr), _ptr(tile_off), dim,
              _ptr(out), _ptr(params), _ptr(momentum_buf), float(lr), float(momentum), float(weight_decay),
              int(bool(first_step)))
    tail = (_ptr(ws), nbytes if ws is not None else 0, _stream())
    if dt == torch.float32:
        st = lib.sg_weighted_aggregate_f32(*common, int(sparse_merge), *tail)
    else:
        st = lib.sg_weighted_aggregate_f64(*common, *tail)
    _capi.check(st, "sg_weighted_aggregate")
    pipe = dt == torch.float32 and compressed is not None and params is not None
    _count(1 + (_sparse_merge_launches(sparse_merge) if pipe else 0) + (1 if ws is not None else 0))
    return out


class MergeLauncher:
    """The all-sparse float32 merge + fused SGD with every pointer bound once (the multi-GPU
    exchange launches it right after its one host synchronisation, so the host path between
    the decision read and the launch is a single ctypes call)."""

    def __init__(self, nw: int, dim: int, compressed, idx, val, row_ptr, tile_off, params, momentum_buf,
                 momentum: float, weight_decay: float, sparse_merge: int = -1):
        require_cuda(params)
        self._fn = _capi.load().sg_weighted_aggregate_f32
        self._sm = int(sparse_merge)
        self._nw, self._dim = nw, dim
        self._w = np.zeros(nw, dtype=np.float64)
        _, self._wp = _capi.weights_ptr(self._w)
        self._ptrs = (compressed.data_ptr(), idx.data_ptr(), val.data_ptr(), row_ptr.data_ptr(),
                      tile_off.data_ptr())
        self._p, self._b = params.data_ptr(), momentum_buf.data_ptr()
        self._mu, self._wd = float(momentum), float(weight_decay)

    def __call__(self, weights, lr: float, first_step: bool, out: torch.Tensor | None = None) -> None:
        self._w[:] = weights
        comp, idx, val, rp, toff = self._ptrs
        st = self._fn(self._nw, self._wp, comp, None, 0, idx, val, rp, toff, self._dim, _ptr(out), self._p,
                      self._b, float(lr), self._mu, self._wd, int(bool(first_step)), self._sm, None, 0, _stream())
        _capi.check(st, "sg_weighted_aggregate")
        _count(1 + _sparse_merge_launches(self._sm))


class PeerMergeLauncher:
    """sg_weighted_aggregate_peers_f32 with every pointer bound once: worker j's payload and
    merge offsets are read through raw device addresses (other GPUs' symmetric buffers)."""

    def __init__(self, dim: int, compressed: torch.Tensor, idx_ptrs, val_ptrs, off_ptrs, params, momentum_buf,
                 momentum: float, weight_decay: float, local_lo: int = 0, local_n: int = 0, sparse_merge: int = -1):
        require_cuda(params)
        nw = len(idx_ptrs)
        self._lo, self._ln, self._sm = int(local_lo), int(local_n), int(sparse_merge)
        self._fn = _capi.load().sg_weighted_aggregate_peers_f32
        self._nw, self._dim = nw, dim
        self._w = np.zeros(nw, dtype=np.float64)
        _, self._wp = _capi.weights_ptr(self._w)
        arr = ctypes.c_void_p * nw
        self._ip, self._vp, self._op = arr(*idx_ptrs), arr(*val_ptrs), arr(*off_ptrs)
        self._comp = compressed.data_ptr()
        self._p, self._b = params.data_ptr(), momentum_buf.data_ptr()
        self._mu, self._wd = float(momentum), float(weight_decay)

    def __call__(self, weights, lr: float, first_step: bool, out: torch.Tensor | None = None) -> None:
        self._w[:] = weights
        st = self._fn(self._nw, self._wp, self._comp, self._ip, self._vp, self._op, self._dim, _ptr(out),
                      self._p, self._b, float(lr), self._mu, self._wd, int(bool(first_step)), self._lo, self._ln,
                      self._sm, _stream())
        _capi.check(st, "sg_weighted_aggregate_peers_f32")
        _count(_sparse_merge_launches(self._sm))


class GuardedDenseLaunchers:
    """The dense side of a multi-GPU step over peer memory, O(D) NVLink bytes per rank:
    this rank's partial (sg_weighted_partial_f32) into its peer-mapped buffer, the
    position-sharded reduce of its slice over every rank's partial (sg_peer_reduce_slice_f32,
    written in place into its own buffer) and the all-gather of the reduced slices fused with
    momentum SGD (sg_peer_allgather_sgd_f32).  Guarded on the gathered decisions: no-ops when
    every worker compressed (``guard`` None: the dense workload, always run)."""

    def __init__(self, k: int, dim: int, ld: int, compressed, idx, val, row_ptr, tile_off, partial: torch.Tensor,
                 partial_ptrs, guard, params, momentum_buf, momentum: float, weight_decay: float, rank: int,
                 agg: torch.Tensor | None = None, agg_ptrs=None, flag_ptrs=None, mc_partial=None, mc_agg=None):
        lib = _capi.load()
        # NVLS mode (multicast addresses given): reduce in the switch + multicast broadcast
        self._mc = (mc_partial, mc_agg) if mc_partial else None
        # fused mode (flag_ptrs given): the whole dense side in one pipelined launch
        self._flags = (ctypes.c_void_p * len(flag_ptrs))(*flag_ptrs) if flag_ptrs is not None else None
        self._epoch = 0
        # push mode (agg given): the reduced slice is pushed into every rank's aggregate buffer
        # (sg_peer_reduce_push_f32) and each rank updates from its own copy
        self._agg = agg.data_ptr() if agg is not None else None
        self._aggp = (ctypes.c_void_p * len(agg_ptrs))(*agg_ptrs) if agg_ptrs is not None else None
        self._own = (ctypes.c_void_p * 1)(self._agg) if agg is not None else None
        self._part, self._red, self._ag = lib.sg_weighted_partial_f32, lib.sg_peer_reduce_slice_f32, \
            lib.sg_peer_allgather_sgd_f32
        self._k, self._dim, self._ld, self._rank = k, dim, ld, int(rank)
        self._w = np.zeros(k, dtype=np.float64)
        _, self._wp = _capi.weights_ptr(self._w)
        self._comp = _ptr(compressed)
        self._idx, self._val = _ptr(idx), _ptr(val)
        self._rp, self._toff = _ptr(row_ptr), _ptr(tile_off)
        self._partial = partial.data_ptr()
        self._pp = (ctypes.c_void_p * len(partial_ptrs))(*partial_ptrs)
        self._guard, self._gn = (guard.data_ptr(), guard.numel()) if guard is not None else (None, 0)
        self._p, self._b = params.data_ptr(), momentum_buf.data_ptr()
        self._mu, self._wd = float(momentum), float(weight_decay)
        self._ws = None

    def partial(self, local_weights, bucket: torch.Tensor) -> None:
        self._w[:] = local_weights
        if self._comp is None:  # dense workload: a weighted row fold, the same kernel family
            st = _capi.load().sg_weighted_aggregate_f32(
                self._k, self._wp, None, bucket.data_ptr(), self._ld, None, None, None, None, self._dim,
                self._partial, None, None, 0.0, 0.0, 0.0, 0, -1, None, 0, _stream())
            _capi.check(st, "sg_weighted_aggregate_f32")
            _count(1)
            return
        st = self._part(self._k, self._wp, self._comp, bucket.data_ptr(), self._ld, self._idx, self._val, self._rp,
                        self._toff, self._dim, self._partial, self._guard, self._gn, None, 0, _stream())
        _capi.check(st, "sg_weighted_partial_f32")
        _count(1)

    def dense_exchange(self, local_weights, bucket: torch.Tensor | None, lr: float, first_step: bool,
                       out: torch.Tensor | None = None) -> None:
        """sg_dense_exchange_f32: fold (bucket rows, or the partial already written) -> reduce ->
        push -> update, pipelined over chunks in one cooperative launch."""
        self._epoch += 1
        if bucket is not None:
            self._w[:] = local_weights
        st = _capi.load().sg_dense_exchange_f32(
            len(self._pp), self._rank, self._k, self._wp, _ptr(bucket), self._ld, self._dim, self._pp, self._aggp,
            self._flags, self._epoch, self._guard, self._gn, _ptr(out), self._p, self._b, float(lr), self._mu,
            self._wd, int(bool(first_step)), _stream())
        _capi.check(st, "sg_dense_exchange_f32")
        _count(1)

    def nvls_reduce_bcast(self) -> None:
        st = _capi.load().sg_nvls_reduce_bcast_f32(len(self._pp), self._rank, self._mc[0], self._mc[1], self._dim,
                                                   self._guard, self._gn, _stream())
        _capi.check(st, "sg_nvls_reduce_bcast_f32")
        _count(1)

    def reduce_push(self) -> None:
        st = _capi.load().sg_peer_reduce_push_f32(len(self._pp), self._pp, None, self._rank, self._guard, self._gn,
                                                  self._dim, self._aggp, _stream())
        _capi.check(st, "sg_peer_reduce_push_f32")
        _count(1)

    def local_sgd(self, lr: float, first_step: bool, out: torch.Tensor | None = None) -> None:
        """Momentum SGD from this rank's pushed copy of the aggregate (guarded like the rest)."""
        st = self._ag(1, self._own, 0, self._guard, self._gn, self._dim, _ptr(out), self._p, self._b,
                      float(lr), self._mu, self._wd, int(bool(first_step)), _stream())
        _capi.check(st, "sg_peer_allgather_sgd_f32")
        _count(1)

    def reduce_slice(self) -> None:
        st = self._red(len(self._pp), self._pp, None, self._rank, self._guard, self._gn, self._dim, self._partial,
                       _stream())
        _capi.check(st, "sg_peer_reduce_slice_f32")
        _count(1)

    def allgather_sgd(self, lr: float, first_step: bool, out: torch.Tensor | None = None) -> None:
        st = self._ag(len(self._pp), self._pp, self._rank, self._guard, self._gn, self._dim, _ptr(out), self._p, self._b,
                      float(lr), self._mu, self._wd, int(bool(first_step)), _stream())
        _capi.check(st, "sg_peer_allgather_sgd_f32")
        _count(1)


def multicast_copy(src: torch.Tensor, mc_dst: int) -> None:
    """Copy ``src`` (int32 words, a multiple of 4) to the multicast address ``mc_dst`` of a
    peer-mapped buffer: every rank's copy receives it (sg_multicast_copy_u32)."""
    require_cuda(src)
    _capi.check(_capi.load().sg_multicast_copy_u32(src.data_ptr(), int(mc_dst), src.numel(), _stream()),
                "sg_multicast_copy_u32")
    _count(1)


class PeerBarrier:
    """sg_peer_signal_wait with the ranks' flag arrays bound once: ``open(epoch, dec_ptrs, each,
    dst)`` -- the opening barrier of a peer step fused with the decision gather; ``guarded(guard)``
    -- a dense-side barrier skipped on the device when every worker compressed."""

    SLOTS = 2

    def __init__(self, rank: int, flag_ptrs, device: torch.device):
        self._lib = _capi.load()
        self._P, self._rank = len(flag_ptrs), int(rank)
        self._flags = (ctypes.c_void_p * len(flag_ptrs))(*flag_ptrs)
        self._counter = torch.zeros(1, dtype=torch.int32, device=device)

    def open(self, epoch: int, dec_ptrs, each: int, dst: torch.Tensor) -> None:
        src = (ctypes.c_void_p * len(dec_ptrs))(*dec_ptrs)
        _capi.check(self._lib.sg_peer_signal_wait(self._P, self._rank, self._flags, 0, int(epoch) & 0xFFFFFFFF or 1,
                                                  self._counter.data_ptr(), None, 0, src, int(each), dst.data_ptr(),
                                                  _stream()), "sg_peer_signal_wait")
        _count(1)

    def guarded(self, guard: torch.Tensor) -> None:
        _capi.check(self._lib.sg_peer_signal_wait(self._P, self._rank, self._flags, 1, 0, self._counter.data_ptr(),
                                                  guard.data_ptr(), guard.numel(), None, 0, None, _stream()),
                    "sg_peer_signal_wait")
        _count(1)


def gather_bytes(src_ptrs, each: int, dst: torch.Tensor) -> None:
    """dst[i*each:(i+1)*each] = bytes at device address src_ptrs[i] (peers' memory allowed)."""
    require_cuda(dst)
    arr = (ctypes.c_void_p * len(src_ptrs))(*src_ptrs)
    _capi.check(_capi.load().sg_gather_bytes(len(src_ptrs), arr, int(each), dst.data_ptr(), _stream()),
                "sg_gather_bytes")
    _count(1)


def sgd_momentum(params, momentum_buf, grad, lr, momentum, weight_decay, first_step):
    require_cuda(params)
    for name, t in (("grad", grad), ("momentum_buf", momentum_buf)):
        require_cuda(t)
        if t.dtype != params.dtype or t.numel() != params.numel():
            raise ValueError(f"{name} must match params in dtype and size "
                             f"({t.dtype}[{t.numel()}] vs {params.dtype}[{params.numel()}])")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
    if params.dtype not in (torch.float32, torch.float64) or not params.is_contiguous():
        raise ValueError("params must be a contiguous float32 or float64 CUDA tensor")
    lib = _capi.load()
    fn = lib.sg_sgd_momentum_f32 if params.dtype == torch.float32 else lib.sg_sgd_momentum_f64
    st = fn(params.data_ptr(), momentum_buf.data_ptr(), grad.data_ptr(), params.numel(), float(lr),
            float(momentum), float(weight_decay), int(bool(first_step)), _stream())
    _capi.check(st, "sg_sgd_momentum")
    _count(1)


def resolve_stream_rows(head, b, out_ptr, pool_ptr, pool_rows, total, out):
    st = _capi.load().sg_resolve_stream_rows(
        len(head), head.data_ptr(), b.data_ptr(), out_ptr.data_ptr(), pool_ptr.data_ptr(),
        pool_rows.data_ptr(), int(total), out.data_ptr(), _stream())
    _capi.check(st, "sg_resolve_stream_rows")
    _count(1)


def inject_rows(base_ptr, base_rows, senders, pick_ptr, picks, out_ptr, out_rows):
    n_dev = base_ptr.numel() - 1
    st = _capi.load().sg_inject_rows(
        n_dev, base_ptr.data_ptr(), base_rows.data_ptr(), senders.numel(), _ptr(senders) if senders.numel() else None,
        _ptr(pick_ptr) if senders.numel() else None, _ptr(picks) if picks.numel() else None,
        out_ptr.data_ptr(), out_rows.data_ptr(), _stream())
    _capi.check(st, "sg_inject_rows")
    _count(1)


def gather_batch(train_x, augment, train_y, rows, x_out, y_out):
    lib = _capi.load()
    fn = lib.sg_gather_batch_f64 if train_x.dtype == torch.float64 else lib.sg_gather_batch_f32
    st = fn(train_x.data_ptr(), _ptr(augment), _ptr(train_y), train_x.shape[1], rows.data_ptr(),
            rows.numel(), x_out.data_ptr(), _ptr(y_out), _stream())
    _capi.check(st, "sg_gather_batch")
    _count(1)
