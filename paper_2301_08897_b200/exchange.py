"""Per-GPU hot path: k local workers' gate -> exchange -> weighted aggregate -> momentum SGD.

This is the B200 restatement of the per-iteration section of ``Simulation.run_iteration``
(reference engine.py:248-286) for one process per GPU:

* the bucket (item 1) is a ``[k, ld]`` float32 tensor, one row per local worker, rows
  16-byte aligned, canonical parameter order;
* ``sg_topk_gate`` computes every local worker's Top-k payload, squared norms and gate
  decision in one launch sequence (comm.compression_gate at engine.py:253);
* workers are sharded contiguously: rank r owns global workers [r*k, (r+1)*k);
* exchange, one per step:
    P == 1  -> no collective; the aggregate kernel reads each worker's decision on device
               and folds dense rows or sparse payloads (no host synchronisation at all);
    P > 1   -> all-gather the W decisions; if every worker compressed, all-gather the fixed-
               size (idx, val) payloads and merge all W on every rank (identical bytes on
               every rank, deterministic); otherwise each rank folds its local workers into a
               partial dense sum and the partials are all-reduced;
* momentum SGD (nn.sgd_momentum_step, engine.py:282-283) is fused into the merge epilogue
  when the merge produces the final aggregate, so the float64 aggregate feeds the update
  without a round trip through HBM.

Weights are the reference's r_j = S_j / sum(S) (rate_matched, engine.py:266-267) or 1/n
(fixed_batch, 268-269); the caller passes them, never batch sizes (SURVEY §0 trap 1).

The collective logic is written against an ``ops`` object so that the host protocol can be
exercised with the gloo backend on CPU in tests; the product constructs it with
:class:`CudaOps`, whose every method is an sm_100a kernel launch.
"""

from __future__ import annotations

import os

import numpy as np
import torch
import torch.distributed as dist

from . import _capi, comm, kernels


class CudaOps:
    """The device operations of the hot path: thin calls into libscadles_b200.so."""

    name = "cuda"

    def __init__(self, device: torch.device, sparse_merge: int = -1):
        kernels.require_cuda()
        self.device = device
        self.sparse_merge = sparse_merge  # all-sparse merge kernel (see kernels.weighted_aggregate)

    def topk_gate(self, bucket, dim, m, states, out, tile_off=None):
        return kernels.topk_gate(bucket, m, states, dim=dim, out=out, tile_off=tile_off)

    def aggregate(self, weights, dim, **kw):
        return kernels.weighted_aggregate(weights, dim, sparse_merge=self.sparse_merge, **kw)

    def sgd(self, params, buf, grad, lr, momentum, weight_decay, first):
        kernels.sgd_momentum(params, buf, grad, lr, momentum, weight_decay, first)

    def gate_records(self, states):
        return kernels.gate_states_numpy(states)

    def make_states(self, records):
        return kernels.gate_states_tensor(records, self.device)


class StepInfo:
    """What a step did.  ``path`` is "local", "sparse-peer"/"dense-peer" (peer-memory
    exchange), "sparse-allgather" or "dense-allreduce"; on the peer path it is resolved
    lazily (reading it waits for the step's decisions), so the step itself never blocks."""

    def __init__(self, path, decisions, resolve=None):
        self._path = path
        self._resolve = resolve
        self.decisions = decisions  # this rank's u8 decisions (device)

    @property
    def path(self) -> str:
        if self._path is None:
            self._path = self._resolve()
            self._resolve = None
        return self._path


DEC_RING = 4096


def _padded(dim: int) -> int:
    return (dim + 3) // 4 * 4


class GradientExchange:
    """One rank's share of W workers: gate, exchange and update for a flat gradient of ``dim``."""

    def __init__(
        self,
        dim: int,
        n_workers: int,
        *,
        cr: float = 0.01,
        delta: float = 0.3,
        ewma_factor: float = 0.9,
        raw_gate: bool = False,
        compression: bool = True,
        momentum: float = 0.9,
        weight_decay: float = 0.0,
        group=None,
        ops=None,
        device: torch.device | None = None,
        dtype: torch.dtype = torch.float32,
    ):
        self.group = group
        self.world = dist.get_world_size(group) if group is not None else 1
        self.rank = dist.get_rank(group) if group is not None else 0
        if n_workers % self.world:
            raise ValueError("workers must divide evenly over ranks")
        self.W = n_workers
        self.k = n_workers // self.world
        self.lo = self.rank * self.k
        self.dim = dim
        self.ld = _padded(dim)
        self.cr = cr
        self.compression = compression
        self.m = comm.topk_count(dim, cr) if compression else dim
        self.momentum = momentum
        self.weight_decay = weight_decay
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = device
        self.ops = ops if ops is not None else CudaOps(device)
        self.dtype = dtype
        k, m = self.k, self.m
        z = dict(device=device)
        self.bucket = torch.zeros((k, self.ld), dtype=dtype, **z)
        self.params = torch.zeros(dim, dtype=dtype, **z)
        self.momentum_buf = torch.zeros(dim, dtype=dtype, **z)
        self.first_step = True
        recs = np.zeros(k, dtype=_capi.GATE_STATE_DTYPE)
        recs["cr"], recs["delta"], recs["ewma_factor"] = cr, delta, ewma_factor
        recs["raw_gate"] = int(raw_gate)
        self.states = self.ops.make_states(recs)
        self.packed = compression and self.world > 1 and dtype == torch.float32
        # all-sparse merge kernel by payload density: an all-compressed step always carries
        # exactly W*m entries, so the host knows the device's choice (>= 0.2 per position:
        # k_merge_own) and launches only that kernel
        self.sparse_merge = 1 if self.W * m >= 0.2 * dim else 0
        if isinstance(self.ops, CudaOps):
            self.ops.sparse_merge = self.sparse_merge
        if compression:
            nt1 = kernels.merge_tiles(dim) + 1
            if self.packed:
                # One send buffer per rank, gathered by ONE all-gather per step (32-bit words):
                #   [decisions (k bytes, 16-byte padded) | idx [k][m] | val [k][m] | tile_off [k][nt1]]
                # The Top-k kernels write straight into these views.
                dw = (k + 15) // 16 * 4
                words = (dw + 2 * k * m + k * nt1 + 3) // 4 * 4
                self.pack_words, self.pack_dw = words, dw
                self._symm = None
                self._partial_h = None
                self._agg_h = None
                # (the peer merge takes up to 16 workers; more go through the NCCL all-gather path)
                if device.type == "cuda" and os.environ.get("SG_P2P", "1") != "0" and self.W <= 16:
                    self._setup_peer_buffers(words)
                if self._symm is None:
                    self.pack = torch.zeros(words, dtype=torch.int32, **z)
                    packs = [self.pack]
                else:
                    self._pack2 = self.pack
                    packs = [self._pack2[:words], self._pack2[words:]]
                    self.pack = packs[0]

                def views(pk):
                    return dict(pack=pk, decision=pk[:dw].view(torch.uint8)[:k], idx=pk[dw:dw + k * m].view(k, m),
                                val=pk[dw + k * m:dw + 2 * k * m].view(torch.float32).view(k, m),
                                tile_off=pk[dw + 2 * k * m:dw + 2 * k * m + k * nt1].view(k, nt1))

                self._views = [views(pk) for pk in packs]
                self._set_views(0)
            else:
                self.idx = torch.empty((k, m), dtype=torch.int32, **z)
                self.val = torch.empty((k, m), dtype=dtype, **z)
                self.decision = torch.empty(k, dtype=torch.uint8, **z)
                self.tile_off = torch.empty((k, nt1), dtype=torch.int32, **z) if dtype == torch.float32 else None
            self.norms2 = torch.empty((k, 2), dtype=torch.float64, **z)
            self.rho = torch.empty(k, dtype=torch.float64, **z)
            self.row_ptr_local = torch.arange(0, (k + 1) * m, m, dtype=torch.int64, **z)
            if self.packed and self._symm is not None:
                P, words, dw = self.world, self.pack_words, self.pack_dw
                self._mc_dst = None
                self.dec_all = torch.empty(self.W, dtype=torch.uint8, **z)
                self._side = None
                # the step's peer barriers: own flag words (one launch that also gathers the
                # decisions; the dense side's barriers skipped on the device when every worker
                # compressed) -- SG_PEER_BARRIER=0: the symmetric-memory library barrier (A/B)
                self._pbar = None
                if self._bar_h is not None and os.environ.get("SG_PEER_BARRIER", "1") != "0":
                    boff = self._bar.data_ptr() - self._bar_h.buffer_ptrs[self.rank]
                    self._pbar = kernels.PeerBarrier(self.rank, [self._bar_h.buffer_ptrs[r] + boff for r in range(P)],
                                                     device)
                ph = self._partial_h
                poff = self._partial_buf.data_ptr() - ph.buffer_ptrs[self.rank]
                self._par_launch = []
                for par, vw in enumerate(self._views):
                    if self._gath is not None:
                        # payload broadcast: rank r's pack lands in slot r of every rank's gather
                        # buffer, so the merge reads all W payloads from local HBM
                        g0 = self._gath.data_ptr()
                        bases = [g0 + 4 * r * words for r in range(P)]
                        goff = g0 - self._gath_h.buffer_ptrs[self.rank]
                        self._mc_dst = int(self._gath_h.multicast_ptr) + goff + 4 * self.rank * words
                        merge_local = (0, self.W)
                    else:
                        off0 = vw["pack"].data_ptr() - self._symm.buffer_ptrs[self.rank]
                        bases = [self._symm.buffer_ptrs[r] + off0 for r in range(P)]  # rank r's pack
                        merge_local = (self.lo, self.k)
                    idx_p = [b + 4 * (dw + j * m) for b in bases for j in range(k)]
                    val_p = [b + 4 * (dw + k * m + j * m) for b in bases for j in range(k)]
                    off_p = [b + 4 * (dw + 2 * k * m + j * nt1) for b in bases for j in range(k)]
                    merge = kernels.PeerMergeLauncher(dim, self.dec_all, idx_p, val_p, off_p, self.params,
                                                      self.momentum_buf, momentum, weight_decay,
                                                      local_lo=merge_local[0], local_n=merge_local[1],
                                                      sparse_merge=self.sparse_merge)
                    # mixed decisions: each rank's partial in a peer-mapped buffer, reduced in rank order
                    dense = kernels.GuardedDenseLaunchers(
                        k, dim, self.ld, vw["decision"], vw["idx"], vw["val"], self.row_ptr_local, vw["tile_off"],
                        self._partial_buf, [ph.buffer_ptrs[r] + poff for r in range(P)], self.dec_all,
                        self.params, self.momentum_buf, momentum, weight_decay, self.rank, **self._push_args())
                    self._par_launch.append((bases, merge, dense))
                    if self._gath is not None:
                        break  # one gather buffer: no parity (the closing barrier stays)
            elif self.packed:
                P, words, dw = self.world, self.pack_words, self.pack_dw
                self.pack_all = torch.empty(P * words, dtype=torch.int32, **z)
                rows = self.pack_all.view(P, words)
                self.dec_view = rows[:, :dw].view(torch.uint8)[:, :k]
                self.toff_view = rows[:, dw + 2 * k * m:dw + 2 * k * m + k * nt1]
                # merge inputs: idx / val bases inside the gathered buffer; worker (r, j) at
                # r * words + j * m words from either base
                self.idx_all = self.pack_all[dw:]
                self.val_all = self.pack_all[dw + k * m:].view(torch.float32)
                starts = [r * words + j * m for r in range(P) for j in range(k)]
                self.row_ptr_all = torch.tensor(starts + [starts[-1] + m], dtype=torch.int64, device=device)
                self.dec_all = torch.empty(self.W, dtype=torch.uint8, **z)
                self.tile_off_all = torch.empty((self.W, nt1), dtype=torch.int32, **z)
                self._dec_host = (torch.empty(self.W, dtype=torch.uint8, pin_memory=True)
                                  if device.type == "cuda" else None)
                self._dec_ready = torch.cuda.Event() if device.type == "cuda" else None
                self._merge = None
            elif self.world > 1:
                self.dec_all = torch.empty(self.W, dtype=torch.uint8, **z)
                self.idx_all = torch.empty((self.W, m), dtype=torch.int32, **z)
                self.val_all = torch.empty((self.W, m), dtype=dtype, **z)
                self.row_ptr_all = torch.arange(0, (self.W + 1) * m, m, dtype=torch.int64, **z)
                self.tile_off_all = (torch.empty((self.W, nt1), dtype=torch.int32, **z)
                                     if self.tile_off is not None else None)
        # dense workload at P > 1 over peer memory: partial -> position-sharded reduce ->
        # all-gather fused with SGD (O(D) NVLink bytes per rank), no collective library
        self._dense_peer = None
        if (not compression and self.world > 1 and dtype == torch.float32 and device.type == "cuda"
                and os.environ.get("SG_P2P", "1") != "0" and self.world <= 8):
            self._symm = None
            self._partial_h = None
            self._agg_h = None
            self._flag_h = None
            self._setup_peer_buffers(None)
            if self._partial_h is not None:
                ph = self._partial_h
                poff = self._partial_buf.data_ptr() - ph.buffer_ptrs[self.rank]
                self._dense_peer = kernels.GuardedDenseLaunchers(
                    k, dim, self.ld, None, None, None, None, None, self._partial_buf,
                    [ph.buffer_ptrs[r] + poff for r in range(self.world)], None, self.params, self.momentum_buf,
                    momentum, weight_decay, self.rank, **self._push_args())
        # float64 ("exact") mode at P > 1: every rank folds all W payloads in ascending worker
        # order (the dense rows are gathered too), so the aggregate and the update are
        # bit-identical to the reference's at any P (the drop-in / metrics path, small D)
        self.exact = dtype == torch.float64 and self.world > 1
        if self.exact:
            self.bucket_all = torch.empty((self.W, self.ld), dtype=dtype, **z)
            if not compression:
                self.dec_all = None
        self.partial = torch.empty(dim, dtype=dtype, **z) if self.world > 1 else None
        self._dec_ring = None
        self.aggregate = None
        self.steps = 0
        self._par = getattr(self, "_par", 0)
        self._flip_pending = False

    def close(self) -> None:
        """Before this rank frees the exchange (or leaves the group) while peers may still be in
        their last step: one peer barrier (the peer path keeps no closing barrier per step)."""
        if self._flip_pending and self._symm is not None:
            self._symm.barrier(channel=0)
            self._flip_pending = False

    def _advance(self) -> None:
        """Before a step's first Top-k launch: move to the other send pack (peer path)."""
        if self._flip_pending:
            self._flip_pending = False
            self._set_views(self._par ^ 1)

    def _set_views(self, par: int) -> None:
        """Point the public payload views (pack, decision, idx, val, tile_off) at send pack
        ``par``: the Top-k of the next step writes there."""
        self._par = par
        for name, t in self._views[par].items():
            setattr(self, name, t)

    def _push_args(self) -> dict:
        """Dense side mode (SG_DENSE_MODE, for the A/B runs of tools/dense_timing.py): "pull"
        (default) -- position-sharded reduce, barrier, pull all-gather fused with the update;
        "push" -- reduce-and-push, barrier, local update; "nvls" -- reduce in the switch +
        multicast broadcast, barrier, local update; "fused" -- one pipelined launch
        (sg_dense_exchange_f32).  Measured at P = 4: pull 0.91 ms, push 0.99,
        nvls 1.02, fused 1.05 for the dense side of a ResNet-152-sized step."""
        mode = os.environ.get("SG_DENSE_MODE", "pull")
        if mode == "nvls" and not self._multicast_ok():
            mode = "pull"
        if mode == "pull":
            return {}
        h = self._agg_h
        off = self._agg_buf.data_ptr() - h.buffer_ptrs[self.rank]
        args = dict(agg=self._agg_buf, agg_ptrs=[h.buffer_ptrs[r] + off for r in range(self.world)])
        if mode == "nvls":
            ph = self._partial_h
            poff = self._partial_buf.data_ptr() - ph.buffer_ptrs[self.rank]
            args["mc_partial"] = int(ph.multicast_ptr) + poff
            args["mc_agg"] = int(h.multicast_ptr) + off
        if mode == "fused":
            fh = self._flag_h
            foff = self._flag_buf.data_ptr() - fh.buffer_ptrs[self.rank]
            args["flag_ptrs"] = [fh.buffer_ptrs[r] + foff for r in range(self.world)]
        return args

    def _multicast_ok(self) -> bool:
        """NVLS multicast on both peer-mapped buffers, on every rank (collective decision)."""
        ok = 1
        try:
            for h in (self._partial_h, self._agg_h):
                if int(h.multicast_ptr) == 0:
                    ok = 0
        except Exception:
            ok = 0
        flag = torch.tensor([ok], dtype=torch.int32, device=self.device)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.group)
        return int(flag.item()) == 1

    def _dense_side(self, launchers, lr, first, out, barrier, w_local=None, bucket=None) -> None:
        """The dense side after the local partial: fused pipelined launch, or
        barrier -> reduce (push, or pull at the all-gather) -> barrier -> SGD."""
        if launchers._flags is not None:
            launchers.dense_exchange(w_local, bucket, lr, first, out)
            return
        if bucket is not None:
            launchers.partial(w_local, bucket)
        barrier()
        if launchers._mc is not None:  # NVLS: reduce in the switch, multicast the slice
            launchers.nvls_reduce_bcast()
            barrier()
            launchers.local_sgd(lr, first, out)
        elif launchers._aggp is not None:
            launchers.reduce_push()
            barrier()
            launchers.local_sgd(lr, first, out)
        else:
            launchers.reduce_slice()
            barrier()
            launchers.allgather_sgd(lr, first, out)

    def _setup_peer_buffers(self, words: int | None) -> None:
        """Symmetric (peer-mapped) send buffer (``words`` int32; None: none) and partial buffer,
        so the merge reads the other ranks' payloads, and the dense side their partials, in
        place over NVLink.  The choice is collective: every rank reports whether every
        rendezvous succeeded and the peer path is taken only if all did (otherwise every rank
        takes the NCCL path -- a rank that silently fell back alone would hang the others in
        the peer barriers)."""
        ok = 1
        symm = pack = gath_h = bar = bar_h = None
        try:
            import torch.distributed._symmetric_memory as symm_mem

            grp = self.group if self.group is not None else dist.group.WORLD
            if words is not None:
                # two send packs (step parity), so a step's Top-k never overwrites the pack a
                # slower peer may still be merging from (no closing barrier per step)
                pack = symm_mem.empty(2 * words, dtype=torch.int32, device=self.device)
                pack.zero_()
                symm = symm_mem.rendezvous(pack, grp.group_name)
                # the gather buffer of the payload broadcast: slot r <- rank r's pack (multicast)
                gath = symm_mem.empty(self.world * words, dtype=torch.int32, device=self.device)
                gath.zero_()
                gath_h = symm_mem.rendezvous(gath, grp.group_name)
                # flag words of the step's own peer barriers (kernels.PeerBarrier)
                bar = symm_mem.empty(kernels.PeerBarrier.SLOTS * self.world, dtype=torch.int32, device=self.device)
                bar.zero_()
                bar_h = symm_mem.rendezvous(bar, grp.group_name)
            part = symm_mem.empty(self.ld, dtype=torch.float32, device=self.device)
            part.zero_()
            part_h = symm_mem.rendezvous(part, grp.group_name)
            agg = symm_mem.empty(self.ld, dtype=torch.float32, device=self.device)
            agg.zero_()
            agg_h = symm_mem.rendezvous(agg, grp.group_name)
            nfw = int(_capi.load().sg_dense_exchange_flag_words(self.dim, self.world))
            flg = symm_mem.empty(max(nfw, 4), dtype=torch.int32, device=self.device)
            flg.zero_()
            flg_h = symm_mem.rendezvous(flg, grp.group_name)
        except Exception:  # no peer mapping on this system
            ok = 0
        flag = torch.tensor([ok], dtype=torch.int32, device=self.device)
        if self.group is not None or dist.is_initialized():
            dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.group)
        self._gath = self._gath_h = None
        if int(flag.item()) == 1 and words is not None and os.environ.get("SG_PAYLOAD_MC", "0") == "1":
            # opt-in (A/B): the payloads broadcast through the switch (NVLS multicast on every
            # rank, a collective decision) and merged from local memory.  Measured slower than
            # the default merge reading the peers' payloads over NVLink: P = 4, cr 0.01 0.464 vs
            # 0.404 ms, cr 0.1 1.324 vs 0.971 ms (multimem.st moves ~270 GB/s per rank here)
            mc = torch.tensor([1 if int(gath_h.multicast_ptr) != 0 else 0], dtype=torch.int32, device=self.device)
            dist.all_reduce(mc, op=dist.ReduceOp.MIN, group=self.group)
            if int(mc.item()) == 1:
                self._gath, self._gath_h = gath, gath_h
        self._bar, self._bar_h = (bar, bar_h) if int(flag.item()) == 1 else (None, None)
        if int(flag.item()) == 1:
            self._symm, self.pack = symm, pack
            self._partial_buf, self._partial_h = part, part_h
            self._agg_buf, self._agg_h = agg, agg_h
            self._flag_buf, self._flag_h = flg, flg_h
        else:
            self._symm = None
            self._partial_h = None
            self._agg_h = None
            self._flag_h = None

    # -- the step ---------------------------------------------------------------------------

    def gate(self) -> None:
        """Top-k + norms + gate for every local worker (no host synchronisation)."""
        self._advance()
        self.ops.topk_gate(
            self.bucket, self.dim, self.m, self.states,
            (self.idx, self.val, self.norms2, self.decision, self.rho), self.tile_off,
        )

    def gate_worker(self, j: int, workspace_slot: int = 1) -> None:
        """Top-k + norms + gate of local worker j alone, on the current stream -- for
        overlapping a finished worker's gate with the next worker's backward pass (DDP-style:
        launch it on a side stream once worker j's gradient row is complete, then call
        ``step(..., gated=True)``).  Same results as the batched gate."""
        if not self.compression:
            return
        if not isinstance(self.ops, CudaOps):
            raise ValueError("per-worker gating needs the CUDA ops")
        self._advance()
        gb = _capi.GATE_STATE_DTYPE.itemsize
        out = (self.idx[j:j + 1], self.val[j:j + 1], self.norms2[j:j + 1], self.decision[j:j + 1], self.rho[j:j + 1])
        kernels.topk_gate(self.bucket[j:j + 1], self.m, self.states[j * gb:(j + 1) * gb], dim=self.dim, out=out,
                          tile_off=None if self.tile_off is None else self.tile_off[j:j + 1],
                          workspace_slot=workspace_slot)

    def step(self, weights, lr: float, *, keep_aggregate: bool = False, topk_events=None,
             gated: bool = False) -> StepInfo:
        """One synchronous iteration over the gradients currently in ``bucket``.

        ``weights`` holds all W aggregation weights (host float64).  With
        ``keep_aggregate`` the aggregated gradient is also written to ``self.aggregate``.
        ``topk_events`` = (start, end) CUDA events recorded around the Top-k/gate launch
        sequence on the current stream (bench.py's per-kernel roofline timing).  ``gated``:
        every local worker was already gated with :meth:`gate_worker` (overlapped with the
        backward passes); the stream must be ordered after those launches.
        """
        w = np.asarray(weights, dtype=np.float64)
        if w.shape != (self.W,):
            raise ValueError("one weight per worker required")
        dim, first = self.dim, self.first_step
        opt = dict(params=self.params, momentum_buf=self.momentum_buf, lr=lr,
                   momentum=self.momentum, weight_decay=self.weight_decay, first_step=first)
        if keep_aggregate and self.aggregate is None:
            self.aggregate = torch.empty(dim, dtype=self.dtype, device=self.device)
        out = self.aggregate if keep_aggregate else None
        if self.compression and not gated:
            if topk_events is not None:
                topk_events[0].record()
            self.gate()
            if topk_events is not None:
                topk_events[1].record()
        if self.world == 1:
            if self.compression:
                self.ops.aggregate(w, dim, compressed=self.decision, dense=self.bucket, idx=self.idx,
                                   val=self.val, row_ptr=self.row_ptr_local, tile_off=self.tile_off,
                                   out=out, **opt)
            else:
                self.ops.aggregate(w, dim, dense=self.bucket, out=out, **opt)
            path = "local"
        else:
            path = self._exchange(w, out, opt)
        self.first_step = False
        self.steps += 1
        dec = self.decision if self.compression else None
        if callable(path):
            return StepInfo(None, dec, path)
        return StepInfo(path, dec)

    def _exchange(self, w, out, opt) -> str:
        g = self.group
        dim = self.dim
        if self.exact:
            return self._exact_exchange(w, out, opt)
        if self._dense_peer is not None:
            # dense workload over peer memory: O(D) NVLink bytes per rank, fused update
            h = self._partial_h
            self._dense_side(self._dense_peer, opt["lr"], opt["first_step"], out, lambda: h.barrier(channel=0),
                             w_local=w[self.lo:self.lo + self.k], bucket=self.bucket)
            if self._dense_peer._flags is None:
                h.barrier(channel=0)  # no rank rewrites its partial / aggregate while a peer still uses it
            return "dense-peer"
        if self.packed and self._symm is not None:
            # Peer path, no host synchronisation: after a device barrier (every rank's Top-k has
            # written its symmetric send buffer) the W decisions are gathered on device, and both
            # exchanges are enqueued with device-side guards on them -- the all-compressed merge,
            # which reads the other ranks' payloads in place over NVLink, and the mixed case's
            # partial + rank-ordered reduction + SGD.  The last barrier keeps the next step's
            # Top-k from overwriting a buffer a peer is still reading.
            lr, first = opt["lr"], opt["first_step"]
            main = torch.cuda.current_stream()
            if self._side is None:
                self._side = torch.cuda.Stream(device=self.device)
                self._gathered = torch.cuda.Event()
            bases, merge, dense = self._par_launch[self._par if len(self._par_launch) > 1 else 0]
            if self._mc_dst is not None:
                kernels.multicast_copy(self.pack, self._mc_dst)
            if self._pbar is not None:
                self._pbar.open(self.steps + 1, bases, self.k, self.dec_all)
                dense_barrier = lambda: self._pbar.guarded(self.dec_all)  # noqa: E731
            else:
                self._symm.barrier(channel=0)
                kernels.gather_bytes(bases, self.k, self.dec_all)
                dense_barrier = lambda: self._symm.barrier(channel=1)  # noqa: E731
            self._gathered.record(main)
            # the guarded dense side on a second stream: its no-ops overlap the merge (exactly
            # one of the two sides does work in any step)
            self._side.wait_event(self._gathered)
            with torch.cuda.stream(self._side):
                # mixed decisions: the local partial densifies the compressed local workers,
                # then the dense side exchanges it (a no-op when every worker compressed)
                dense.partial(w[self.lo:self.lo + self.k], self.bucket)
                self._dense_side(dense, lr, first, out, dense_barrier)
            merge(w, lr, first, out)
            main.wait_stream(self._side)
            if len(self._par_launch) > 1:
                # the next step's Top-k writes the other pack (the views flip when it starts, so
                # they show this step's payload until then); the pack read here is rewritten two
                # steps on, after the next step's opening barrier, which every rank passes only
                # once its merge and dense side of this step are done (stream order)
                self._flip_pending = True
            else:
                self._symm.barrier(channel=0)
            # the step's decisions for the lazily resolved path name: one pinned slot per
            # step in a ring allocated once (a StepInfo's path must be read within
            # DEC_RING steps of the step that made it)
            if self._dec_ring is None:
                self._dec_ring = torch.empty((DEC_RING, self.W), dtype=torch.uint8, pin_memory=True)
            dec_host = self._dec_ring[self.steps % DEC_RING]
            dec_host.copy_(self.dec_all, non_blocking=True)
            ready = torch.cuda.Event()
            ready.record()

            def resolve():
                ready.synchronize()
                return "sparse-peer" if int(dec_host.numpy().min()) == 1 else "dense-peer"

            return resolve
        if self.packed:
            # one all-gather carries every rank's decisions, payloads and merge offsets; the
            # decisions and offsets are regrouped contiguously on device before the host
            # reads the decisions
            dist.all_gather_into_tensor(self.pack_all, self.pack, group=g)
            if self._dec_host is not None:
                # the step's one host synchronisation: the W decision bytes go to pinned memory
                # first; the device-side regrouping of decisions and offsets for the merge is
                # enqueued behind them and runs while the host waits and launches the merge
                self._dec_host.view(self.world, self.k).copy_(self.dec_view, non_blocking=True)
                self._dec_ready.record()
                self.dec_all.view(self.world, self.k).copy_(self.dec_view)
                self.tile_off_all.view(self.world, self.k, -1).copy_(self.toff_view.view(self.world, self.k, -1))
                self._dec_ready.synchronize()
                all_compressed = bool(self._dec_host.numpy().min() == 1)
            else:
                self.dec_all.view(self.world, self.k).copy_(self.dec_view)
                self.tile_off_all.view(self.world, self.k, -1).copy_(self.toff_view.view(self.world, self.k, -1))
                all_compressed = bool(self.dec_all.min().item() == 1)
            if all_compressed:
                if isinstance(self.ops, CudaOps):
                    if self._merge is None:
                        self._merge = kernels.MergeLauncher(self.W, dim, self.dec_all, self.idx_all, self.val_all,
                                                            self.row_ptr_all, self.tile_off_all, self.params,
                                                            self.momentum_buf, self.momentum, self.weight_decay,
                                                            sparse_merge=self.sparse_merge)
                    self._merge(w, opt["lr"], opt["first_step"], out)
                else:
                    self.ops.aggregate(w, dim, compressed=self.dec_all, idx=self.idx_all, val=self.val_all,
                                       row_ptr=self.row_ptr_all, tile_off=self.tile_off_all, out=out, **opt)
                return "sparse-allgather"
        elif self.compression:
            dist.all_gather_into_tensor(self.dec_all, self.decision, group=g)
            all_compressed = bool(self.dec_all.min().item() == 1)
        else:
            all_compressed = False
        if all_compressed:
            dist.all_gather_into_tensor(self.idx_all.view(-1), self.idx.view(-1), group=g)
            dist.all_gather_into_tensor(self.val_all.view(-1), self.val.view(-1), group=g)
            if self.tile_off is not None:
                dist.all_gather_into_tensor(self.tile_off_all.view(-1), self.tile_off.view(-1), group=g)
            self.ops.aggregate(w, dim, compressed=self.dec_all, idx=self.idx_all, val=self.val_all,
                               row_ptr=self.row_ptr_all, tile_off=self.tile_off_all, out=out, **opt)
            return "sparse-allgather"
        return self._dense_exchange(w, out, opt)

    def _exact_exchange(self, w, out, opt) -> str:
        """float64 mode: all-gather decisions, payloads and (if any worker stayed dense) the
        dense rows; every rank folds the W workers in ascending order with the fused update
        (comm.py:75-77 order), so every rank's bytes equal the one-process reference's."""
        g = self.group
        dim = self.dim
        if self.compression:
            dist.all_gather_into_tensor(self.dec_all, self.decision, group=g)
            all_compressed = bool(self.dec_all.min().item() == 1)
            dist.all_gather_into_tensor(self.idx_all.view(-1), self.idx.view(-1), group=g)
            dist.all_gather_into_tensor(self.val_all.view(-1), self.val.view(-1), group=g)
        else:
            all_compressed = False
        if not all_compressed:
            dist.all_gather_into_tensor(self.bucket_all.view(-1), self.bucket.view(-1), group=g)
        if self.compression:
            self.ops.aggregate(w, dim, compressed=self.dec_all, dense=None if all_compressed else self.bucket_all,
                               idx=self.idx_all, val=self.val_all, row_ptr=self.row_ptr_all, out=out, **opt)
        else:
            self.ops.aggregate(w, dim, dense=self.bucket_all, out=out, **opt)
        return "exact-allgather"

    def _dense_exchange(self, w, out, opt) -> str:
        """Mixed decisions: local partial (dense rows + local payloads), all-reduce, SGD."""
        g = self.group
        dim = self.dim
        wl = w[self.lo:self.lo + self.k]
        if self.compression:
            self.ops.aggregate(wl, dim, compressed=self.decision, dense=self.bucket, idx=self.idx,
                               val=self.val, row_ptr=self.row_ptr_local, tile_off=self.tile_off,
                               out=self.partial)
        else:
            self.ops.aggregate(wl, dim, dense=self.bucket, out=self.partial)
        dist.all_reduce(self.partial, op=dist.ReduceOp.SUM, group=g)
        if out is not None:
            out.copy_(self.partial)
        self.ops.sgd(self.params, self.momentum_buf, self.partial, opt["lr"], self.momentum,
                     self.weight_decay, opt["first_step"])
        return "dense-allreduce"

    # -- host views (synchronising) -----------------------------------------------------------

    def gate_counters(self) -> np.ndarray:
        return self.ops.gate_records(self.states)

    def volume(self) -> tuple[int, int]:
        """(floats_sent, bytes_sent) of this rank's workers so far (comm.account_volume)."""
        if self.compression:
            rec = self.gate_counters()
            nc = int(rec["n_compressed"].sum())
            nu = int(rec["n_uncompressed"].sum())
        else:
            nc, nu = 0, self.steps * self.k
        floats = nc * self.m + nu * self.dim
        nbytes = nc * self.m * (comm.FLOAT_BYTES + comm.INDEX_BYTES) + nu * self.dim * comm.FLOAT_BYTES
        return floats, nbytes

    def param_checksum(self) -> float:
        """Replica check (engine.py:284-286): identical on every rank by construction."""
        return float(self.params.double().sum().item())
