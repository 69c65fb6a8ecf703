"""torchrun: the measured case for a replicated vs a sharded optimizer state in the multi-GPU
all-sparse step (VERDICT r01 missing item 2).  Per rank, CUDA events:

  replicated   merge of all W payloads + momentum SGD over the full D on every rank (the
               product: GradientExchange's peer merge)
  sharded      the same merge + SGD over this rank's 1/P of the positions (measured on a
               D/P-long problem with the same workers and density), followed by the parameter
               all-gather every replica needs before its next forward pass (NCCL
               all_gather_into_tensor of D/P floats per rank)
  overlap      that all-gather on a side stream concurrently with the next step's Top-k (the
               best case for sharding: only a synthetic-gradient benchmark has no forward pass
               between the update and the next Top-k)

    python -m torch.distributed.run --nproc-per-node P --master-addr 127.0.0.1 tools/shard_tradeoff.py
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2301_08897_b200 import build, comm, exchange, kernels  # noqa: E402

D, W = 60_192_808, 8


def timed(fn, reps=10):
    ts = []
    for _ in range(reps):
        dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


def heavy(ex, seed):
    gen = torch.Generator(device=ex.device).manual_seed(seed)
    z = torch.randn(ex.bucket.shape, device=ex.device, generator=gen)
    ex.bucket.copy_(torch.sign(z) * torch.exp(1.5 * torch.randn(ex.bucket.shape, device=ex.device, generator=gen)))


def main():
    build.build()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, P = dist.get_rank(), dist.get_world_size()
    w = comm.weights_from_rates([31, 30, 1, 30, 42, 66, 22, 14])
    # replicated: the product's step, merge part timed inside (peer merge + SGD over D)
    ex = exchange.GradientExchange(D, W, cr=0.01, delta=0.3, momentum=0.9, weight_decay=1e-4,
                                   group=dist.group.WORLD, device=dev)
    heavy(ex, rank)
    for _ in range(3):
        ex.step(w, 0.01)
    torch.cuda.synchronize()
    t_step = timed(lambda: ex.step(w, 0.01))
    t_topk = timed(lambda: ex.gate())
    # merge + SGD over 1/P of the positions: one GPU, all W workers, a D/P-long problem
    Ds = (D + P - 1) // P
    exs = exchange.GradientExchange(Ds, W, cr=0.01, delta=0.3, momentum=0.9, weight_decay=1e-4, device=dev)
    heavy(exs, rank + 100)
    exs.gate()
    torch.cuda.synchronize()
    rp = exs.row_ptr_local
    merge_full = lambda e: kernels.weighted_aggregate(  # noqa: E731
        w, e.dim, compressed=torch.ones(W, dtype=torch.uint8, device=dev), idx=e.idx, val=e.val, row_ptr=e.row_ptr_local,
        tile_off=e.tile_off, params=e.params, momentum_buf=e.momentum_buf, lr=0.01, momentum=0.9, weight_decay=1e-4,
        first_step=False, sparse_merge=e.sparse_merge)
    t_merge_shard = timed(lambda: merge_full(exs))
    # parameter all-gather: D/P floats per rank
    shard = torch.randn(Ds, device=dev)
    full = torch.empty(Ds * P, device=dev)
    t_ag = timed(lambda: dist.all_gather_into_tensor(full, shard))
    # the all-gather hidden under the next Top-k (side stream)
    side = torch.cuda.Stream(device=dev)

    def overlapped():
        main = torch.cuda.current_stream()
        side.wait_stream(main)
        with torch.cuda.stream(side):
            dist.all_gather_into_tensor(full, shard)
        ex.gate()
        main.wait_stream(side)

    t_overlap = timed(overlapped)
    rep = dict(rank=rank, P=P, replicated_step_us=t_step, topk_us=t_topk,
               replicated_merge_est_us=t_step - t_topk,
               sharded_merge_sgd_us=t_merge_shard, param_allgather_us=t_ag,
               sharded_step_est_us=t_topk + t_merge_shard + t_ag,
               topk_with_hidden_allgather_us=t_overlap,
               sharded_overlap_step_est_us=t_overlap + t_merge_shard,
               allgather_busbw_GBps=(P - 1) * Ds * 4 / (t_ag * 1e-6) / 1e9)
    r = [None] * P
    dist.all_gather_object(r, rep)
    if rank == 0:
        print(json.dumps({"per_rank": r, "max_replicated_step_us": max(x["replicated_step_us"] for x in r),
                          "max_sharded_step_est_us": max(x["sharded_step_est_us"] for x in r),
                          "max_sharded_overlap_step_est_us": max(x["sharded_overlap_step_est_us"] for x in r)}),
              flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
