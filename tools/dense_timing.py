"""torchrun: per-phase device time of the dense side of a multi-GPU step over peer memory
(the dense workload: partial -> barrier -> position-sharded reduce -> barrier -> all-gather +
SGD -> barrier), CUDA events on the compute stream, median of 10 steps, plus NCCL's
all_reduce of the same buffer for reference (busbw).

    python -m torch.distributed.run --nproc-per-node P --master-addr 127.0.0.1 tools/dense_timing.py
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
from paper_2301_08897_b200 import build, comm, exchange  # noqa: E402

D, W = 60_192_808, 8


def main():
    build.build()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, P = dist.get_rank(), dist.get_world_size()
    ex = exchange.GradientExchange(D, W, compression=False, momentum=0.9, weight_decay=1e-4,
                                   group=dist.group.WORLD, device=dev)
    ex.bucket.normal_()
    w = comm.weights_from_rates([31, 30, 1, 30, 42, 66, 22, 14])
    dp, h = ex._dense_peer, ex._partial_h
    for _ in range(3):
        ex.step(w, 0.01)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
    rows = []
    wl = w[ex.lo:ex.lo + ex.k]
    if dp._flags is not None:  # fused: one pipelined launch for the whole dense side
        ts = []
        for _ in range(10):
            dist.barrier()
            torch.cuda.synchronize()
            ev[0].record()
            dp.dense_exchange(wl, ex.bucket, 0.01, False, None)
            ev[6].record()
            torch.cuda.synchronize()
            ts.append(ev[0].elapsed_time(ev[6]))
        t = torch.tensor([float(np.median(ts))], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            L = (D + P - 1) // P
            print(json.dumps(dict(P=P, mode="fused", total_us_max_over_ranks=round(float(t.item()) * 1e3, 1),
                                  nvlink_GBps_per_direction=round(2 * (P - 1) * L * 4 / (float(t.item()) * 1e-3) / 1e9 / 2, 1))),
                  flush=True)
        dist.destroy_process_group()
        return
    for _ in range(10):
        dist.barrier()
        torch.cuda.synchronize()
        ev[0].record()
        dp.partial(wl, ex.bucket)
        ev[1].record()
        h.barrier(channel=0)
        ev[2].record()
        if dp._mc is not None:
            dp.nvls_reduce_bcast()
        elif dp._aggp is not None:
            dp.reduce_push()
        else:
            dp.reduce_slice()
        ev[3].record()
        h.barrier(channel=0)
        ev[4].record()
        if dp._aggp is not None:
            dp.local_sgd(0.01, False, None)
        else:
            dp.allgather_sgd(0.01, False, None)
        ev[5].record()
        h.barrier(channel=0)
        ev[6].record()
        torch.cuda.synchronize()
        rows.append([ev[i].elapsed_time(ev[i + 1]) for i in range(6)] + [ev[0].elapsed_time(ev[6])])
    med = np.median(np.array(rows), axis=0) * 1000
    # NCCL all-reduce of the same 4D bytes (busbw convention 2(P-1)/P * bytes / t)
    buf = torch.randn(D, device=dev)
    for _ in range(3):
        dist.all_reduce(buf)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        a.record()
        dist.all_reduce(buf)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    t_ar = float(np.median(ts)) / 1e3
    L = (D + P - 1) // P
    nvl = (P - 1) * L * 4  # bytes read over NVLink per rank, each of the two phases
    rep = dict(rank=rank, P=P, mode="nvls" if dp._mc is not None else ("pull" if dp._aggp is None else "push"),
               partial_us=med[0], bar1_us=med[1], reduce_us=med[2], bar2_us=med[3],
               allgather_sgd_us=med[4], bar3_us=med[5], total_us=med[6],
               reduce_nvlink_GBps=nvl / (med[2] * 1e-6) / 1e9, allgather_nvlink_GBps=nvl / (med[4] * 1e-6) / 1e9,
               nvls_reduce_bcast_GBps_4D=4 * D / (med[2] * 1e-6) / 1e9,
               nccl_allreduce_us=t_ar * 1e6, nccl_busbw_GBps=2 * (P - 1) / P * 4 * D / t_ar / 1e9)
    if rank == 0:
        print(json.dumps({k: (round(v, 1) if isinstance(v, float) else v) for k, v in rep.items()}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
