"""torchrun check of the pool-sharded sampler: every rank holds only its
devices' train rows, injected samples travel between GPUs in one all-gather per step, and each
rank's batches must equal -- bit for bit -- the replicated-dataset DeviceSampler's batches for
the same devices (same host planning and seeds on every rank).  Also times both per step.

    python -m torch.distributed.run --nproc-per-node P --master-addr 127.0.0.1 tools/multi_sampler_check.py
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
from paper_2301_08897_b200 import build, streams  # noqa: E402

N_TRAIN, F, LABELS, N_DEV, LPD = 12_000, 3072, 100, 8, 25
RATES = [31, 30, 1, 30, 42, 66, 22, 14]


def main():
    build.build()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    k = N_DEV // world
    lo = rank * k
    rng = np.random.default_rng(0)  # identical data on every rank
    train_x = rng.standard_normal((N_TRAIN, F))
    train_y = rng.integers(0, LABELS, N_TRAIN)
    augment = rng.standard_normal((N_TRAIN, F)) * 0.01
    pools = streams.partition(train_y, N_DEV, "noniid", LPD, seed=1)
    rep = streams.DeviceSampler(train_x, train_y, pools, device=dev)
    rep.set_augmentation(augment)
    sh = streams.ShardedSampler(train_x, train_y, pools, lo, k, device=dev)
    sh.set_augmentation(augment)
    rates = [r * 4 for r in RATES]
    b = [min(max(r, 8), 1024) for r in rates]
    bufs = [streams.StreamBuffer(r) for r in rates]
    pick_rng = np.random.default_rng(2)
    ok, times_sh, times_rep, moved = True, [], [], 0
    for it in range(12):
        wait = max(streams.streaming_wait(len(q), b[d], rates[d]) for d, q in enumerate(bufs))
        for q in bufs:
            q.enqueue_arrivals(wait)
        draws = [q.draw_batch(b[d]) for d, q in enumerate(bufs)]
        ab = [(0.5, 0.5), (0.25, 0.25), (0.1, 0.1), (0.05, 0.05)][it % 4]
        plan = streams.injection_plan(N_DEV, ab[0], ab[1], b, seed=100 + it)
        picks = streams.injection_picks(plan, b, pick_rng)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        dist.barrier()
        e[0].record()
        x, y, ptr = sh.stage(draws, plan, picks)
        e[1].record()
        xr, yr, ptr_r = rep.stage(draws, plan, picks)
        e[2].record()
        torch.cuda.synchronize()
        times_sh.append(e[0].elapsed_time(e[1]))
        times_rep.append(e[1].elapsed_time(e[2]))
        a, z = int(ptr_r[lo]), int(ptr_r[lo + k])
        same = (np.array_equal(np.asarray(ptr) + a, ptr_r[lo:lo + k + 1])
                and torch.equal(x.view(torch.int64), xr[a:z].view(torch.int64)) and torch.equal(y, yr[a:z]))
        ok &= bool(same)
        moved += sum(c for _, c in plan) * F * 8
    t = torch.tensor([1.0 if ok else 0.0], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    ok = bool(t.item() == 1.0)
    if rank == 0:
        print(json.dumps({"world": world, "steps": 12, "bit_identical_to_replicated": ok,
                          "stage_ms_sharded_median": float(np.median(times_sh[2:])),
                          "stage_ms_replicated_median": float(np.median(times_rep[2:])),
                          "shard_rows_per_rank": int(sh._rows.size), "replicated_rows": N_TRAIN,
                          "shared_bytes_total": moved, "ok": ok}), flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
