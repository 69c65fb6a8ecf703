"""BASELINE config 4 as ONE workload: non-IID CIFAR-100-shaped streams with data injection
feeding VGG-19-sized (D = 143,667,240) weighted Top-k aggregation, per step:

  host: stream buffers advance by the streaming wait (engine.py:208-221), each device draws its
        rate-matched batch (streams.py:58-134), injection plan + picks (datagen.py:182-210);
  GPU:  batches staged on the device (id range -> pool row, injected rows, x = train_x[rows] +
        augment[rows] in binary64: streams.DeviceSampler / ShardedSampler at P > 1), then the
        exchange step over the bucket (Top-k + norms + gate, exchange, weighted merge, fused
        momentum SGD: exchange.GradientExchange.step) with the S1 rate weights of this step's
        batch sizes.

The gradient producer (VGG-19 forward/backward) is out of scope: the bucket holds
the synthetic "heavy" gradients of SURVEY §8(d) (8 x 575 MB, larger than L2).

    python tools/config4.py [--steps 10] [--warmup 3] [--cr 0.01]
    torchrun --nproc-per-node P tools/config4.py ...      (P | 8)

Prints one JSON line (rank 0): step time (max over ranks, CUDA events), the share spent
staging, aggregated gradient elements/s, rows/s.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2301_08897_b200 import build, exchange, streams  # noqa: E402

VGG19 = 143_667_240
N_TRAIN, F, LABELS, N_DEV, LPD = 50_000, 3072, 100, 8, 25


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--cr", type=float, default=0.01)
    ap.add_argument("--delta", type=float, default=0.3)
    ap.add_argument("--dim", type=int, default=VGG19)
    ap.add_argument("--scale", type=int, default=8, help="S1 rates x scale = samples per second per device")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD
    build.build()
    rank = dist.get_rank() if group else 0
    rates_s1, w_s1 = bench.rates_weights(N_DEV)
    rates = [r * args.scale for r in rates_s1]
    b = [min(max(r, 8), 1024) for r in rates]

    rng = np.random.default_rng(0)
    train_x = rng.standard_normal((N_TRAIN, F))
    train_y = rng.integers(0, LABELS, N_TRAIN)
    augment = rng.standard_normal((N_TRAIN, F)) * 0.01
    pools = streams.partition(train_y, N_DEV, "noniid", LPD, seed=1)
    ex = exchange.GradientExchange(args.dim, N_DEV, cr=args.cr, delta=args.delta, momentum=0.9,
                                   weight_decay=1e-4, group=group, device=dev)
    if group is None:
        ds = streams.DeviceSampler(train_x, train_y, pools, device=dev)
    else:
        ds = streams.ShardedSampler(train_x, train_y, pools, ex.lo, ex.k, group=group, device=dev)
    ds.set_augmentation(augment)
    bench.synth_bucket(ex, "heavy", ex.lo)
    bufs = [streams.StreamBuffer(r) for r in rates]
    pick_rng = np.random.default_rng(2)
    lr = 0.1 * sum(rates_s1) / (N_DEV * 64)

    def step(it, ev=None):
        wait = max(streams.streaming_wait(len(q), b[d], rates[d]) for d, q in enumerate(bufs))
        for q in bufs:
            q.enqueue_arrivals(wait)
        draws = [q.draw_batch(b[d]) for d, q in enumerate(bufs)]
        plan = streams.injection_plan(N_DEV, 0.5, 0.5, b, seed=100 + it)
        picks = streams.injection_picks(plan, b, pick_rng)
        x, y, ptr = ds.stage(draws, plan, picks)
        if ev is not None:
            ev.record()
        info = ex.step(w_s1, lr)
        return int(ptr[-1]), info

    for it in range(args.warmup):
        step(it)
    info = None
    torch.cuda.synchronize()
    if group:
        dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    mids = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    rows = 0
    s.record()
    for i in range(args.steps):
        starts[i].record()
        n, info = step(args.warmup + i, mids[i])
        rows += n
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / args.steps
    stage_ms = float(np.median([a.elapsed_time(m) for a, m in zip(starts, mids)]))
    if group:
        t = torch.tensor([ms, stage_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, stage_ms = t.tolist()
        r = torch.tensor([rows], device=dev)
        dist.all_reduce(r)
        rows = int(r.item())
    if rank == 0:
        print(json.dumps({
            "workload": "BASELINE config 4: non-IID CIFAR-100-shaped streams (8 devices, 25 labels each, injection "
                        f"alpha=beta=0.5, batches {b}) feeding VGG-19-sized weighted Top-k aggregation",
            "dim": args.dim, "workers": N_DEV, "n_gpus": world, "cr": args.cr, "delta": args.delta,
            "steps": args.steps, "ms_per_step": ms, "stage_ms_median": stage_ms,
            "grad_elems_per_s": N_DEV * args.dim / (ms / 1e3), "rows_per_s": rows / args.steps / (ms / 1e3),
            "path": info.path,
            "data": "synthetic (seeded CIFAR-100-shaped train set; heavy-tailed gradients, no model backward)",
        }), flush=True)
    if group:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
