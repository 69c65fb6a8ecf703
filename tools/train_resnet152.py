"""Real-model bucket producer: ResNet-152 data-parallel steps where
autograd writes every worker's gradient straight into its bucket row and the ScaDLES exchange
(gate -> exchange -> weighted merge -> fused momentum SGD) updates the model in place.

    python -m torch.distributed.run --nproc-per-node P --master-addr 127.0.0.1 \
        tools/train_resnet152.py [--steps 5] [--res 224]

W = 8 workers sharded W/P per GPU; worker j trains on its own stream batch of
b_j = clamp(S_j, 8, 1024) synthetic images (S = the S1 rates), weights r = S / sum(S)
(engine.py:266-267), lr = 0.1 * sum(S) / (W * 64) (engine.py:155-159, 277-281), momentum 0.9,
weight decay 1e-4.  Forward/backward under bf16 autocast, fp32 parameters and gradients.
Prints one JSON line (rank 0): per-step device times of the backward passes and of the
exchange (timed after a barrier, so it excludes the wait for the rank with the larger stream
batches), the step's path, the losses, and whether every rank's replica is bit-identical.
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

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2301_08897_b200 import build, comm, exchange, model_bucket  # noqa: E402

RATES = [31, 30, 1, 30, 42, 66, 22, 14]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--res", type=int, default=224)
    ap.add_argument("--cr", type=float, default=0.01)
    ap.add_argument("--delta", type=float, default=0.3)
    ap.add_argument("--stats", action="store_true", help="print the Top-k diagnostics of the last step")
    ap.add_argument("--overlap", action="store_true",
                    help="gate each worker on a side stream as soon as its backward is done (overlaps the next "
                         "worker's forward/backward); the step then only exchanges and merges")
    args = ap.parse_args()
    build.build()
    import torchvision

    local = int(os.environ.get("LOCAL_RANK", "0"))
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world_env > 1:
        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD
    rank = dist.get_rank() if group is not None else 0
    W = len(RATES)
    torch.manual_seed(0)  # identical initial replica on every rank
    model = torchvision.models.resnet152(num_classes=1000).to(dev)
    D = model_bucket.flat_size(model)
    ex = exchange.GradientExchange(D, W, cr=args.cr, delta=args.delta, momentum=0.9, weight_decay=1e-4,
                                   group=group, device=dev)
    model_bucket.bind(model, ex)
    model.train()
    batch = [min(max(s, 8), 1024) for s in RATES]
    w = comm.weights_from_rates(RATES)
    lr = 0.1 * sum(RATES) / (W * 64)
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    loss_fn = torch.nn.CrossEntropyLoss()
    rows = []
    side = torch.cuda.Stream(device=dev)
    main = torch.cuda.current_stream()
    for step in range(args.steps):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        e[0].record()
        losses = []
        for j in range(ex.k):
            g = ex.lo + j
            x = torch.randn((batch[g], 3, args.res, args.res), device=dev, generator=gen)
            y = torch.randint(0, 1000, (batch[g],), device=dev, generator=gen)
            model_bucket.worker_grads(model, ex, j)
            with torch.autocast("cuda", dtype=torch.bfloat16):
                loss = loss_fn(model(x), y)
            loss.backward()
            losses.append(loss.detach())
            if args.overlap:  # worker j's row is complete: its gate runs beside the next backward
                done = torch.cuda.Event()
                done.record(main)
                side.wait_event(done)
                with torch.cuda.stream(side):
                    ex.gate_worker(j)
        model_bucket.release_grads(model)
        if args.overlap:
            main.wait_stream(side)
        e[1].record()
        if group is not None:  # time the exchange itself, not the wait for the slowest rank's backward
            torch.cuda.synchronize()
            dist.barrier()
            e[1].record()
        if args.overlap:
            e[3].record()
            e[4].record()
        info = ex.step(w, lr, topk_events=None if args.overlap else (e[3], e[4]), gated=args.overlap)
        e[2].record()
        torch.cuda.synchronize()
        rows.append(dict(step=step, backward_ms=e[0].elapsed_time(e[1]), exchange_ms=e[1].elapsed_time(e[2]),
                         topk_ms=e[3].elapsed_time(e[4]), path=info.path,
                         losses=[round(float(v), 4) for v in losses]))
    if args.stats:
        from paper_2301_08897_b200 import kernels

        st = kernels.topk_stats(torch.float32, ex.k, ex.dim, ex.m, dev)
        print(json.dumps(dict(rank=rank, m=ex.m, stats_C_boundary_fb_slow=st.tolist(),
                              decisions=ex.decision.cpu().tolist(), rho=[round(float(r), 4) for r in ex.rho.cpu()])),
              flush=True)
    # replicas: bit-identical parameters on every rank (engine.py:284-286)
    same = True
    if group is not None:
        t = ex.params.view(torch.int32)
        ts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
        dist.all_gather(ts, t)
        same = all(bool(torch.equal(ts[0], x)) for x in ts)
    # the model really is the exchange's parameter vector
    p0 = next(model.parameters())
    bound = p0.data_ptr() == ex.params.data_ptr()
    if rank == 0:
        print(json.dumps(dict(model="resnet152", params=D, workers=W, overlap=args.overlap, gpus=dist.get_world_size() if group else 1,
                              workers_per_gpu=ex.k, res=args.res, batches=batch, lr=lr, replicas_identical=same,
                              params_bound=bound, steady_backward_ms=float(np.median([r["backward_ms"] for r in rows[1:]] or [0])),
                              steady_exchange_ms=float(np.median([r["exchange_ms"] for r in rows[1:]] or [0])),
                              steady_topk_ms=float(np.median([r["topk_ms"] for r in rows[1:]] or [0])),
                              steps=rows)), flush=True)
    if group is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
