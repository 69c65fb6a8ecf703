"""torchrun checker: the NCCL exchange (P ranks, W/P workers each) against one GPU holding all W.

    python -m torch.distributed.run --nproc-per-node P --master-addr 127.0.0.1 tools/multi_check.py

Sparse all-gather path: params/aggregate must be bit-identical to the single-GPU run (same
fold of the same payloads).  Dense all-reduce path: within the fp32 tolerance, and identical
on every rank.  Prints one JSON line on rank 0 and exits non-zero on a mismatch.
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

D = 4_000_037
W = int(os.environ.get("SG_CHECK_WORKERS", "8"))  # W = P gives one worker per rank (the 8-GPU shape)


def fill(ex, family, step):
    for j in range(ex.k):
        g = ex.lo + j
        gen = torch.Generator(device=ex.device).manual_seed(1000 * step + g)
        z = torch.randn(D, device=ex.device, generator=gen)
        if family == "heavy" or (family == "mixed" and g % 2):
            z = torch.sign(z) * torch.exp(1.5 * torch.randn(D, device=ex.device, generator=gen))
        ex.bucket[j, :D].copy_(z * (1 + 0.1 * g))


def run(family, cr, delta, group, dev, steps=3):
    compression = cr is not None
    ex = exchange.GradientExchange(D, W, cr=cr or 0.01, delta=delta or 0.3, compression=compression, momentum=0.9,
                                   weight_decay=1e-4, group=group, device=dev)
    w = comm.weights_from_rates(([31, 30, 1, 30, 42, 66, 22, 14] * 8)[:W])
    paths = []
    for s in range(steps):
        fill(ex, family, s)
        paths.append(ex.step(w, 0.05, keep_aggregate=True).path)
    torch.cuda.synchronize()
    return ex.params.cpu().numpy(), ex.aggregate.cpu().numpy(), paths


def main():
    build.build()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    ok = True
    report = {"world": world, "cases": []}
    # (heavy, 0.1: all compressed at 0.8 kept entries per position -> k_merge_own over peer memory)
    # (None: the dense workload, compression off -> peer reduce-scatter + all-gather/SGD or NCCL)
    for family, cr, delta in (("heavy", 0.01, 0.5), ("normal", 0.01, 0.3), ("mixed", 0.1, 0.5), ("heavy", 0.1, 0.5),
                              ("normal", None, None)):
        p, a, paths = run(family, cr, delta, dist.group.WORLD, dev)
        # every rank holds identical bytes
        t = torch.from_numpy(p).to(dev)
        ts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(ts, t)
        same = all(bool(torch.equal(ts[0], x)) for x in ts)
        case = {"family": family, "paths": paths, "ranks_identical": same}
        if rank == 0:
            p1, a1, paths1 = run(family, cr, delta, None, dev)
            if paths[-1] in ("sparse-allgather", "sparse-peer"):
                case["bit_identical_to_1gpu"] = bool(np.array_equal(p, p1) and np.array_equal(a, a1))
                ok &= case["bit_identical_to_1gpu"]
            else:
                scale = np.abs(a1.astype(np.float64)).max()
                err = float(np.max(np.abs(a.astype(np.float64) - a1)) / scale)
                perr = float(np.linalg.norm(p.astype(np.float64) - p1) / np.linalg.norm(p1))
                case.update(agg_max_rel=err, params_norm_rel=perr)
                ok &= err <= 1e-5 and perr <= 1e-5
        ok &= same
        report["cases"].append(case)
    report["ok"] = bool(ok)
    if rank == 0:
        print(json.dumps(report), flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
