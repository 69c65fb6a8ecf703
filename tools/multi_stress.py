"""torchrun stress of the multi-GPU exchange protocol: many steps whose decisions switch between
all-compressed (sparse peer merge) and mixed (guarded dense side) every few steps, so buffer
reuse across the device barriers, the guarded launches and the peer reads are all exercised.
Every step checks that all ranks hold bit-identical parameters; at the end rank 0 replays the
same steps on one GPU and compares (the sparse steps are bit-identical, the dense ones differ
by the rank-ordered reduction, so the comparison is normwise at the fp32 tolerance).

    python -m torch.distributed.run --nproc-per-node P --master-addr 127.0.0.1 tools/multi_stress.py [--steps 40]
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
from paper_2301_08897_b200 import build, comm, exchange  # noqa: E402

D, W = 2_000_003, 8
RATES = [31, 30, 1, 30, 42, 66, 22, 14]


def family(step):
    return ("heavy", "heavy", "normal", "heavy", "mixed", "heavy", "heavy")[step % 7]


def fill(ex, step, lo, k):
    fam = family(step)
    for j in range(k):
        g = lo + j
        gen = torch.Generator(device=ex.device).manual_seed(7919 * step + g)
        z = torch.randn(D, device=ex.device, generator=gen)
        if fam == "heavy" or (fam == "mixed" and g % 2):
            z = torch.sign(z) * torch.exp(1.5 * torch.randn(D, device=ex.device, generator=gen))
        ex.bucket[j, :D].copy_(z * (1 + 0.1 * g))


def run(group, dev, steps, check_ranks):
    ex = exchange.GradientExchange(D, W, cr=0.01, delta=0.3, raw_gate=True, momentum=0.9, weight_decay=1e-4, group=group,
                                   device=dev)
    w = comm.weights_from_rates(RATES)
    paths, mismatches = [], 0
    for s in range(steps):
        fill(ex, s, ex.lo, ex.k)
        paths.append(ex.step(w, 0.02).path)
        if check_ranks:
            t = ex.params.view(torch.int32)
            ts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
            dist.all_gather(ts, t)
            mismatches += int(not all(bool(torch.equal(ts[0], x)) for x in ts))
    torch.cuda.synchronize()
    return ex.params.cpu().numpy().astype(np.float64), paths, mismatches


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=40)
    args = ap.parse_args()
    build.build()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank = dist.get_rank()
    p, paths, mism = run(dist.group.WORLD, dev, args.steps, True)
    ok = mism == 0
    rep = {"world": dist.get_world_size(), "steps": args.steps, "rank_mismatch_steps": mism,
           "paths": {q: paths.count(q) for q in sorted(set(paths))}}
    if rank == 0:
        p1, _, _ = run(None, dev, args.steps, False)
        rel = float(np.linalg.norm(p - p1) / np.linalg.norm(p1))
        rep["params_norm_rel_vs_1gpu"] = rel
        ok &= rel <= 1e-5
    rep["ok"] = bool(ok)
    if rank == 0:
        print(json.dumps(rep), flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
