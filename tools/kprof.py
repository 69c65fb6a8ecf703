"""Per-kernel device time inside a steady-state step loop (torch.profiler / CUPTI; the kernels
run back to back as in bench.py, unlike an ncu launch list, which serialises and cools them).

    python tools/kprof.py [--cr 0.1] [--steps 10]
"""

from __future__ import annotations

import argparse
import sys
from collections import defaultdict
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2301_08897_b200 import build, comm, exchange  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=bench.R_DIM)
    ap.add_argument("--cr", type=float, default=0.01)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--workers", type=int, default=8)
    args = ap.parse_args()
    build.build()
    dev = torch.device("cuda", 0)
    W = args.workers
    rates, w = bench.rates_weights(W)
    ex = exchange.GradientExchange(args.dim, W, cr=args.cr, delta=0.3, momentum=0.9, weight_decay=1e-4, device=dev)
    bench.synth_bucket(ex, "heavy", 0)
    for _ in range(5):
        ex.step(w, 0.01)
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(args.steps):
            ex.step(w, 0.01)
        torch.cuda.synchronize()
    agg = defaultdict(lambda: [0, 0.0])
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            name = e.name.split("(")[0].replace("void ", "")[:40]
            agg[name][0] += 1
            agg[name][1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    tot = 0.0
    for name, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{name:42s} n={n:4d} per-step={t / args.steps:9.1f}us")
        tot += t
    print(f"total per step {tot / args.steps:.1f}us")


if __name__ == "__main__":
    main()
