"""A few full hot-path steps at ResNet-152 size for launch lists / ncu captures."""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2301_08897_b200 import build, exchange  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=60_192_808)
    ap.add_argument("--workers", type=int, default=8)
    ap.add_argument("--cr", type=float, default=0.01)
    ap.add_argument("--delta", type=float, default=0.3)
    ap.add_argument("--family", default="heavy")
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    build.build()
    dev = torch.device("cuda", 0)
    ex = exchange.GradientExchange(args.dim, args.workers, cr=args.cr, delta=args.delta, device=dev)
    gen = torch.Generator(device=dev).manual_seed(0)
    z = torch.randn(ex.bucket.shape, device=dev, generator=gen)
    if args.family == "heavy":
        z = torch.sign(z) * torch.exp(1.5 * torch.randn(ex.bucket.shape, device=dev, generator=gen))
    elif args.family == "tie":  # heavy ties at the threshold: the oversized-boundary (slow) resolve
        z = torch.round(z * 2) / 2
    ex.bucket.copy_(z)
    w = np.full(args.workers, 1.0 / args.workers)
    for _ in range(args.steps):
        info = ex.step(w, 0.01)
    torch.cuda.synchronize()
    from paper_2301_08897_b200 import kernels
    st = kernels.topk_stats(torch.float32, ex.k, ex.dim, ex.m, dev)
    print(info.path, ex.decision.cpu().tolist(), "m", ex.m, "stats[C, boundary, fb, slow]", st.tolist())


if __name__ == "__main__":
    main()
