"""Quick per-kernel timing probe (CUDA events) for development runs under gpurun."""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2301_08897_b200 import build, comm, kernels  # noqa: E402

R = 60_192_808


def timeit(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=R)
    ap.add_argument("--k", type=int, default=8)
    args = ap.parse_args()
    build.build()
    dev = torch.device("cuda", 0)
    D, k = args.dim, args.k
    ld = (D + 3) // 4 * 4
    gen = torch.Generator(device=dev).manual_seed(0)
    bucket = torch.randn((k, ld), device=dev, generator=gen)
    heavy = torch.sign(bucket) * torch.exp(1.5 * torch.randn((k, ld), device=dev, generator=gen))
    res = {}
    for fam, b in (("normal", bucket), ("heavy", heavy)):
        for cr in (0.1, 0.01, 0.001):
            m = comm.topk_count(D, cr)
            recs = np.zeros(k, dtype=kernels._capi.GATE_STATE_DTYPE)
            recs["cr"], recs["delta"], recs["ewma_factor"] = cr, 0.3, 0.9
            st = kernels.gate_states_tensor(recs, dev)
            out = (torch.empty((k, m), dtype=torch.int32, device=dev), torch.empty((k, m), device=dev),
                   torch.empty((k, 2), dtype=torch.float64, device=dev), torch.empty(k, dtype=torch.uint8, device=dev),
                   torch.empty(k, dtype=torch.float64, device=dev))
            us = timeit(lambda: kernels.topk_gate(b, m, st, dim=D, out=out))
            byt = k * (4 * D + 8 * m)
            res[f"topk_{fam}_{cr}"] = {"us": us, "GBs": byt / us / 1e3, "frac": byt / us / 1e3 / bench.peaks()[0]}
            torch.cuda.synchronize()
            res[f"topk_{fam}_{cr}"]["dec"] = out[3].cpu().tolist()
    # aggregate: dense only / sparse only, fused SGD
    w = np.full(k, 1.0 / k)
    p = torch.zeros(D, device=dev)
    buf = torch.zeros(D, device=dev)
    us = timeit(lambda: kernels.weighted_aggregate(w, D, dense=bucket, params=p, momentum_buf=buf, lr=0.1, momentum=0.9))
    byt = k * 4 * D + 16 * D
    res["agg_dense_sgd"] = {"us": us, "GBs": byt / us / 1e3, "frac": byt / us / 1e3 / bench.peaks()[0]}
    m = comm.topk_count(D, 0.01)
    idx, val, _, _, _ = kernels.topk_gate(bucket, m, dim=D)
    comp = torch.ones(k, dtype=torch.uint8, device=dev)
    rp = torch.arange(0, (k + 1) * m, m, dtype=torch.int64, device=dev)
    us = timeit(lambda: kernels.weighted_aggregate(w, D, compressed=comp, idx=idx, val=val, row_ptr=rp, params=p,
                                                   momentum_buf=buf, lr=0.1, momentum=0.9))
    byt = k * 8 * m + 16 * D
    res["agg_sparse_sgd_0.01"] = {"us": us, "GBs": byt / us / 1e3, "frac": byt / us / 1e3 / bench.peaks()[0]}
    out = torch.empty(D, device=dev)
    us = timeit(lambda: kernels.weighted_aggregate(w, D, compressed=comp, idx=idx, val=val, row_ptr=rp, out=out))
    byt = k * 8 * m + 4 * D
    res["agg_sparse_0.01"] = {"us": us, "GBs": byt / us / 1e3, "frac": byt / us / 1e3 / bench.peaks()[0]}
    us = timeit(lambda: out.copy_(bucket[0, :D]))
    res["torch_copy"] = {"us": us, "GBs": 8 * D / us / 1e3}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
