"""Top-k launch-sequence device time (CUDA events, steady state) for k workers per GPU at the
ResNet-152 gradient length, heavy-tailed synthetic gradients; roofline fraction of the
algorithmic k*(4D + 8m) bytes against the measured HBM copy peak.

    python tools/topk_timing.py [--dim D] [--ks 1,2,4,8] [--crs 0.001,0.01,0.1]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2301_08897_b200 import build, comm, kernels  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=bench.R_DIM)
    ap.add_argument("--ks", default="1,2,4,8")
    ap.add_argument("--crs", default="0.001,0.01,0.1")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--family", default="heavy")
    ap.add_argument("--fused", action="store_true", help="the persistent one-kernel variant")
    args = ap.parse_args()
    build.build()
    dev = torch.device("cuda", 0)
    hbm, kind = bench.peaks()
    D = args.dim
    ld = (D + 3) // 4 * 4
    rows = []
    for k in [int(x) for x in args.ks.split(",")]:
        g = torch.empty((k, ld), device=dev)
        for j in range(k):
            gen = torch.Generator(device=dev).manual_seed(j)
            z = torch.randn(ld, device=dev, generator=gen)
            if args.family == "heavy":
                z = torch.sign(z) * torch.exp(1.5 * torch.randn(ld, device=dev, generator=gen))
            g[j] = z
        for cr in [float(x) for x in args.crs.split(",")]:
            m = comm.topk_count(D, cr)
            idx = torch.empty((k, m), dtype=torch.int32, device=dev)
            val = torch.empty((k, m), device=dev)
            n2 = torch.empty((k, 2), dtype=torch.float64, device=dev)
            toff = torch.empty((k, kernels.merge_tiles(D) + 1), dtype=torch.int32, device=dev)
            out = (idx, val, n2, None, None)
            for _ in range(3):
                kernels.topk_gate(g, m, dim=D, out=out, tile_off=toff, fused=args.fused)
            torch.cuda.synchronize()
            ts = []
            for _ in range(args.iters):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                kernels.topk_gate(g, m, dim=D, out=out, tile_off=toff, fused=args.fused)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b) * 1e3)
            ts.sort()
            med = ts[len(ts) // 2]
            st = kernels.topk_stats(torch.float32, k, D, m, dev, fused=args.fused)
            ph = kernels.topk_phases(k, D, m, dev).astype(np.float64) if args.fused else np.zeros((k, 1, 16))
            t0 = ph[:, :, 0].min()
            names = ["start", "sample_loaded", "sample_flushed", "sample_barrier", "est", "main_loop", "main_barrier",
                     "boundary_scan", "arrived", "leader_all_arrived", "leader_resolved", "leader_flag", "flag_seen",
                     "written", "cta_done"]
            phases = {}
            for i, name in enumerate(names):
                v = ph[:, :, i] - t0
                v = v[(ph[:, :, i] > 0) & (v >= 0) & (v < 1e9)]
                if v.size:
                    phases[name] = [round(float(np.median(v)) / 1e3, 1), round(float(v.max()) / 1e3, 1)]
            v = ph[:, :, 15] - t0
            v = v[(v >= 0) & (v < 1e9)]
            phases["cleanup_end"] = round(float(v.max()) / 1e3, 1) if v.size else None
            alg = k * (4 * D + 8 * m)
            rows.append(dict(k=k, cr=cr, us_median=round(med, 1), us_min=round(ts[0], 1),
                             frac=round(alg / (med * 1e-6) / 1e9 / hbm, 4), alg_bytes=alg,
                             c_over_m=round(float(st[:, 0].mean()) / m, 4), slow=int(st[:, 3].sum()),
                             phases_us_median_max=phases))
            print(json.dumps(rows[-1]), flush=True)
        del g
        torch.cuda.empty_cache()
    print(json.dumps({"peak_gbs": hbm, "peak_kind": kind, "dim": D, "rows": rows}))


if __name__ == "__main__":
    main()
