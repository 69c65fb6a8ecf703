"""Warm per-kernel timeline of one exchange step (Top-k chain + merge) from a diagnostic build
(-DSG_STAMPS: every kernel's first-CTA start and last-CTA end on %globaltimer).  Unlike an ncu
launch list (cold caches, serialised launches) this shows the chain as it runs: PDL overlap,
launch gaps, the main pass's prologue during the estimate.

    python tools/stamps.py [--workers 1] [--cr 0.01] [--iters 30]

Builds gpurun_out/diag/libscadles_b200_stamps.so (the product library is untouched) and
prints, per kernel, the median start/end (us, relative to the step's first kernel start).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2301_08897_b200 import _capi, build  # noqa: E402

TOPK = {0: "sample_est", 1: "main_tma(resident)", 6: "main_tma(after wait)", 2: "main_fb", 3: "collect", 4: "resolve",
        5: "write", 8: "se:zeroed", 9: "se:sampled", 10: "se:bucketed", 11: "se:last:h1", 12: "se:last:b1 bounds",
        13: "se:last:level2", 14: "write:body done", 15: "write:last CTA"}
AGG = {0: "merge_ws", 1: "merge", 2: "merge_own"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=1)
    ap.add_argument("--dim", type=int, default=bench.R_DIM)
    ap.add_argument("--cr", type=float, default=0.01)
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--family", default="heavy")
    ap.add_argument("--nvcc", default="", help="extra nvcc flags of the diagnostic build (A/B of compile-time constants)")
    ap.add_argument("--tag", default="stamps")
    args = ap.parse_args()
    out = ROOT / "gpurun_out" / "diag" / f"libscadles_b200_{args.tag}.so"
    out.parent.mkdir(parents=True, exist_ok=True)
    build.build_variant(out, ["-DSG_STAMPS"] + args.nvcc.split())
    _capi.LIB_PATH = out  # (or SG_LIB_PATH)
    lib = _capi.load()
    from paper_2301_08897_b200 import exchange

    dev = torch.device("cuda", 0)
    W = args.workers
    rates, w = bench.rates_weights(W)
    ex = exchange.GradientExchange(args.dim, W, cr=args.cr, delta=0.3, momentum=0.9, weight_decay=1e-4, device=dev)
    bench.synth_bucket(ex, args.family, 0)
    buf = (ctypes.c_ulonglong * 32)()
    for name in ("sg_diag_stamps_topk", "sg_diag_stamps_agg"):
        getattr(lib, name).argtypes = [ctypes.c_void_p]
    rows = []
    for it in range(args.iters + 3):
        torch.cuda.synchronize()
        lib.sg_diag_stamps_topk(buf)
        lib.sg_diag_stamps_agg(buf)
        ex.step(w, 0.05)
        torch.cuda.synchronize()
        r = {}
        lib.sg_diag_stamps_topk(buf)
        v = list(buf)
        for i, n in TOPK.items():
            if v[2 * i + 1]:
                r[n] = (v[2 * i], v[2 * i + 1])
        lib.sg_diag_stamps_agg(buf)
        v = list(buf)
        for i, n in AGG.items():
            if v[2 * i + 1]:
                r[n] = (v[2 * i], v[2 * i + 1])
        if it >= 3:
            rows.append(r)
    names = [n for n in list(TOPK.values()) + list(AGG.values()) if all(n in r for r in rows)]
    res = {}
    for n in names:
        s = np.array([r[n][0] - min(x[0] for x in r.values()) for r in rows], dtype=np.float64) / 1e3
        e = np.array([r[n][1] - min(x[0] for x in r.values()) for r in rows], dtype=np.float64) / 1e3
        res[n] = {"start_us": round(float(np.median(s)), 2), "end_us": round(float(np.median(e)), 2),
                  "dur_us": round(float(np.median(e - s)), 2)}
    for n, x in sorted(res.items(), key=lambda t: t[1]["start_us"]):
        print(f"{n:22s} start {x['start_us']:8.2f}  end {x['end_us']:8.2f}  dur {x['dur_us']:8.2f} us", file=sys.stderr)
    print(json.dumps({"workers": W, "dim": args.dim, "cr": args.cr, "iters": args.iters, "kernels": res}))


if __name__ == "__main__":
    main()
