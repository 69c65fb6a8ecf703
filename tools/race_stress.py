"""Race / determinism stress (also the small case run under compute-sanitizer, one tool per
gpurun call: tools/gpu/call63.sh): every kernel family with shared-memory hand-offs, mbarrier rings,
cooperative grid barriers, decoupled look-back or device-side flags is re-run many times on
fixed inputs, with shapes chosen to exercise its concurrent paths, and every output byte is
compared across repetitions (a race shows up as a run-to-run difference) and once against
the oracle.

    python tools/race_stress.py [--reps 50] [--quick]

Covered: the Top-k launch chain (k_sample .. k_main_tma .. k_collect .. cooperative k_resolve
(oversized ties) .. k_write .. k_finish), the persistent fused Top-k (leader/flag sync, pool
chunks, exact fallback), k_merge_ws (named-barrier producer/consumer, atomicExch lists),
k_merge_own (cp.async staging), k_merge (mixed dense/sparse).  Prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import comm_ref  # noqa: E402  (test infrastructure: the checker)
from paper_2301_08897_b200 import build, kernels  # noqa: E402


def family(kind, D, seed, dev):
    gen = torch.Generator(device=dev).manual_seed(seed)
    z = torch.randn(D, device=dev, generator=gen)
    if kind == "heavy":
        return torch.sign(z) * torch.exp(1.5 * torch.randn(D, device=dev, generator=gen))
    if kind == "ties":
        return torch.round(z * 2) / 2  # massive ties at the threshold: oversized boundary
    if kind == "hot":  # concentrated payloads (real-gradient-like): 3 % of the row carries the mass
        z[: D // 33] *= 50
        return z
    return z


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--dim", type=int, default=0, help="override D (small for compute-sanitizer runs)")
    args = ap.parse_args()
    build.build()
    dev = torch.device("cuda", 0)
    reps = 8 if args.quick else args.reps
    report = {"reps": reps, "cases": []}
    ok_all = True
    D = args.dim if args.dim > 0 else (1_000_003 if args.quick else 4_000_037)
    cases = [("heavy", 8, 0.01, False), ("ties", 2, 0.3, False), ("hot", 8, 0.1, False), ("heavy", 8, 0.01, True),
             ("ties", 2, 0.3, True), ("hot", 4, 0.1, True), ("heavy", 1, 0.001, True)]
    rates = [31, 30, 1, 30, 42, 66, 22, 14]
    for kind, k, cr, fused in cases:
        ld = (D + 3) // 4 * 4
        g = torch.zeros((k, ld), device=dev)
        for j in range(k):
            g[j, :D] = family(kind, D, 100 * j + 7, dev)
        m = comm_ref.topk_count(D, cr)
        nt = kernels.merge_tiles(D)
        w = comm_ref.rate_weights(rates[:k])
        p0 = torch.randn(D, device=dev, generator=torch.Generator(device=dev).manual_seed(3))
        first = None
        mismatches = 0
        for r in range(reps):
            idx = torch.empty((k, m), dtype=torch.int32, device=dev)
            val = torch.empty((k, m), device=dev)
            n2 = torch.empty((k, 2), dtype=torch.float64, device=dev)
            toff = torch.empty((k, nt + 1), dtype=torch.int32, device=dev)
            kernels.topk_gate(g, m, dim=D, out=(idx, val, n2, None, None), tile_off=toff, fused=fused)
            # all-sparse merge + fused SGD through both merge kernels, and the mixed path
            outs = [idx, val, n2, toff]
            for sm in (0, 1):
                p = p0.clone()
                b = torch.zeros_like(p)
                out = torch.empty(D, device=dev)
                kernels.weighted_aggregate(w, D, compressed=torch.ones(k, dtype=torch.uint8, device=dev), idx=idx,
                                           val=val, row_ptr=torch.arange(0, (k + 1) * m, m, dtype=torch.int64,
                                                                         device=dev), tile_off=toff, out=out,
                                           params=p, momentum_buf=b, lr=0.05, momentum=0.9, weight_decay=1e-4,
                                           first_step=False, sparse_merge=sm)
                outs += [out, p, b]
            comp = torch.tensor([j % 2 for j in range(k)], dtype=torch.uint8, device=dev)
            p = p0.clone()
            b = torch.zeros_like(p)
            out = torch.empty(D, device=dev)
            kernels.weighted_aggregate(w, D, compressed=comp, dense=g, idx=idx, val=val,
                                       row_ptr=torch.arange(0, (k + 1) * m, m, dtype=torch.int64, device=dev),
                                       tile_off=toff, out=out, params=p, momentum_buf=b, lr=0.05, momentum=0.9,
                                       weight_decay=1e-4, first_step=False)
            outs += [out, p, b]
            snap = [t.cpu().numpy().copy() for t in outs]
            if first is None:
                first = snap
                # one oracle check per case: worker 0's indices
                want = comm_ref.topk_indices_threshold(g[0, :D].cpu().numpy().astype(np.float64), m)
                oracle_ok = bool(np.array_equal(snap[0][0].view(np.uint32).astype(np.int64), want))
                # both all-sparse merge kernels agree bit for bit
                merge_agree = all(np.array_equal(snap[4 + i].view(np.uint32), snap[7 + i].view(np.uint32))
                                  for i in range(3))
            else:
                mismatches += sum(not np.array_equal(a.view(np.uint8), b_.view(np.uint8)) for a, b_ in zip(first, snap))
        case = dict(kind=kind, k=k, cr=cr, fused=fused, D=D, mismatching_outputs=mismatches, oracle_idx_ok=oracle_ok,
                    merge_kernels_agree=merge_agree)
        if not fused:
            case["stats_chain"] = kernels.topk_stats(torch.float32, k, D, m, dev).tolist()[0]
        else:
            case["stats_fused"] = kernels.topk_stats(torch.float32, k, D, m, dev, fused=True).tolist()[0]
        ok_all &= mismatches == 0 and oracle_ok and merge_agree
        report["cases"].append(case)
        print(json.dumps(case), flush=True)
    report["ok"] = bool(ok_all)
    print(json.dumps(report))
    sys.exit(0 if ok_all else 1)


if __name__ == "__main__":
    main()
