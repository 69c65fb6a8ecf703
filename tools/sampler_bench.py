"""BASELINE config 4's data side: non-IID CIFAR-100-shaped streams with data injection, staged
on the device (streams.DeviceSampler: id ranges -> pool rows, injected batches, x = train_x[rows]
+ augment[rows] in binary64), timed per iteration against the reference algorithm in numpy on
the host (oracle/streams_ref: inject + materialize; test infrastructure, the CPU leg only).

    python tools/sampler_bench.py [--iters 50] [--scale 8]

Shape: 50,000 x 3072 float64 train set (32x32x3), 100 labels, 8 devices, 25 labels per device
(non-IID), S1 rates x scale as batch sizes, injection alpha = beta = 0.5.  Moved bytes per
iteration = rows x F x 8 x 3 (train_x and augment read, batch written); peak from
MEASURED_PEAKS.json as in bench.py.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2301_08897_b200 import build, streams  # noqa: E402

N_TRAIN, F, LABELS, N_DEV, LPD = 50_000, 3072, 100, 8, 25
RATES = [31, 30, 1, 30, 42, 66, 22, 14]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--scale", type=int, default=8)
    ap.add_argument("--cpu-iters", type=int, default=5)
    args = ap.parse_args()
    build.build()
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(0)
    train_x = rng.standard_normal((N_TRAIN, F))
    train_y = rng.integers(0, LABELS, N_TRAIN)
    augment = rng.standard_normal((N_TRAIN, F)) * 0.01
    pools = streams.partition(train_y, N_DEV, "noniid", LPD, seed=1)
    ds = streams.DeviceSampler(train_x, train_y, pools, device=dev)
    ds.set_augmentation(augment)
    rates = [r * args.scale for r in RATES]
    b = [min(max(r, 8), 1024) for r in rates]
    bufs = [streams.StreamBuffer(r) for r in rates]
    pick_rng = np.random.default_rng(2)

    def draw(it):
        wait = max(streams.streaming_wait(len(q), b[d], rates[d]) for d, q in enumerate(bufs))
        for q in bufs:
            q.enqueue_arrivals(wait)
        draws = [q.draw_batch(b[d]) for d, q in enumerate(bufs)]
        plan = streams.injection_plan(N_DEV, 0.5, 0.5, b, seed=100 + it)
        picks = streams.injection_picks(plan, b, pick_rng)
        return draws, plan, picks

    for it in range(5):
        ds.stage(*draw(it))
    torch.cuda.synchronize()
    rows_total, dev_ms, wall = 0, [], 0.0
    for it in range(args.iters):
        draws, plan, picks = draw(5 + it)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        s.record()
        x, y, ptr = ds.stage(draws, plan, picks)
        e.record()
        torch.cuda.synchronize()
        wall += time.perf_counter() - t0
        dev_ms.append(s.elapsed_time(e))
        rows_total += int(ptr[-1])
    rows_it = rows_total / args.iters
    bytes_it = rows_it * F * 8 * 3
    hbm, kind = bench.peaks()
    # CPU leg: the reference algorithm (numpy) on the same shapes
    from oracle import streams_ref

    t_cpu = 0.0
    for it in range(args.cpu_iters):
        draws, plan, picks = draw(1000 + it)
        t0 = time.perf_counter()
        batches = [[int(pools[d][a % len(pools[d])]) for a in draws[d]] for d in range(N_DEV)]
        out, _ = streams_ref.inject(batches, plan, F * 8, np.random.default_rng(it))
        for d in range(N_DEV):
            streams_ref.materialize(train_x, augment, train_y, out[d])
        t_cpu += time.perf_counter() - t0
    dev_med = float(np.median(dev_ms))
    print(json.dumps({
        "workload": f"non-IID CIFAR-100-shaped streams: {N_DEV} devices, {LPD} labels/device, batches {b}, injection 0.5/0.5",
        "rows_per_iter": rows_it, "bytes_per_iter": bytes_it,
        "stage_ms_device_median": dev_med, "stage_ms_wall_mean": wall / args.iters * 1e3,
        "rows_per_s_device": rows_it / (dev_med / 1e3), "achieved_GBps": bytes_it / (dev_med / 1e3) / 1e9,
        "hbm_peak_GBps": hbm, "peak_kind": kind, "frac": bytes_it / (dev_med / 1e3) / 1e9 / hbm,
        "cpu_reference_ms": t_cpu / args.cpu_iters * 1e3, "cpu_cores": 1,
    }), flush=True)


if __name__ == "__main__":
    main()
