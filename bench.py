#!/usr/bin/env python3
"""Benchmark of the ScaDLES gradient-aggregation hot path on B200.

One step = one synchronous iteration of the hot path over one batch of synthetic gradients
of ResNet-152 size (60,192,808 fp32 elements) for W = 8 workers: per-worker Top-k (cr 0.01)
+ squared norms + EWMA gate, the exchange (local at N=1; decision all-gather then sparse
all-gather or dense all-reduce over NCCL at N>1), the stream-rate-weighted aggregation with
decompression, and the fused momentum-SGD update.  Workers are sharded k = W/N per GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0).  `value` = aggregated gradient elements per second for the
whole job (W*D per step / device time, max over ranks); `e2e` = the same through the public
API with host (pinned) gradient buffers copied in and the aggregate copied out every step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

R_DIM = 60_192_808  # ResNet-152 parameter count (torchvision)
METRIC = "aggregated grad elems/sec & HBM GB/s (%roofline) per step at 1/2/4/8 B200 vs CPU"
UNIT = "elem/s"
MEASURED = ROOT / "MEASURED_PEAKS.json"
FALLBACK_HBM = 6650.0  # B200_PROFILING.md fallback, GB/s
NVLINK_GBPS = 900.0  # NVLink 5 per direction per GPU, nominal (N > 1 measures the NCCL busbw instead)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["topk", "dense"], default="topk")
    ap.add_argument("--dim", type=int, default=R_DIM)
    ap.add_argument("--workers", type=int, default=8)
    ap.add_argument("--cr", type=float, default=0.01)
    ap.add_argument("--delta", type=float, default=0.3)
    ap.add_argument("--family", choices=["heavy", "normal", "mixed"], default="heavy")
    ap.add_argument("--cpu-steps", type=int, default=1, help="timed reference steps of our line's cpu_baseline")
    ap.add_argument("--cpu-variant", choices=["B", "A"], default="B", help="A: also time one serial 1-core step")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def peaks():
    try:
        d = json.loads(MEASURED.read_text())
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


def rates_weights(W: int):
    from paper_2301_08897_b200 import comm
    from paper_2301_08897_b200.streams import RateDistribution, derive_seed, sample_rates

    rates = sample_rates(RateDistribution("uniform", 38, 24), W, derive_seed(0, "rates"))
    return rates, comm.weights_from_rates(rates)


# ---------------------------------------------------------------------------------------
# CPU leg: the UNMODIFIED reference (streamsgd from baseline/_ref, tools/install_ref.py) at the
# bench's own shape, timed on the host cores.  The oracle port (oracle/comm_ref.py) is only a
# declared fallback when baseline/_ref is absent ("kind": "port").
#
# One reference step = the per-iteration hot path of engine.py:248-283 minus the MLP:
#   W x comm.compression_gate(g_j, state_j)       (comm.py:129-160, np.lexsort Top-k)
#   comm.weighted_aggregate(payloads, r)          (comm.py:67-78)
#   nn.sgd_momentum_step(opt, params, agg, lr)    (nn.py:161-172)
# Variant B (SPEC.md:454 allows per-device parallelism): the W gates run in W
# persistent worker processes (one per device, gradients in shared memory, one OpenBLAS
# thread each), the aggregate and the update run serially in the parent.  Variant A (one
# core, everything serial) is `python bench.py --impl reference --cpu-variant A`.
# ---------------------------------------------------------------------------------------
REF_DIR = ROOT / "baseline" / "_ref"


def _ref_modules():
    """(comm, nn, kind): the reference modules from baseline/_ref, else the oracle port."""
    if (REF_DIR / "streamsgd" / "comm.py").exists():
        if str(REF_DIR) not in sys.path:
            sys.path.insert(0, str(REF_DIR))
        import streamsgd.comm as rcomm
        import streamsgd.nn as rnn

        return rcomm, rnn, "reference"
    return None, None, "port"


def _cpu_grad(D, family, j, seed=0):
    """Worker j's synthetic gradient on the host: the bench's distributions,
    float32 values held as float64 (the reference's dtype)."""
    rng = np.random.default_rng(1000 * seed + j)
    z = rng.standard_normal(D, dtype=np.float32)
    if family == "heavy" or (family == "mixed" and j % 2 == 0):
        z = np.sign(z) * np.exp(np.float32(1.5) * rng.standard_normal(D, dtype=np.float32))
    return (z * np.float32(1 + 0.1 * j)).astype(np.float32).astype(np.float64)


def _gate_worker(conn, j, D, family, cr, delta, shm_name):
    """Persistent device process j: owns g_j (shared memory) and its CompressionState."""
    from multiprocessing import shared_memory

    rcomm, _, kind = _ref_modules()
    shm = shared_memory.SharedMemory(name=shm_name)
    g = np.ndarray((D,), dtype=np.float64, buffer=shm.buf)
    g[:] = _cpu_grad(D, family, j)
    if kind == "reference":
        state = rcomm.CompressionState(cr=cr, delta=delta)
    else:
        from oracle import comm_ref

        state = comm_ref.GateState(cr, delta)
    conn.send("ready")
    while True:
        cmd = conn.recv()
        if cmd == "stop":
            break
        if kind == "reference":
            dec = rcomm.compression_gate(g, state)
            # a dense payload IS the input array (comm.py:160): the parent maps the same memory
            conn.send(("sparse", dec.payload) if dec.compressed else ("dense", None))
        else:
            c, payload, _, _, _ = comm_ref.gate(g, state, "lexsort")
            conn.send(("sparse", (D, *payload)) if c else ("dense", None))
    del g
    shm.close()


class CpuReference:
    """W persistent gate processes + the serial aggregate/update in this process."""

    def __init__(self, W, D, family, cr, delta, compression=True):
        import multiprocessing as mp
        from multiprocessing import shared_memory

        self.W, self.D, self.cr, self.delta, self.compression = W, D, cr, delta, compression
        self.comm, self.nn, self.kind = _ref_modules()
        _, self.w = rates_weights(W)
        self.lr = 0.1 * sum(rates_weights(W)[0]) / (W * 64)
        os.environ["OPENBLAS_NUM_THREADS"] = "1"  # inherited by the spawned gate processes
        ctx = mp.get_context("spawn")
        self.shm = [shared_memory.SharedMemory(create=True, size=8 * D) for _ in range(W)]
        self.g = [np.ndarray((D,), dtype=np.float64, buffer=m.buf) for m in self.shm]
        self.conns, self.procs = [], []
        for j in range(W):
            a, b = ctx.Pipe()
            pr = ctx.Process(target=_gate_worker, args=(b, j, D, family, cr, delta, self.shm[j].name), daemon=True)
            pr.start()
            self.conns.append(a)
            self.procs.append(pr)
        for c in self.conns:
            assert c.recv() == "ready"
        self.params = np.zeros(D)
        if self.kind == "reference":
            self.opt = self.nn.OptimizerState(momentum=0.9, weight_decay=1e-4)

    def step(self) -> float:
        from oracle import comm_ref  # port fallback only

        t0 = time.perf_counter()
        if self.compression:
            for c in self.conns:
                c.send("step")
            payloads = []
            for j, c in enumerate(self.conns):
                what, payload = c.recv()
                payloads.append(payload if what == "sparse" else self.g[j])
        else:
            payloads = list(self.g)
        if self.kind == "reference":
            agg = self.comm.weighted_aggregate(payloads, self.w)
            self.nn.sgd_momentum_step(self.opt, self.params, agg, self.lr)
        else:
            agg = comm_ref.aggregate(payloads, self.w)
            comm_ref.sgd_momentum(self.params, None, agg, self.lr, 0.9, 1e-4)
        return time.perf_counter() - t0

    def close(self):
        for c in self.conns:
            try:
                c.send("stop")
            except Exception:
                pass
        for pr in self.procs:
            pr.join(timeout=10)
        for m in self.shm:
            m.close()
            m.unlink()


def _cpu_serial_step(W, D, family, cr, delta, q):
    """Variant A: one process, OPENBLAS_NUM_THREADS=1, the W gates one after another."""
    rcomm, rnn, kind = _ref_modules()
    _, w = rates_weights(W)
    gs = [_cpu_grad(D, family, j) for j in range(W)]
    states = [rcomm.CompressionState(cr=cr, delta=delta) for _ in range(W)]
    t0 = time.perf_counter()
    payloads = [rcomm.compression_gate(g, s).payload for g, s in zip(gs, states)]
    agg = rcomm.weighted_aggregate(payloads, w)
    rnn.sgd_momentum_step(rnn.OptimizerState(momentum=0.9, weight_decay=1e-4), np.zeros(D), agg, 0.01)
    q.put(time.perf_counter() - t0)


def host_info():
    model = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    blas = "unknown"
    try:
        cfg = np.show_config(mode="dicts")
        b = cfg.get("Build Dependencies", {}).get("blas", {})
        blas = f"{b.get('name', '?')} {b.get('version', '?')}"
    except Exception:
        pass
    return {"cpu_model": model, "cpu_count": os.cpu_count(), "numpy": np.__version__, "blas": blas}


def cpu_measure(args, W, steps, warmup=1):
    """Variant B at the bench's D: `steps` timed reference steps after `warmup` untimed ones."""
    ref = CpuReference(W, args.dim, args.family, args.cr, args.delta, args.workload == "topk")
    try:
        for _ in range(warmup):
            ref.step()
        times = [ref.step() for _ in range(steps)]
    finally:
        ref.close()
    t = statistics.median(times)
    hi = host_info()
    src = ("unmodified streamsgd (baseline/_ref): comm.compression_gate x W, comm.weighted_aggregate, "
           "nn.sgd_momentum_step" if ref.kind == "reference" else "oracle port oracle/comm_ref.py (baseline/_ref absent)")
    return {
        "value": W * args.dim / t,
        "unit": UNIT,
        "cores": W,
        "kind": ref.kind,
        "sample": f"the full bench workload: W={W} workers x D={args.dim} f64 (fp32-valued, {args.family} family), "
                  f"cr {args.cr}, delta {args.delta}, per step; {src}; variant B: {W} gate processes "
                  f"(1 OpenBLAS thread each) + serial aggregate/update; median of {steps} steps after {warmup} "
                  f"warm-up; host {hi['cpu_model']} ({hi['cpu_count']} logical CPUs), numpy {hi['numpy']}, {hi['blas']}",
        "step_s": t,
        "steps_s": times,
        "host": hi,
        "same_config": True,
    }


def cpu_measure_serial(args, W):
    """Variant A: one timed serial step in a fresh single-threaded process."""
    import multiprocessing as mp

    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pr = ctx.Process(target=_cpu_serial_step, args=(W, args.dim, args.family, args.cr, args.delta, q))
    pr.start()
    t = q.get()
    pr.join()
    return t


def workload_config(args, W, D, rates, k, world):
    size = "ResNet-152-sized" if D == R_DIM else ("VGG-19-sized" if D == 143_667_240 else "flat-gradient")
    compression = args.workload == "topk"
    return {
        "workload": (f"{size} adaptive Top-k aggregation: W={W} workers x D={D}, cr={args.cr}, "
                     f"delta={args.delta}, S1 rates {rates}, gate+exchange+weighted merge+fused momentum SGD"
                     if compression else
                     f"{size} weighted dense aggregation: W={W} workers x D={D}, S1 rates {rates}, "
                     f"+ fused momentum SGD"),
        "family": args.family, "workers_per_gpu": k,
        "parallelism": f"workers sharded {k}/GPU over {world} GPU(s)",
    }


def run_reference(args):
    """`--impl reference`: the reference's own CPU implementation of the path at the SAME
    config as our arm (D, W, cr, delta, family, rates), rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    W = args.workers
    rates, _ = rates_weights(W)
    warm = min(args.warmup, 1)  # CPU code has no warm-up effect beyond first touch
    cb = cpu_measure(args, W, steps=args.steps, warmup=warm)
    line = {
        "metric": METRIC, "value": cb["value"], "unit": UNIT, "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": warm,
        "ms_per_step": cb["step_s"] * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, W, args.dim, rates, max(W // max(args.gpus, 1), 1), args.gpus),
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "same_config": True, "host": cb["host"], "step_s": cb["steps_s"],
        "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    if args.cpu_variant == "A":
        t = cpu_measure_serial(args, W)
        line["variant_a"] = {"value": W * args.dim / t, "unit": UNIT, "cores": 1, "step_s": t,
                             "sample": "one serial step (W gates, aggregate, update), OPENBLAS_NUM_THREADS=1"}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------
# GPU leg
# ---------------------------------------------------------------------------------------
class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id):
        self.gpu_id = gpu_id
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu_id), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.th.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def synth_bucket(ex, family, rank_lo, seed=0):
    """The synthetic gradients of SURVEY §8(d): worker j's row from its own seeded generator,
    N(0,1)*(1 + 0.1 j) ("normal") or sign(z)*exp(1.5 z') ("heavy": the mixed-gate regime);
    "mixed" alternates heavy (even j) and normal (odd j) workers."""
    import torch

    dev = ex.device
    for j in range(ex.k):
        gj = rank_lo + j
        gen = torch.Generator(device=dev).manual_seed(seed * 1000 + gj)
        z = torch.randn(ex.dim, device=dev, generator=gen)
        if family == "heavy" or (family == "mixed" and gj % 2 == 0):
            z = torch.sign(z) * torch.exp(1.5 * torch.randn(ex.dim, device=dev, generator=gen))
        ex.bucket[j, :ex.dim].copy_(z * (1 + 0.1 * gj))


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2301_08897_b200 import build, comm, exchange, kernels

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        # NCCL prints its version line on fd 1 when the communicator comes up: point fd 1 at
        # stderr for that, so stdout carries only the JSON line
        sys.stdout.flush()
        saved = os.dup(1)
        os.dup2(2, 1)
        try:
            dist.init_process_group("nccl", device_id=dev)
            dist.barrier()
            torch.cuda.synchronize()
        finally:
            os.dup2(saved, 1)
            os.close(saved)
        group = dist.group.WORLD
    build.build()
    W, D = args.workers, args.dim
    rates, w = rates_weights(W)
    lr = 0.1 * sum(rates) / (W * 64)  # scale_lr(base 0.1, sum S, n*64), nn.py:184-190
    compression = args.workload == "topk"
    ex = exchange.GradientExchange(D, W, cr=args.cr, delta=args.delta, compression=compression, momentum=0.9,
                                   weight_decay=1e-4, group=group, device=dev)
    synth_bucket(ex, args.family, ex.lo)
    torch.cuda.synchronize()

    def barrier():
        if group is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def reduce_max(x: float) -> float:
        if group is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # NVLink roofline denominator at N > 1: the measured NCCL all-reduce bus bandwidth of a
    # D-float buffer on this box (busbw = 2(P-1)/P * bytes / t), not the nominal 900 GB/s
    nvl_peak, nvl_kind = NVLINK_GBPS, "nominal"
    if world > 1:
        buf = torch.randn(D, device=dev)
        for _ in range(2):
            dist.all_reduce(buf)
        barrier()
        a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_ev.record()
        for _ in range(3):
            dist.all_reduce(buf)
        b_ev.record()
        barrier()
        t_ar = reduce_max(a_ev.elapsed_time(b_ev)) / 3 / 1e3
        nvl_peak, nvl_kind = 2 * (world - 1) / world * 4 * D / t_ar / 1e9, "measured NCCL all-reduce busbw"
        del buf

    # ---- device-resident timing -------------------------------------------------------
    cvd = os.environ.get("CUDA_VISIBLE_DEVICES", "")
    clocks = Clocks(cvd.split(",")[local] if cvd else local)
    clocks.start()  # sampled over warm-up, timed region and the e2e leg (>= several hundred ms)
    time.sleep(0.3)
    for _ in range(args.warmup):
        ex.step(w, lr)
    K = args.steps
    ev_topk = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    launches0 = kernels.LAUNCHES["n"]
    infos = []
    s_ev.record()
    for i in range(K):
        infos.append(ex.step(w, lr, topk_events=ev_topk[i] if compression else None))
    e_ev.record()
    paths = [info.path for info in infos]  # (read after the timed region: may wait for decisions)
    barrier()
    launches = kernels.LAUNCHES["n"] - launches0
    t_ms = reduce_max(s_ev.elapsed_time(e_ev))
    topk_ms = [a.elapsed_time(b) for a, b in ev_topk] if compression else []
    value = W * D * K / (t_ms / 1e3)
    hbm, hbm_kind = peaks()
    m = ex.m
    k = ex.k
    roof = None
    if compression:
        topk_avg = statistics.mean(topk_ms) / 1e3
        alg = k * (4 * D + 8 * m)
        achieved = alg / topk_avg / 1e9
        traffic = None
        tf = ROOT / "profiles" / "traffic.json"
        if tf.exists():
            try:
                traffic = json.loads(tf.read_text()).get(f"topk_k{k}_cr{args.cr}")
            except Exception:
                traffic = None
        roof = {"kernel": "sg_topk_gate_f32 (Top-k + norms + gate launch sequence)", "bound": "hbm",
                "achieved": achieved, "peak": hbm, "peak_kind": hbm_kind, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": traffic, "alg_bytes_per_launch": alg, "avg_launch_us": topk_avg * 1e6}
    # whole-step algorithmic HBM bytes per GPU (SGD fused: 16 B/elem)
    all_sparse = all(p in ("local", "sparse-allgather", "sparse-peer") for p in paths) and compression and \
        bool((ex.decision == 1).all().item())
    if compression and all_sparse:
        step_bytes = k * (4 * D + 8 * m) + W * 8 * m + 16 * D
    elif compression:
        step_bytes = k * (4 * D + 8 * m) + k * 4 * D + 16 * D
    else:
        step_bytes = k * 4 * D + 16 * D
    step_s = t_ms / 1e3 / K
    step_roof = {"bytes_per_step": step_bytes, "achieved": step_bytes / step_s / 1e9, "frac": step_bytes / step_s / 1e9 / hbm}
    # NVLink bytes each GPU receives per step: the other ranks' sparse payloads,
    # or the dense all-reduce's 2(P-1)/P * 4D (busbw convention); nominal 900 GB/s per direction
    if world > 1:
        nvl = (world - 1) * k * 8 * m if (compression and all_sparse) else 2 * (world - 1) / world * 4 * D
        nvl_frac = nvl / step_s / 1e9 / nvl_peak
        step_roof["nvlink"] = {"bytes_per_step": nvl, "achieved": nvl / step_s / 1e9, "peak": nvl_peak,
                               "peak_kind": nvl_kind, "frac": nvl_frac}
        step_roof["binding"] = "nvlink" if nvl_frac > step_roof["frac"] else "hbm"
    else:
        step_roof["binding"] = "hbm"

    # ---- end to end through the public API with host buffers --------------------------
    e2e = None
    if not args.no_e2e:
        # Pinned host gradients in, aggregate (and decisions) out, every step, through the
        # public GradientExchange.step.  Two device buckets and two copy streams pipeline the
        # steps: step s+1's H2D (copy-in stream) overlaps step s's compute and D2H (copy-out
        # stream); PCIe is full duplex.
        host = torch.empty((k, ex.ld), dtype=torch.float32, pin_memory=True)
        host.copy_(ex.bucket)
        agg_host = torch.empty(D, dtype=torch.float32, pin_memory=True)
        dec_host = torch.empty(k, dtype=torch.uint8, pin_memory=True)
        buckets = [ex.bucket, torch.empty_like(ex.bucket)]
        main = torch.cuda.current_stream()
        cin, cout = torch.cuda.Stream(), torch.cuda.Stream()
        ev = lambda: torch.cuda.Event()  # noqa: E731
        ready, freed, outd = [ev(), ev()], [ev(), ev()], ev()
        for i in range(2):
            freed[i].record(main)
        outd.record(main)

        def e2e_steps(n):
            cin.wait_event(freed[0])
            with torch.cuda.stream(cin):
                buckets[0].copy_(host, non_blocking=True)
            ready[0].record(cin)
            for s in range(n):
                b, nb = s % 2, (s + 1) % 2
                if s + 1 < n:  # next step's inputs, as soon as its bucket is free
                    cin.wait_event(freed[nb])
                    with torch.cuda.stream(cin):
                        buckets[nb].copy_(host, non_blocking=True)
                    ready[nb].record(cin)
                main.wait_event(ready[b])
                main.wait_event(outd)  # the aggregate buffer is read out before it is rewritten
                ex.bucket = buckets[b]
                ex.step(w, lr, keep_aggregate=True)
                freed[b].record(main)
                cout.wait_stream(main)
                with torch.cuda.stream(cout):
                    agg_host.copy_(ex.aggregate, non_blocking=True)
                    if compression:
                        dec_host.copy_(ex.decision, non_blocking=True)
                outd.record(cout)
            main.wait_stream(cout)

        ke = max(3, K // 4)
        e2e_steps(2)
        s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        s2.record()
        e2e_steps(ke)
        e2.record()
        barrier()
        te = reduce_max(s2.elapsed_time(e2))
        ex.bucket = buckets[0]
        e2e = {"value": W * D * ke / (te / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(k * ex.ld * 4),
               "d2h_bytes_per_step": int(D * 4 + (k if compression else 0)), "steps": ke,
               "path": "GradientExchange.step on pinned host gradients (H2D) with the aggregate and "
                       "decisions copied back (D2H) every step; two device buckets, copy-in/out "
                       "streams overlap step s+1's H2D with step s's compute and D2H"}

    clk = clocks.stop()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_measure(args, W, steps=args.cpu_steps, warmup=0)
        cpu = {k_: cb[k_] for k_ in ("value", "unit", "cores", "kind", "sample")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": t_ms / K, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32 (f64 accumulation)", "data": "synthetic",
            "config": {
                **workload_config(args, W, D, rates, k, world),
                "l2": (f"inputs larger than L2 ({k} x {D * 4 / 1e6:.0f} MB bucket per GPU)" if k * D * 4 > 126e6 else
                       f"inputs L2-resident ({k} x {D * 4 / 1e6:.1f} MB bucket per GPU): sweep point, not a bench line"),
                "paths": sorted(set(paths)),
            },
            "roofline": roof,
            "step_roofline": step_roof,
            "per_gpu_value": k * D * K / (t_ms / 1e3),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
        }
        if roof is not None:
            line["topk_us"] = {"mean": statistics.mean(topk_ms) * 1e3, "min": min(topk_ms) * 1e3}
        print(json.dumps(line), flush=True)
    if group is not None:
        ex.close()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
