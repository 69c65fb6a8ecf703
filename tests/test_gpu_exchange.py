"""GPU parity of the per-GPU batched step (gate -> aggregate -> fused momentum SGD) against the
oracle's step_reference on the same float32 inputs upcast to float64.

Bar (north_star): Top-k indices and gate decisions bit-exact; aggregated gradient and
post-step weights within rel 1e-5 on the abs-sum scale.  The kernels compute
in binary64 on the upcast inputs and round once, so the observed error is <= 0.5 ulp fp32.
"""

import numpy as np
import pytest
import torch

from oracle import comm_ref

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _grads(W, D, fam, seed):
    rng = np.random.default_rng(seed)
    out = []
    for j in range(W):
        z = rng.standard_normal(D, dtype=np.float32)
        if fam == "heavy":
            g = np.sign(z) * np.exp(1.5 * rng.standard_normal(D, dtype=np.float32))
        elif fam == "mixed":
            g = z * (1 + 0.1 * j) if j % 2 else np.sign(z) * np.exp(1.5 * rng.standard_normal(D, dtype=np.float32))
        else:
            g = z * (1 + 0.1 * j)
        out.append(g.astype(np.float32))
    return out


@pytest.mark.parametrize("fam,cr,delta", [("heavy", 0.01, 0.3), ("normal", 0.01, 0.3), ("mixed", 0.1, 0.5),
                                          ("heavy", 0.001, 1.0)])
def test_step_matches_oracle(cuda, fam, cr, delta):
    from paper_2301_08897_b200 import exchange

    W, D = 8, 1_000_003
    rates = [31, 30, 1, 30, 42, 66, 22, 14]
    w = comm_ref.rate_weights(rates)
    lr, mu, wd = 0.1 * sum(rates) / (W * 64), 0.9, 1e-4
    ex = exchange.GradientExchange(D, W, cr=cr, delta=delta, momentum=mu, weight_decay=wd, device=cuda)
    p = np.random.default_rng(1).standard_normal(D, dtype=np.float32) * 0.01
    ex.params.copy_(torch.from_numpy(p))
    states = [comm_ref.GateState(cr, delta) for _ in range(W)]
    p64, b64 = p.astype(np.float64), None
    for step in range(3):
        gs = _grads(W, D, fam, seed=10 * step + 1)
        ex.bucket[:, :D].copy_(torch.from_numpy(np.stack(gs)))
        ex.step(w, lr, keep_aggregate=True)
        # oracle from the GPU's previous state (re-anchored each step)
        pw, bw, agg, dec = comm_ref.step_reference([g.astype(np.float64) for g in gs], states, w, p64, b64,
                                                   lr, mu, wd, method="threshold")
        got_dec = ex.decision.cpu().numpy().astype(bool).tolist()
        assert got_dec == dec, (step, got_dec, dec)
        scale = sum(wj * np.abs(g.astype(np.float64)) for wj, g in zip(w, gs))
        a = ex.aggregate.cpu().numpy().astype(np.float64)
        assert np.all(np.abs(a - agg) <= TOL * scale + 1e-30)
        assert np.linalg.norm(a - agg) <= TOL * np.linalg.norm(agg)
        assert np.array_equal(ex.aggregate.cpu().numpy().view(np.uint32), agg.astype(np.float32).view(np.uint32))
        pg = ex.params.cpu().numpy()
        bg = ex.momentum_buf.cpu().numpy()
        assert np.array_equal(pg.view(np.uint32), pw.astype(np.float32).view(np.uint32))
        assert np.array_equal(bg.view(np.uint32), bw.astype(np.float32).view(np.uint32))
        p64, b64 = pg.astype(np.float64), bg.astype(np.float64)
    rec = ex.gate_counters()
    assert rec["n_compressed"].tolist() == [s.n_compressed for s in states]


def test_step_at_resnet152_size_properties(cuda):
    """Full ResNet-152 gradient length, 8 workers on one GPU: indices exact for worker 0 via the
    O(D) threshold oracle, every worker's kept set sums to s_topk, replica checksum stable."""
    from paper_2301_08897_b200 import exchange

    W, D = 8, 60_192_808
    ex = exchange.GradientExchange(D, W, cr=0.01, delta=0.3, device=cuda)
    gen = torch.Generator(device=cuda).manual_seed(7)
    z = torch.randn((W, ex.ld), device=cuda, generator=gen)
    ex.bucket.copy_(torch.sign(z) * torch.exp(1.5 * torch.randn((W, ex.ld), device=cuda, generator=gen)))
    w = np.full(W, 1.0 / W)
    ex.step(w, 0.01, keep_aggregate=True)
    g0 = ex.bucket[0, :D].cpu().numpy()
    want = comm_ref.topk_indices_threshold(g0.astype(np.float64), ex.m)
    assert np.array_equal(ex.idx[0].cpu().numpy().astype(np.int64), want)
    for j in range(W):
        v = ex.val[j].double()
        assert abs(float((v * v).sum()) - float(ex.norms2[j, 1])) <= 1e-9 * float(ex.norms2[j, 1])
    assert bool((ex.decision == 1).all())
    # sparse aggregate mass equals the weighted sum of kept values
    total = float(ex.aggregate.double().sum())
    want_total = sum(w[j] * float(ex.val[j].double().sum()) for j in range(W))
    assert abs(total - want_total) <= 1e-6 * sum(w[j] * float(ex.val[j].double().abs().sum()) for j in range(W))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_multi_gpu_exchange_matches_single_gpu(cuda):
    """torchrun over all visible GPUs (NCCL): sparse all-gather path bit-identical to one GPU,
    dense all-reduce path within fp32 tolerance, replicas identical on every rank."""
    import json
    import subprocess
    import sys

    from conftest import ROOT

    import os

    n = 4 if torch.cuda.device_count() >= 4 else 2
    # peer path (symmetric buffers read in place by the merge) and the NCCL all-gather path
    # (and one worker per rank, the 8-GPU shape: W = P)
    # (SG_PAYLOAD_MC=1: the payloads broadcast through the switch and merged from local memory,
    # instead of the default merge reading the peers' payloads over NVLink)
    for port, p2p, workers, sparse_path, mc in (("29531", "1", "8", "sparse-peer", "0"),
                                                ("29532", "0", "8", "sparse-allgather", "0"),
                                                ("29533", "1", str(n), "sparse-peer", "0"),
                                                ("29534", "1", "8", "sparse-peer", "1")):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
               "--master-addr", "127.0.0.1", "--master-port", port, str(ROOT / "tools" / "multi_check.py")]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600,
                           env={**os.environ, "SG_P2P": p2p, "SG_CHECK_WORKERS": workers, "SG_PAYLOAD_MC": mc})
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
        rep = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
        assert rep["ok"] and rep["world"] == n
        assert rep["cases"][0]["paths"] == [sparse_path] * 3, rep["cases"][0]
        dense_path = "dense-peer" if p2p == "1" else "dense-allreduce"
        assert rep["cases"][-1]["paths"] == [dense_path] * 3, rep["cases"][-1]  # the dense workload


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_multi_gpu_protocol_stress(cuda):
    """20 steps whose decisions switch between all-compressed and mixed (tools/multi_stress.py):
    every rank bit-identical after every step, on the peer path and the NCCL path."""
    import json
    import os
    import subprocess
    import sys

    from conftest import ROOT

    n = 4 if torch.cuda.device_count() >= 4 else 2
    for port, p2p, paths in (("29541", "1", {"dense-peer", "sparse-peer"}),
                             ("29542", "0", {"dense-allreduce", "sparse-allgather"})):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
               "--master-addr", "127.0.0.1", "--master-port", port, str(ROOT / "tools" / "multi_stress.py"),
               "--steps", "20"]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env={**os.environ, "SG_P2P": p2p})
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
        rep = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
        assert rep["ok"] and rep["rank_mismatch_steps"] == 0
        assert set(rep["paths"]) == paths, rep


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_multicast_payload_broadcast_keeps_every_bit_pattern(cuda):
    """The payload broadcast (multimem.st through the switch) delivers NaN payloads, -0, infinities
    and index words in float32's NaN range unchanged into every rank's slot (tools/mc_check.py)."""
    import json
    import os
    import subprocess
    import sys

    from conftest import ROOT

    n = 4 if torch.cuda.device_count() >= 4 else 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29545", str(ROOT / "tools" / "mc_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=dict(os.environ))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    rep = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert rep["ok"] and rep["world"] == n
