"""Element-by-element parity of the EXACT benchmarked configuration ("checked on
every benchmarked input"): W = 8 workers x D = 60,192,808 (ResNet-152) on one GPU, S1 stream-rate
weights, delta 0.3, the bench's own synthetic gradients (bench.synth_bucket, new seed every
step), cr in {0.1, 0.01, 0.001} -- the bench/sweep points -- plus a mixed heavy/normal family
at cr 0.01 for the mixed-decision path.  Two steps each, so the EWMA gate state carries over.

Per step and worker, against the oracle (oracle/comm_ref.py, the O(D) threshold Top-k that
tests/test_oracle.py pins to the reference's lexsort):
  * gate decision equal; rho within 1e-12 relative; |rho_ref - delta| logged, near-ties
    (< 1e-12) counted and required to be 0;
  * every worker's kept indices AND values bit-exact;
  * the aggregate within 1e-5 on the abs-sum scale (per element) and normwise -- and in fact
    bit-equal to the float32 rounding of the oracle's float64 aggregate;
  * params / momentum re-anchored each step to the GPU's previous state: bit-equal to the
    float32 rounding of the oracle's update (so within the 1e-5 bound).
"""

import sys

import numpy as np
import pytest
import torch

from conftest import ROOT
from oracle import comm_ref

pytestmark = pytest.mark.gpu

sys.path.insert(0, str(ROOT))
import bench  # noqa: E402

TOL = 1e-5
R = 60_192_808
W = 8
DELTA = 0.3


@pytest.mark.parametrize("family,cr", [("heavy", 0.1), ("heavy", 0.01), ("heavy", 0.001), ("mixed", 0.01)])
def test_bench_config_full_size(cuda, family, cr):
    from paper_2301_08897_b200 import exchange

    rates, w = bench.rates_weights(W)
    assert rates == [31, 30, 1, 30, 42, 66, 22, 14]
    lr, mu, wd = 0.1 * sum(rates) / (W * 64), 0.9, 1e-4
    ex = exchange.GradientExchange(R, W, cr=cr, delta=DELTA, momentum=mu, weight_decay=wd, device=cuda)
    p0 = torch.randn(R, device=cuda, generator=torch.Generator(device=cuda).manual_seed(5)) * 0.01
    ex.params.copy_(p0)
    states = [comm_ref.GateState(cr, DELTA) for _ in range(W)]
    p64 = ex.params.cpu().numpy().astype(np.float64)
    b64 = None
    margins, paths = [], []
    for step in range(2):
        bench.synth_bucket(ex, family, 0, seed=step)
        paths.append(ex.step(w, lr, keep_aggregate=True).path)
        torch.cuda.synchronize()
        dec = ex.decision.cpu().numpy().astype(bool)
        rho = ex.rho.cpu().numpy()
        idx = ex.idx.cpu().numpy().view(np.uint32)
        val = ex.val.cpu().numpy()
        payloads = []
        scale = np.zeros(R)
        for j in range(W):
            g = ex.bucket[j, :R].cpu().numpy().astype(np.float64)
            c, payload, r_ref, _, _ = comm_ref.gate(g, states[j], "threshold")
            margins.append(abs(r_ref - DELTA))
            assert bool(dec[j]) == c, (step, j, rho[j], r_ref)
            assert abs(rho[j] - r_ref) <= 1e-12 * max(1.0, abs(r_ref)), (step, j, rho[j], r_ref)
            want_i, want_v = comm_ref.topk(g, cr, "threshold")
            assert np.array_equal(idx[j].astype(np.int64), want_i), (step, j)
            assert np.array_equal(val[j].astype(np.float64).view(np.uint64), want_v.view(np.uint64)), (step, j)
            if c:
                payloads.append((R, *payload))
                scale[payload[0]] += w[j] * np.abs(payload[1])
            else:
                payloads.append(g)
                scale += w[j] * np.abs(g)
            del g
        agg = comm_ref.aggregate(payloads, w)
        del payloads
        a32 = ex.aggregate.cpu().numpy()
        a = a32.astype(np.float64)
        assert np.all(np.abs(a - agg) <= TOL * scale + 1e-30)
        assert np.linalg.norm(a - agg) <= TOL * np.linalg.norm(agg)
        assert np.array_equal(a32.view(np.uint32), agg.astype(np.float32).view(np.uint32))
        pw, bw = comm_ref.sgd_momentum(p64, b64, agg, lr, mu, wd)
        pg = ex.params.cpu().numpy()
        bg = ex.momentum_buf.cpu().numpy()
        bound = TOL * (np.abs(p64) + lr * (mu * (np.abs(b64) if b64 is not None else 0.0) + scale + wd * np.abs(p64)))
        assert np.all(np.abs(pg.astype(np.float64) - pw) <= bound + 1e-30)
        assert np.array_equal(pg.view(np.uint32), pw.astype(np.float32).view(np.uint32))
        assert np.array_equal(bg.view(np.uint32), bw.astype(np.float32).view(np.uint32))
        p64, b64 = pg.astype(np.float64), bg.astype(np.float64)
    near = sum(m < 1e-12 for m in margins)
    print(f"[bench-parity {family} cr={cr}] paths={paths} decisions ok; min |rho_ref - delta| = {min(margins):.3e}; "
          f"near-ties {near}")
    assert near == 0
    rec = ex.gate_counters()
    assert rec["n_compressed"].tolist() == [s.n_compressed for s in states]
    assert rec["n_uncompressed"].tolist() == [s.n_uncompressed for s in states]
