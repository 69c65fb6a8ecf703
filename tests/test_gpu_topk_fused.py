"""GPU: the persistent float32 Top-k kernel's rare paths (csrc/topk_fused.cu), forced with data
built against its sampler.  The kernel estimates the threshold from a stratified sample (one
32-element chunk per stratum at a hashed offset, reproduced here); adversarial rows make the
estimate wrong on purpose:

* undershoot: only the sampled positions hold large values, so fewer than m keys reach the
  estimate -> the exact multi-pass fallback ("slow mode");
* overflow: only UNsampled positions hold large values, so the candidate pool (~2m) cannot
  hold every key above the estimate -> slow mode;
* massive ties: a constant row longer than the pool -> slow mode.

Every case must still equal the oracle (np.lexsort order) bit for bit, with the right merge
offsets and norms; stats report the path taken."""

import numpy as np
import pytest
import torch

from oracle import comm_ref

pytestmark = pytest.mark.gpu

SAMPLE, CHUNK = 131072, 32
M64 = (1 << 64) - 1


def mix64(x):
    x ^= x >> 33
    x = (x * 0xff51afd7ed558ccd) & M64
    x ^= x >> 33
    x = (x * 0xc4ceb9fe1a85ec53) & M64
    x ^= x >> 33
    return x


def sampled_mask(D, w=0):
    nch = SAMPLE // CHUNK
    stratum = D // nch
    mask = np.zeros(D, dtype=bool)
    for c in range(nch):
        h = mix64((c * 0x9e3779b97f4a7c15 + w) & M64) & 0xFFFFFFFF
        off = (h * (stratum - CHUNK + 1)) >> 32
        mask[c * stratum + off: c * stratum + off + CHUNK] = True
    return mask


def run(cuda, g, m):
    from paper_2301_08897_b200 import kernels

    D = g.size
    nt = kernels.merge_tiles(D)
    toff = torch.empty((1, nt + 1), dtype=torch.int32, device=cuda)
    idx, val, norms2, _, _ = kernels.topk_gate(torch.from_numpy(g).to(cuda), m, tile_off=toff, fused=True)
    want = comm_ref.topk_indices_threshold(g.astype(np.float64), m)
    got = idx[0].cpu().numpy().view(np.uint32).astype(np.int64)
    assert np.array_equal(got, want)
    assert np.array_equal(val[0].cpu().numpy().view(np.uint32), g[want].view(np.uint32))
    bounds = np.searchsorted(want, np.arange(nt + 1) * kernels.MERGE_TILE)
    assert np.array_equal(toff[0].cpu().numpy(), bounds)
    g64 = g.astype(np.float64)
    n = norms2[0].cpu().numpy()
    for a, b in ((n[0], g64 @ g64), (n[1], g64[want] @ g64[want])):
        if np.isfinite(b):
            assert abs(a - b) <= 1e-10 * abs(b) + 1e-300
        else:
            assert np.isnan(a) == np.isnan(b)
    return kernels.topk_stats(torch.float32, 1, D, m, cuda, fused=True)[0]


def test_estimate_undershoot_takes_exact_fallback(cuda):
    D = (1 << 22) + 3
    mask = sampled_mask(D)
    rng = np.random.default_rng(1)
    g = (rng.standard_normal(D) * 1e-3).astype(np.float32)
    g[mask] = (10 + rng.random(int(mask.sum()))).astype(np.float32)
    m = comm_ref.topk_count(D, 0.1)  # m > sampled positions: fewer than m keys reach est
    st = run(cuda, g, m)
    assert int(st[2]) == 1 and int(st[3]) == 1, st


def test_pool_overflow_takes_exact_fallback(cuda):
    D = 60_192_808
    mask = sampled_mask(D)
    rng = np.random.default_rng(2)
    g = (10 + rng.random(D)).astype(np.float32)
    g[mask] = (rng.standard_normal(int(mask.sum())) * 1e-3).astype(np.float32)
    m = comm_ref.topk_count(D, 0.001)
    st = run(cuda, g, m)
    assert int(st[3]) == 1 and int(st[0]) > 2 * m, st


def test_constant_row_longer_than_the_pool(cuda):
    D = 60_192_808
    g = np.full(D, 0.25, dtype=np.float32)
    g[123] = 1.0
    g[D - 1] = -1.0
    m = comm_ref.topk_count(D, 0.001)
    st = run(cuda, g, m)
    assert int(st[3]) == 1, st


@pytest.mark.parametrize("cr", [0.001, 0.01, 0.1])
def test_fast_path_candidate_count_is_tight(cuda, cr):
    """The sample estimate keeps C = count(key >= est) close to m (SURVEY §7 hard part 1):
    the candidate traffic is 8 C bytes on top of the 4 D of the single read."""
    D = 60_192_808
    gen = torch.Generator(device=cuda).manual_seed(3)
    z = torch.randn(D, device=cuda, generator=gen)
    g = torch.sign(z) * torch.exp(1.5 * torch.randn(D, device=cuda, generator=gen))
    from paper_2301_08897_b200 import kernels

    m = comm_ref.topk_count(D, cr)
    kernels.topk_gate(g, m, fused=True)
    st = kernels.topk_stats(torch.float32, 1, D, m, cuda, fused=True)[0]
    assert int(st[3]) == 0 and int(st[2]) == 0
    ratio = int(st[0]) / m
    print(f"[fused cr={cr}] C/m = {ratio:.4f}, boundary {int(st[1])}")
    assert 1.0 <= ratio <= {0.001: 1.5, 0.01: 1.15, 0.1: 1.06}[cr]


@pytest.mark.parametrize("D", [1, 17, 4096, 4097, 100_003, (1 << 22) + 5])
@pytest.mark.parametrize("cr", [0.001, 0.01, 0.1, 0.5, 1.0])
@pytest.mark.parametrize("fam", ["normal", "heavy", "ties", "edge"])
def test_fused_matches_oracle(cuda, D, cr, fam):
    """The fused variant over the launch-chain test families (same bar: bit-exact)."""
    from test_gpu_topk import _family

    if fam == "edge" and D < 8:
        pytest.skip("edge family needs room")
    g = _family(fam, D, seed=D * 5 + int(cr * 1000))
    m = comm_ref.topk_count(D, cr)
    run(cuda, g, m)


def test_fused_batched_rows_padding_and_state(cuda):
    """k workers, padded rows, gate states: fused == launch chain, bit for bit (idx, val,
    merge offsets, norms, decisions, EWMA states)."""
    from paper_2301_08897_b200 import kernels
    from test_gpu_topk import _family

    k, D, ld = 8, 300_001, 300_004
    host = np.zeros((k, ld), dtype=np.float32)
    for j in range(k):
        host[j, :D] = _family(["normal", "heavy", "ties", "edge"][j % 4], D, seed=200 + j)
    dev = torch.from_numpy(host).to(cuda)
    nt = kernels.merge_tiles(D)
    recs = np.zeros(k, dtype=__import__("paper_2301_08897_b200._capi", fromlist=["x"]).GATE_STATE_DTYPE)
    recs["cr"], recs["delta"], recs["ewma_factor"] = 0.01, 0.3, 0.9
    outs = []
    for fused in (False, True):
        st = kernels.gate_states_tensor(recs, cuda)
        toff = torch.empty((k, nt + 1), dtype=torch.int32, device=cuda)
        for _ in range(3):
            r = kernels.topk_gate(dev, comm_ref.topk_count(D, 0.01), st, dim=D, tile_off=toff, fused=fused)
        outs.append([t.cpu().numpy() for t in r[:2]] + [toff.cpu().numpy(), r[3].cpu().numpy(),
                                                         kernels.gate_states_numpy(st)])
    for a, b in zip(outs[0], outs[1]):
        if a.dtype.names:
            for f in ("n_compressed", "n_uncompressed"):
                assert np.array_equal(a[f], b[f])
            assert np.allclose(a["ewma_full"], b["ewma_full"], rtol=1e-12, equal_nan=True)
        else:
            assert np.array_equal(a, b)


def test_auto_variant_takes_the_pool_above_the_workspace_budget(cuda, monkeypatch):
    """topk_gate(fused=None) takes the launch chain within TOPK_WS_BUDGET and the ~2m-pool
    variant above it (e.g. D = 1e9 at k = 8: 69 GB of chain workspace); same indices and values."""
    from paper_2301_08897_b200 import kernels

    D, k = 1_000_003, 2
    m = comm_ref.topk_count(D, 0.01)
    rng = np.random.default_rng(5)
    g = torch.from_numpy((np.sign(rng.standard_normal((k, D))) * np.exp(1.5 * rng.standard_normal((k, D))))
                         .astype(np.float32)).to(cuda)
    assert not kernels.topk_use_fused(torch.float32, k, D, m)
    ref = kernels.topk_gate(g, m)
    monkeypatch.setattr(kernels, "TOPK_WS_BUDGET", 0)  # force the pool variant
    assert kernels.topk_use_fused(torch.float32, k, D, m)
    assert not kernels.topk_use_fused(torch.float64, k, D, m)  # float64 has only the chain
    got = kernels.topk_gate(g, m)
    assert torch.equal(ref[0], got[0]) and torch.equal(ref[1], got[1])
    # the norms are fixed-order sums in both variants, over different partitions
    assert torch.allclose(ref[2], got[2], rtol=1e-12, atol=0)
    want = comm_ref.topk_indices_threshold(g[1].cpu().numpy().astype(np.float64), m)
    assert np.array_equal(got[0][1].cpu().numpy().astype(np.int64), want)
