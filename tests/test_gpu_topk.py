"""GPU parity: Top-k sparsification (item 3) against the reference golden vectors and the oracle.

Bar: indices bit-exact (same set, ascending), values bit-exact (copies of the input)."""

import numpy as np
import pytest
import torch

from conftest import load_npz
from oracle import comm_ref

pytestmark = pytest.mark.gpu


def test_golden_topk_float64_dropin(cuda):
    from paper_2301_08897_b200 import comm

    z, meta = load_npz("topk")
    for i, mt in enumerate(meta):
        g = z[f"g{i}"]
        sp = comm.topk_sparsify(g, mt["cr"])
        assert sp.nnz == mt["m"], (i, mt)
        assert np.array_equal(sp.indices, z[f"idx{i}"]), (i, mt)
        got, want = sp.values, z[f"val{i}"]
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (i, mt)


def test_golden_topk_float32_path(cuda):
    from paper_2301_08897_b200 import kernels

    z, meta = load_npz("topk")
    n = 0
    for i, mt in enumerate(meta):
        g = z[f"g{i}"]
        g32 = g.astype(np.float32)
        if not np.array_equal(g32.astype(np.float64), g, equal_nan=True):
            continue  # not float32-representable
        idx, val, norms2, _, _ = kernels.topk_gate(torch.from_numpy(g32).to(cuda), mt["m"])
        assert np.array_equal(idx[0].cpu().numpy().astype(np.int64), z[f"idx{i}"]), (i, mt)
        assert np.array_equal(val[0].cpu().numpy().view(np.uint32), z[f"val{i}"].astype(np.float32).view(np.uint32))
        n += 1
    assert n >= 24


def _family(fam: str, D: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    z = rng.standard_normal(D, dtype=np.float32)
    if fam == "normal":
        return z
    if fam == "heavy":
        return (np.sign(z) * np.exp(1.5 * rng.standard_normal(D, dtype=np.float32))).astype(np.float32)
    if fam == "ties":
        g = (np.round(z * 8) / 8).astype(np.float32)
        g[D // 2] = g[0]
        g[D // 3] = -g[0]
        g[D - 1] = abs(g[0])
        return g
    if fam == "edge":
        g = z.copy()
        g[rng.integers(0, D, 64)] = 0.0
        g[rng.integers(0, D, 64)] = -0.0
        g[D // 7] = np.nan
        g[D // 5] = np.inf
        g[D // 3] = -np.inf
        return g
    raise ValueError(fam)


@pytest.mark.parametrize("D", [1, 3, 17, 4096, 4097, 100_003, 1 << 20, (1 << 22) + 5])
@pytest.mark.parametrize("cr", [0.001, 0.01, 0.1, 0.5, 1.0])
@pytest.mark.parametrize("fam", ["normal", "heavy", "ties", "edge"])
def test_topk_matches_oracle(cuda, D, cr, fam):
    from paper_2301_08897_b200 import kernels

    if fam == "edge" and D < 8:
        pytest.skip("edge family needs room")
    g = _family(fam, D, seed=D * 7 + int(cr * 1000))
    m = comm_ref.topk_count(D, cr)
    idx, val, norms2, _, _ = kernels.topk_gate(torch.from_numpy(g).to(cuda), m)
    want = comm_ref.topk_indices_threshold(g.astype(np.float64), m)
    got = idx[0].cpu().numpy().astype(np.int64)
    assert np.array_equal(got, want)
    assert np.array_equal(val[0].cpu().numpy().view(np.uint32), g[want].view(np.uint32))
    g64 = g.astype(np.float64)
    s_full = float(g64 @ g64)
    s_topk = float(g64[want] @ g64[want])
    n = norms2[0].cpu().numpy()
    for a, b in ((n[0], s_full), (n[1], s_topk)):
        if np.isfinite(b):
            assert abs(a - b) <= 1e-10 * abs(b) + 1e-300
        else:
            assert np.isnan(a) == np.isnan(b)


def _layers(D: int, seed: int) -> np.ndarray:
    """Real-gradient shape: small entries everywhere, a few contiguous "layers" holding the
    large ones (candidate-dense tiles in the main pass), bfloat16-rounded values (ties)."""
    rng = np.random.default_rng(seed)
    g = rng.standard_normal(D, dtype=np.float32) * np.float32(1e-4)
    for b in range(3):
        lo = int(rng.integers(0, max(1, D - D // 60)))
        n = D // 100 + 1
        g[lo:lo + n] = rng.standard_normal(min(n, D - lo), dtype=np.float32) * np.float32(10.0 ** -b)
    u = g.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return u.view(np.float32)


@pytest.mark.parametrize("D", [1 << 20, (1 << 22) + 5, 10_000_019])
@pytest.mark.parametrize("cr", [0.001, 0.01, 0.1])
def test_topk_concentrated_layers(cuda, D, cr):
    """Candidates crowded into a few contiguous blocks (the staged dense-tile placement of the
    main pass and the candidate-count split of collect/write), bit-exact in both variants."""
    from paper_2301_08897_b200 import kernels

    k = 2
    host = np.stack([_layers(D, seed=D + 31 * j + int(cr * 1e4)) for j in range(k)])
    dev = torch.from_numpy(host).to(cuda)
    m = comm_ref.topk_count(D, cr)
    for fused in (False, True):
        idx, val, norms2, _, _ = kernels.topk_gate(dev, m, fused=fused)
        for j in range(k):
            want = comm_ref.topk_indices_threshold(host[j].astype(np.float64), m)
            assert np.array_equal(idx[j].cpu().numpy().astype(np.int64), want), (j, fused)
            assert np.array_equal(val[j].cpu().numpy().view(np.uint32), host[j][want].view(np.uint32))


def test_topk_batched_rows_and_padding(cuda):
    """k workers in one launch, rows with a padded leading dimension."""
    from paper_2301_08897_b200 import kernels

    k, D, ld = 8, 300_001, 300_004
    rng = np.random.default_rng(3)
    host = np.zeros((k, ld), dtype=np.float32)
    for j in range(k):
        host[j, :D] = _family(["normal", "heavy", "ties", "edge"][j % 4], D, seed=100 + j)
    dev = torch.from_numpy(host).to(cuda)
    nt = kernels.merge_tiles(D)
    for cr in (0.001, 0.01, 0.1):
        m = comm_ref.topk_count(D, cr)
        toff = torch.full((k, nt + 1), -7, dtype=torch.int32, device=cuda)
        idx, val, norms2, _, _ = kernels.topk_gate(dev, m, dim=D, tile_off=toff)
        for j in range(k):
            want = comm_ref.topk_indices_threshold(host[j, :D].astype(np.float64), m)
            assert np.array_equal(idx[j].cpu().numpy().astype(np.int64), want), (j, cr)
            bounds = np.searchsorted(want, np.arange(nt + 1) * kernels.MERGE_TILE)
            assert np.array_equal(toff[j].cpu().numpy(), bounds), (j, cr)


def test_topk_float64_large_matches_lexsort(cuda):
    from paper_2301_08897_b200 import comm

    rng = np.random.default_rng(11)
    g = rng.normal(size=200_001)
    g[::1000] = g[0]
    for cr in (0.001, 0.01, 0.1):
        sp = comm.topk_sparsify(g, cr)
        idx, _ = comm_ref.topk(g, cr, "lexsort")
        assert np.array_equal(sp.indices, idx)


def test_topk_constant_and_all_nan(cuda):
    """Pathological ties: every key equal -> the lowest m indices (fallback path)."""
    from paper_2301_08897_b200 import kernels

    for fill in (1.5, 0.0, np.nan):
        g = np.full(1 << 18, fill, dtype=np.float32)
        m = comm_ref.topk_count(g.size, 0.01)
        idx, _, _, _, _ = kernels.topk_gate(torch.from_numpy(g).to(cuda), m)
        assert np.array_equal(idx[0].cpu().numpy(), np.arange(m))
        # the whole row is one tie group: the oversized-boundary (cooperative) resolve ran
        st = kernels.topk_stats(torch.float32, 1, g.size, m, cuda)
        assert int(st[0, 3]) == 1, st


@pytest.mark.parametrize("D,cr,fam", [(143_667_240, 0.01, "heavy"), (143_667_240, 0.1, "heavy"),
                                      ((1 << 30) + 5, 0.01, "ties")])
def test_topk_full_size_properties(cuda, D, cr, fam):
    """BASELINE sizes too large for the host oracle (VGG-19, the 1B end of the sweep): the
    size-independent properties of the reference's selection, checked on the device.  Exactly m
    ascending indices; values are bit copies; every dropped |g| <= every kept |g| (no element
    above the threshold T = min kept |g| is dropped, none below is kept); ties at T go to the
    lowest indices (np.lexsort order); merge offsets count the kept indices below each tile;
    the squared norms match a float64 reduction."""
    from paper_2301_08897_b200 import kernels

    m = comm_ref.topk_count(D, cr)
    ld = (D + 3) // 4 * 4
    gen = torch.Generator(device=cuda).manual_seed(11)
    g = torch.randn((1, ld), device=cuda, generator=gen)
    if fam == "heavy":
        g.mul_(torch.exp(1.5 * torch.randn((1, ld), device=cuda, generator=gen)))
    else:  # family (iii): quantised values, so the threshold sits inside a large tie group
        g.mul_(8).round_().div_(8)
    g[0, D:] = 0
    nt = kernels.merge_tiles(D)
    toff = torch.empty((1, nt + 1), dtype=torch.int32, device=cuda)
    idx, val, norms2, _, _ = kernels.topk_gate(g, m, dim=D, tile_off=toff)
    x = g[0, :D]
    i = idx[0].long()
    assert i.numel() == m
    assert bool((i[1:] > i[:-1]).all()) and int(i[0]) >= 0 and int(i[-1]) < D
    assert torch.equal(val[0].view(torch.int32), x[i].view(torch.int32))
    a = x.abs()
    T = float(a[i].min())
    kept = torch.zeros(D, dtype=torch.bool, device=cuda)
    kept[i] = True
    assert int((a > T).sum()) <= m <= int((a >= T).sum())
    assert not bool((~kept & (a > T)).any())
    tie = a == T
    n_tie_kept = m - int((a > T).sum())
    tie_idx = torch.nonzero(tie).flatten()
    assert torch.equal(torch.nonzero(tie & kept).flatten(), tie_idx[:n_tie_kept])
    bounds = torch.searchsorted(i, torch.arange(nt + 1, device=cuda, dtype=torch.int64) * kernels.MERGE_TILE)
    assert torch.equal(toff[0].long(), bounds)
    s_full = float((x.double() ** 2).sum())
    s_topk = float((val[0].double() ** 2).sum())
    assert abs(float(norms2[0, 0]) - s_full) <= 1e-9 * s_full
    assert abs(float(norms2[0, 1]) - s_topk) <= 1e-9 * s_topk


def _chain_sample_mask(D, w=0, nch=512, chunk=256):
    """The launch chain's sample positions for worker w (k_sample_est_f32, 16-byte-aligned rows):
    one 256-element chunk per stratum of D // 512 at a hashed, 4-aligned offset."""
    M64 = (1 << 64) - 1

    def mix64(x):
        x ^= x >> 33
        x = (x * 0xff51afd7ed558ccd) & M64
        x ^= x >> 33
        x = (x * 0xc4ceb9fe1a85ec53) & M64
        x ^= x >> 33
        return x

    stratum = D // nch
    mask = np.zeros(D, dtype=bool)
    for c in range(nch):
        h = mix64((c * 0x9e3779b97f4a7c15 + w) & M64) & 0xFFFFFFFF
        off = (h * (stratum - chunk - 3 + 1)) >> 32
        start = ((c * stratum + 3) & ~3) + (off & ~3)
        mask[start:start + chunk] = True
    return mask


def test_chain_estimate_undershoot_takes_the_fallback_pass(cuda):
    """Large values only at the chain's sampled positions: the estimate lands above every other
    key, fewer than m keys reach it, and the fallback pass (every element a candidate) must still
    give the reference's selection bit for bit, with the merge offsets and norms."""
    from paper_2301_08897_b200 import kernels

    D = 4_000_036  # a multiple of 4: the sampler's 16-byte path (the positions reproduced here)
    rng = np.random.default_rng(12)
    g = (rng.standard_normal(D) * 1e-3).astype(np.float32)
    mask = _chain_sample_mask(D)
    g[mask] = (10.0 + rng.random(int(mask.sum()))).astype(np.float32)
    m = comm_ref.topk_count(D, 0.1)  # 400,004 > the 131,072 sampled keys
    nt = kernels.merge_tiles(D)
    toff = torch.empty((1, nt + 1), dtype=torch.int32, device=cuda)
    idx, val, norms2, _, _ = kernels.topk_gate(torch.from_numpy(g).to(cuda), m, tile_off=toff, fused=False)
    st = kernels.topk_stats(torch.float32, 1, D, m, cuda)
    assert int(st[0, 2]) == 1, st  # the fallback pass ran
    want = comm_ref.topk_indices_threshold(g.astype(np.float64), m)
    got = idx[0].cpu().numpy().astype(np.int64)
    assert np.array_equal(got, want)
    assert np.array_equal(val[0].cpu().numpy().view(np.uint32), g[want].view(np.uint32))
    t = toff[0].cpu().numpy()
    assert np.array_equal(t[:-1], np.searchsorted(want, np.arange(nt) * 4096))
    assert t[-1] == m
    n = norms2[0].cpu().numpy()
    g64 = g.astype(np.float64)
    assert abs(n[0] - np.dot(g64, g64)) <= 1e-12 * np.dot(g64, g64)
    assert abs(n[1] - np.dot(g64[want], g64[want])) <= 1e-12 * np.dot(g64[want], g64[want])
