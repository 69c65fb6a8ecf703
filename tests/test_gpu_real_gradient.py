"""GPU: Top-k, gate and merge parity on a REAL gradient: ResNet-152
(torchvision, seeded random init, bf16 autocast) backward on a synthetic batch, written by
autograd straight into the exchange bucket (model_bucket.worker_grads).  Real gradients
concentrate the kept entries in a few layers and carry bf16-rounded ties -- the cases the
adaptive collect/write split and the fused kernel's pool exist for.  Indices and values
bit-exact against the oracle for both float32 Top-k variants; the merged update equals the
float32 rounding of the oracle's float64 fold."""

import numpy as np
import pytest
import torch

from oracle import comm_ref

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def resnet_grads(cuda):
    torchvision = pytest.importorskip("torchvision")
    from paper_2301_08897_b200 import exchange, model_bucket

    torch.manual_seed(0)
    model = torchvision.models.resnet152(num_classes=1000).to(cuda)
    D = model_bucket.flat_size(model)
    ex = exchange.GradientExchange(D, 2, cr=0.01, delta=0.3, momentum=0.9, weight_decay=1e-4, device=cuda)
    model_bucket.bind(model, ex)
    gen = torch.Generator(device=cuda).manual_seed(1)
    loss_fn = torch.nn.CrossEntropyLoss()
    for j in range(2):
        x = torch.randn((8, 3, 224, 224), device=cuda, generator=gen)
        y = torch.randint(0, 1000, (8,), device=cuda, generator=gen)
        model_bucket.worker_grads(model, ex, j)
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss_fn(model(x), y).backward()
    model_bucket.release_grads(model)
    torch.cuda.synchronize()
    return ex


@pytest.mark.parametrize("cr", [0.01, 0.1])
@pytest.mark.parametrize("fused", [False, True])
def test_real_gradient_topk_bit_exact(cuda, resnet_grads, cr, fused):
    from paper_2301_08897_b200 import kernels

    ex = resnet_grads
    D = ex.dim
    m = comm_ref.topk_count(D, cr)
    nt = kernels.merge_tiles(D)
    toff = torch.empty((2, nt + 1), dtype=torch.int32, device=cuda)
    idx, val, n2, _, _ = kernels.topk_gate(ex.bucket, m, dim=D, tile_off=toff, fused=fused)
    for j in range(2):
        g = ex.bucket[j, :D].cpu().numpy()
        want = comm_ref.topk_indices_threshold(g.astype(np.float64), m)
        got = idx[j].cpu().numpy().view(np.uint32).astype(np.int64)
        assert np.array_equal(got, want), (j, cr, fused)
        assert np.array_equal(val[j].cpu().numpy().view(np.uint32), g[want].view(np.uint32))
        bounds = np.searchsorted(want, np.arange(nt + 1) * kernels.MERGE_TILE)
        assert np.array_equal(toff[j].cpu().numpy(), bounds)
        # concentration: the kept entries crowd into a small share of the merge tiles
        per_tile = np.diff(bounds)
        top = np.sort(per_tile)[::-1]
        assert top[: max(1, nt // 100)].sum() > 0.05 * m


def test_real_gradient_step_matches_oracle(cuda, resnet_grads):
    """gate -> weighted merge -> fused momentum SGD on the two real gradients."""
    ex = resnet_grads
    D = ex.dim
    w = comm_ref.rate_weights([31, 30])
    p_before = ex.params.cpu().numpy().astype(np.float64)
    gs = [ex.bucket[j, :D].cpu().numpy().astype(np.float64) for j in range(2)]
    ex.first_step = True
    ex.step(w, 0.05, keep_aggregate=True)
    torch.cuda.synchronize()
    states = [comm_ref.GateState(0.01, 0.3) for _ in range(2)]
    pw, bw, agg, dec = comm_ref.step_reference(gs, states, w, p_before, None, 0.05, 0.9, 1e-4, method="threshold")
    assert ex.decision.cpu().numpy().astype(bool).tolist() == dec
    assert np.array_equal(ex.aggregate.cpu().numpy().view(np.uint32), agg.astype(np.float32).view(np.uint32))
    assert np.array_equal(ex.params.cpu().numpy().view(np.uint32), pw.astype(np.float32).view(np.uint32))
