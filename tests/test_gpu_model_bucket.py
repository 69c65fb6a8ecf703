"""Real-model bucket producer: autograd writes a worker's gradient in
place into its bucket row in canonical flat order, and the exchange's SGD updates the model."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _mlp():
    torch.manual_seed(3)
    return torch.nn.Sequential(torch.nn.Linear(96, 64), torch.nn.ReLU(), torch.nn.Linear(64, 32),
                               torch.nn.ReLU(), torch.nn.Linear(32, 10))


def test_bucket_rows_are_the_flat_gradients_and_sgd_updates_the_model(cuda):
    from paper_2301_08897_b200 import exchange, model_bucket

    model = _mlp().to(cuda)
    ref = _mlp().to(cuda)  # same init, plain autograd
    D = model_bucket.flat_size(model)
    ex = exchange.GradientExchange(D, 2, cr=0.1, delta=1.0, momentum=0.9, weight_decay=1e-4, device=cuda)
    model_bucket.bind(model, ex)
    # the model's parameters are views of the exchange's flat vector, values preserved
    assert torch.equal(ex.params, torch.cat([p.detach().flatten() for p in ref.parameters()]))
    gen = torch.Generator(device=cuda).manual_seed(5)
    xs = [torch.randn(7, 96, device=cuda, generator=gen) for _ in range(2)]
    flats = []
    for j in range(2):
        model_bucket.worker_grads(model, ex, j)
        model(xs[j]).square().mean().backward()
        ref.zero_grad(set_to_none=True)
        ref(xs[j]).square().mean().backward()
        flats.append(torch.cat([p.grad.flatten() for p in ref.parameters()]))
        # canonical order (layers in order, weight before bias), written in place
        assert torch.equal(ex.bucket[j, :D], flats[j])
    model_bucket.release_grads(model)
    before = ex.params.clone()
    w = np.array([0.25, 0.75])
    ex.step(w, 0.05, keep_aggregate=True)
    torch.cuda.synchronize()
    assert not torch.equal(ex.params, before)
    # the model sees the update without a copy
    assert torch.equal(torch.cat([p.detach().flatten() for p in model.parameters()]), ex.params)
    assert next(model.parameters()).data_ptr() == ex.params.data_ptr()


def test_resnet_bucket_layout(cuda):
    """A torchvision ResNet binds and trains through the bucket (conv backward is not bitwise
    deterministic, so the gradient check here is normwise)."""
    torchvision = pytest.importorskip("torchvision")
    from paper_2301_08897_b200 import exchange, model_bucket

    torch.manual_seed(0)
    model = torchvision.models.resnet18(num_classes=10).to(cuda)
    torch.manual_seed(0)
    ref = torchvision.models.resnet18(num_classes=10).to(cuda)
    D = model_bucket.flat_size(model)
    ex = exchange.GradientExchange(D, 1, cr=0.01, delta=0.3, device=cuda)
    model_bucket.bind(model, ex)
    x = torch.randn(4, 3, 32, 32, device=cuda)
    model_bucket.worker_grads(model, ex, 0)
    model(x).sum().backward()
    ref(x).sum().backward()
    flat = torch.cat([p.grad.flatten() for p in ref.parameters()])
    err = (ex.bucket[0, :D] - flat).norm() / flat.norm()
    assert float(err) < 1e-5
    model_bucket.release_grads(model)
    info = ex.step(np.array([1.0]), 0.01)
    assert info.path == "local"
