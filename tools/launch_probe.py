"""Event-timed cost of a near-empty float32 Top-k call (D = 4096, k = 1) and of a trivial torch
kernel, back to back in one stream: the launch overhead of the cooperative Top-k kernel."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2301_08897_b200 import build, kernels  # noqa: E402

build.build()
dev = torch.device("cuda", 0)
g = torch.randn(4096, device=dev)
x = torch.zeros(1, device=dev)
for name, fn in (("topk_4096", lambda: kernels.topk_gate(g, 41)), ("torch_add", lambda: x.add_(1))):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(100):
        fn()
    b.record()
    torch.cuda.synchronize()
    print(f"{name}: {a.elapsed_time(b) * 10:.1f} us per call (100 back to back)")
