"""torchrun: device-time breakdown of one GradientExchange step per rank (Top-k/gate, the
packed all-gather, the host decision check, the merge), CUDA events on the compute stream.

    python -m torch.distributed.run --nproc-per-node P --master-addr 127.0.0.1 tools/multi_timing.py
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2301_08897_b200 import build, comm, exchange  # noqa: E402

D, W = 60_192_808, 8


def main():
    build.build()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank = dist.get_rank()
    ex = exchange.GradientExchange(D, W, cr=0.01, delta=0.3, momentum=0.9, weight_decay=1e-4,
                                   group=dist.group.WORLD, device=dev)
    gen = torch.Generator(device=dev).manual_seed(rank)
    z = torch.randn(ex.bucket.shape, device=dev, generator=gen)
    ex.bucket.copy_(torch.sign(z) * torch.exp(1.5 * torch.randn(ex.bucket.shape, device=dev, generator=gen)))
    w = comm.weights_from_rates([31, 30, 1, 30, 42, 66, 22, 14])
    for _ in range(3):
        ex.step(w, 0.01)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    rows = []
    from paper_2301_08897_b200 import kernels

    # ev0 step start | ev1 Top-k done | ev2 right before the merge launch | ev3 merge done
    for cls in (kernels.MergeLauncher, kernels.PeerMergeLauncher):
        orig = cls.__call__

        def timed(self, *a, _orig=orig, **k):
            ev[2].record()
            r = _orig(self, *a, **k)
            ev[3].record()
            return r

        cls.__call__ = timed
    for _ in range(10):
        dist.barrier()
        torch.cuda.synchronize()
        ev[0].record()
        info = ex.step(w, 0.01, topk_events=(torch.cuda.Event(), ev[1]))
        ev[4].record()
        torch.cuda.synchronize()
        rows.append([ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3]),
                     ev[3].elapsed_time(ev[4]), ev[0].elapsed_time(ev[4])])
    med = np.median(np.array(rows), axis=0) * 1000
    rep = dict(rank=rank, path=info.path, topk_us=med[0], exchange_and_check_us=med[1], merge_us=med[2],
               tail_us=med[3], step_us=med[4])
    print(json.dumps({k: (round(v, 1) if isinstance(v, float) else v) for k, v in rep.items()}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
