"""torchrun: the payload broadcast (sg_multicast_copy_u32, multimem.st through the NVSwitch)
carries every 32-bit pattern unchanged -- NaN payloads, -0, infinities, index words in the NaN
range of float32 -- into every rank's slot.  Prints one JSON line (rank 0); exit 1 on mismatch.

    python -m torch.distributed.run --nproc-per-node P --master-addr 127.0.0.1 tools/mc_check.py
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
from paper_2301_08897_b200 import build, kernels  # noqa: E402

WORDS = 1 << 16


def pattern(rank: int) -> np.ndarray:
    rng = np.random.default_rng(1000 + rank)
    w = rng.integers(0, 1 << 32, WORDS, dtype=np.uint64).astype(np.uint32)
    special = np.array([0x7FC00000, 0x7FC00001, 0x7FFFFFFF, 0xFFFFFFFF, 0xFF800001, 0x7F800000, 0xFF800000,
                        0x80000000, 0x00000000, 0x00000001, 0x7F800001, 0x7FBFFFFF], dtype=np.uint32)
    w[:special.size] = special
    w[special.size:2 * special.size] = special + np.uint32(rank)
    return w


def main():
    build.build()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    import torch.distributed._symmetric_memory as symm_mem

    rank, P = dist.get_rank(), dist.get_world_size()
    buf = symm_mem.empty(P * WORDS, dtype=torch.int32, device=dev)
    buf.fill_(0x5A5A5A5A)
    h = symm_mem.rendezvous(buf, dist.group.WORLD.group_name)
    if int(h.multicast_ptr) == 0:
        if rank == 0:
            print(json.dumps({"world": P, "multicast": False, "ok": True}))
        dist.destroy_process_group()
        return
    src = torch.from_numpy(pattern(rank).view(np.int32)).to(dev)
    off = buf.data_ptr() - h.buffer_ptrs[rank]
    kernels.multicast_copy(src, int(h.multicast_ptr) + off + 4 * rank * WORDS)
    h.barrier(channel=0)
    got = buf.cpu().numpy().view(np.uint32).reshape(P, WORDS)
    ok = all(np.array_equal(got[r], pattern(r)) for r in range(P))
    flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(json.dumps({"world": P, "multicast": True, "words_per_rank": WORDS, "ok": bool(flag.item())}))
    dist.destroy_process_group()
    sys.exit(0 if flag.item() else 1)


if __name__ == "__main__":
    main()
