"""torchrun probe: symmetric-memory rendezvous, peer views and device barriers on this box."""
import os

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    t = symm_mem.empty(1 << 20, dtype=torch.int32, device=dev)
    t.fill_(rank + 1)
    h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
    print(rank, "handle", type(h).__name__, [n for n in dir(h) if not n.startswith("_")], flush=True)
    h.barrier(channel=0)
    peer = h.get_buffer((rank + 1) % world, (1 << 20,), torch.int32)
    print(rank, "peer sum", int(peer.sum().item()), "ptrs", [hex(p) for p in h.buffer_ptrs], flush=True)
    # a peer read inside a torch kernel, and a raw-pointer offset
    local_ptr, peer_ptr = h.buffer_ptrs[rank], h.buffer_ptrs[(rank + 1) % world]
    print(rank, "delta words", (peer_ptr - local_ptr) // 4, flush=True)
    from torch._C._distributed_c10d import _SymmetricMemory as S
    try:
        print(rank, "device multicast support", S.has_multicast_support(torch._C._autograd.DeviceType.CUDA, local), flush=True)
    except Exception as e:  # noqa: BLE001
        print(rank, "has_multicast_support(device) failed", repr(e), flush=True)
    try:
        print(rank, "handle multicast_ptr", h.multicast_ptr, flush=True)
    except Exception as e:  # noqa: BLE001
        print(rank, "multicast_ptr failed", repr(e), flush=True)
    h.barrier(channel=0)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
