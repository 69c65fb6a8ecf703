"""CPU, world_size 2 over gloo: the pool-sharded sampler protocol (SURVEY §8(f) rank 4,
streams.ShardedSampler) with the three sampler kernels replaced by a numpy stand-in that has
their contract.  Each rank holds only its devices' train rows; injected samples move by one
padded all-gather per step.  Every rank's batches must equal, bit for bit, the replicated
sampler's batches for the same devices (and the reference's datagen.inject order, which
tests/test_gpu_dropin.py pins on the GPU)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from host_ops import NumpySamplerOps
from paper_2301_08897_b200 import streams

N_TRAIN, F, LABELS, N_DEV, LPD = 1_200, 24, 100, 8, 25
RATES = [31, 30, 1, 30, 42, 66, 22, 14]


def data():
    rng = np.random.default_rng(0)
    train_x = rng.standard_normal((N_TRAIN, F))
    train_y = rng.integers(0, LABELS, N_TRAIN)
    augment = rng.standard_normal((N_TRAIN, F)) * 0.01
    pools = streams.partition(train_y, N_DEV, "noniid", LPD, seed=1)
    return train_x, train_y, augment, pools


def batches(sampler_stage, steps=8):
    rates = [r * 2 for r in RATES]
    b = [min(max(r, 8), 1024) for r in rates]
    bufs = [streams.StreamBuffer(r) for r in rates]
    pick_rng = np.random.default_rng(2)
    out = []
    for it in range(steps):
        wait = max(streams.streaming_wait(len(q), b[d], rates[d]) for d, q in enumerate(bufs))
        for q in bufs:
            q.enqueue_arrivals(wait)
        draws = [q.draw_batch(b[d]) for d, q in enumerate(bufs)]
        ab = [(0.5, 0.5), (0.25, 0.25), (0.1, 0.1), (0.0, 0.0)][it % 4]
        plan = streams.injection_plan(N_DEV, ab[0], ab[1], b, seed=100 + it) if ab[0] else None
        picks = streams.injection_picks(plan, b, pick_rng) if plan else None
        x, y, ptr = sampler_stage(draws, plan, picks)
        out.append((x.numpy().copy(), y.numpy().copy(), np.asarray(ptr).copy()))
    return out


def run(rank, world, port, result):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    train_x, train_y, augment, pools = data()
    k = N_DEV // world
    sh = streams.ShardedSampler(train_x, train_y, pools, rank * k, k, ops=NumpySamplerOps())
    sh.set_augmentation(augment)
    result[rank] = (batches(sh.stage), int(sh._rows.size))
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_sampler_two_ranks_match_replicated():
    train_x, train_y, augment, pools = data()
    rep = streams.DeviceSampler(train_x, train_y, pools, ops=NumpySamplerOps())
    rep.set_augmentation(augment)
    want = batches(rep.stage)
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        res = mgr.dict()
        port = free_port()
        procs = [ctx.Process(target=run, args=(r, 2, port, res)) for r in range(2)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(timeout=240)
            assert p.exitcode == 0
        res = dict(res)
    k = N_DEV // 2
    for rank in range(2):
        got, nrows = res[rank]
        assert nrows < N_TRAIN  # the shard, not the replicated set
        lo = rank * k
        for (x, y, ptr), (xr, yr, pr) in zip(got, want):
            a, z = int(pr[lo]), int(pr[lo + k])
            assert np.array_equal(ptr + a, pr[lo:lo + k + 1])
            assert np.array_equal(x.view(np.uint64), xr[a:z].view(np.uint64))
            assert np.array_equal(y, yr[a:z])


def test_empty_pool_raises_like_reference():
    """engine.py:224-227 evaluates a % len(pool): an empty pool is a ZeroDivisionError."""
    pools = [np.arange(5), np.zeros(0, dtype=np.int64)]
    s = streams.DeviceSampler(np.zeros((5, 2)), np.zeros(5), pools, ops=NumpySamplerOps())
    s.stage([range(0, 3), range(0, 0)])  # an empty pool that draws nothing is fine
    with pytest.raises(ZeroDivisionError):
        s.stage([range(0, 3), range(0, 2)])
