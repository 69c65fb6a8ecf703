"""CPU, world_size 2 over gloo: the multi-GPU exchange protocol of exchange.GradientExchange
(decision all-gather -> sparse all-gather + merge, or local partial + all-reduce) driven with
oracle-backed test ops in place of the CUDA kernels.  Checks both ranks end bit-identical
and equal to the single-process result (sparse path) or within the fp32 tolerance (dense
all-reduce path, whose cross-rank fold order differs from the reference by design)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import comm_ref

D, W = 20_011, 4
RATES = [43, 63, 25, 73]


class OracleOps:
    """Test-only stand-in for exchange.CudaOps with the kernels' numeric contract."""

    name = "oracle"

    def __init__(self, cr, delta):
        self.cr, self.delta = cr, delta

    def make_states(self, records):
        return records.copy()

    def gate_records(self, states):
        return states.copy()

    def topk_gate(self, bucket, dim, m, states, out, tile_off=None):
        idx, val, norms2, decision, rho = out
        for j in range(bucket.shape[0]):
            st = comm_ref.GateState(self.cr, self.delta, float(states[j]["ewma_factor"]), bool(states[j]["raw_gate"]))
            st.ewma_full, st.ewma_topk = float(states[j]["ewma_full"]), float(states[j]["ewma_topk"])
            st.initialized = bool(states[j]["initialized"])
            st.n_compressed, st.n_uncompressed = int(states[j]["n_compressed"]), int(states[j]["n_uncompressed"])
            g = bucket[j, :dim].numpy().astype(np.float64)
            c, _, r, s_full, s_topk = comm_ref.gate(g, st, "threshold")
            i, v = comm_ref.topk(g, self.cr, "threshold")
            idx[j] = torch.from_numpy(i.astype(np.int32))
            val[j] = torch.from_numpy(v.astype(np.float32))
            norms2[j, 0], norms2[j, 1] = s_full, s_topk
            decision[j], rho[j] = int(c), r
            if tile_off is not None:  # the merge offsets sg_topk_gate_f32 produces
                edges = np.arange(tile_off.shape[1], dtype=np.int64) * 4096
                tile_off[j] = torch.from_numpy(np.searchsorted(i, edges).astype(np.int32))
            for f in ("ewma_full", "ewma_topk", "n_compressed", "n_uncompressed"):
                states[j][f] = getattr(st, f)
            states[j]["initialized"] = 1

    def aggregate(self, weights, dim, compressed=None, dense=None, idx=None, val=None, row_ptr=None, tile_off=None,
                  out=None, params=None, momentum_buf=None, lr=0.0, momentum=0.0, weight_decay=0.0, first_step=False):
        payloads = []
        for j in range(len(weights)):
            if compressed is not None and int(compressed[j]):
                # with tile offsets only the row starts are read (rows may sit apart)
                lo = int(row_ptr[j])
                hi = lo + int(tile_off[j, -1]) if tile_off is not None else int(row_ptr[j + 1])
                flat_i, flat_v = idx.reshape(-1), val.reshape(-1)
                payloads.append((dim, flat_i[lo:hi].numpy().astype(np.int64), flat_v[lo:hi].numpy().astype(np.float64)))
            else:
                payloads.append(dense[j, :dim].numpy().astype(np.float64))
        agg = comm_ref.aggregate(payloads, weights)
        if out is not None:
            out.copy_(torch.from_numpy(agg.astype(np.float32)))
        if params is not None:
            p = params.numpy().astype(np.float64)
            b = None if first_step else momentum_buf.numpy().astype(np.float64)
            p, b = comm_ref.sgd_momentum(p, b, agg, lr, momentum, weight_decay)
            params.copy_(torch.from_numpy(p.astype(np.float32)))
            momentum_buf.copy_(torch.from_numpy(b.astype(np.float32)))
        return out

    def sgd(self, params, buf, grad, lr, momentum, weight_decay, first):
        p = params.numpy().astype(np.float64)
        b = None if first else buf.numpy().astype(np.float64)
        p, b = comm_ref.sgd_momentum(p, b, grad.numpy().astype(np.float64), lr, momentum, weight_decay)
        params.copy_(torch.from_numpy(p.astype(np.float32)))
        buf.copy_(torch.from_numpy(b.astype(np.float32)))


def grads(family, step):
    rng = np.random.default_rng(100 + step)
    out = []
    for j in range(W):
        z = rng.standard_normal(D)
        heavy = np.sign(z) * np.exp(1.5 * rng.standard_normal(D))
        g = {"heavy": heavy, "normal": z, "mixed": heavy if j % 2 else z}[family]
        out.append((g * (1 + 0.1 * j)).astype(np.float32))
    return out


def run(rank, world, family, cr, delta, steps, port, result):
    from paper_2301_08897_b200 import exchange

    group = None
    if world > 1:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        group = dist.group.WORLD
    ex = exchange.GradientExchange(D, W, cr=cr, delta=delta, momentum=0.9, weight_decay=1e-4, group=group,
                                   ops=OracleOps(cr, delta), device=torch.device("cpu"))
    w = comm_ref.rate_weights(RATES)
    paths = []
    for s in range(steps):
        gs = grads(family, s)
        for j in range(ex.k):
            ex.bucket[j, :D] = torch.from_numpy(gs[ex.lo + j])
        paths.append(ex.step(w, 0.05, keep_aggregate=True).path)
    result[rank] = (ex.params.numpy().copy(), ex.aggregate.numpy().copy(), paths, ex.volume())
    if group is not None:
        dist.barrier()
        dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("family,cr,delta,path", [("heavy", 0.01, 0.5, "sparse-allgather"),
                                                  ("normal", 0.01, 0.3, "dense-allreduce"),
                                                  ("mixed", 0.1, 0.5, "dense-allreduce")])
def test_two_rank_protocol(family, cr, delta, path):
    single = {}
    run(0, 1, family, cr, delta, 3, 0, single)
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        res = mgr.dict()
        port = free_port()
        procs = [ctx.Process(target=run, args=(r, 2, family, cr, delta, 3, port, res)) for r in range(2)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(timeout=240)
            assert p.exitcode == 0
        res = dict(res)
    p0, a0, paths0, vol0 = res[0]
    p1, a1, paths1, vol1 = res[1]
    assert paths0 == paths1 == [path] * 3
    assert np.array_equal(p0, p1) and np.array_equal(a0, a1)  # replicas identical (engine.py:284-286)
    ps, as_, _, vols = single[0]
    # accounting: the two ranks' workers together sent what the single process sent
    assert (vol0[0] + vol1[0], vol0[1] + vol1[1]) == vols
    if path == "sparse-allgather":
        assert np.array_equal(p0, ps) and np.array_equal(a0, as_)
    else:
        scale = np.abs(as_.astype(np.float64)).max()
        assert np.max(np.abs(a0.astype(np.float64) - as_)) <= 1e-5 * scale
        assert np.linalg.norm(p0.astype(np.float64) - ps) <= 1e-5 * np.linalg.norm(ps)
