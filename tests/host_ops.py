"""Test-only stand-ins for the sm_100a kernels with the kernels' numeric contract, so the
multi-rank host protocols (exchange, sharded sampler, per-rank runner) run on CPU over gloo.
They are built on the oracle (oracle/comm_ref.py) and are never used by the product path."""

import numpy as np
import torch

from oracle import comm_ref


class OracleOps:
    """exchange.CudaOps stand-in; results are rounded to the tensors' own dtype (float64
    tensors get the oracle's float64 bits, like the f64 kernels)."""

    name = "oracle"

    def __init__(self, cr, delta, method="lexsort"):
        self.cr, self.delta, self.method = cr, delta, method

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
            c, _, r, s_full, s_topk = comm_ref.gate(g, st, self.method)
            i, v = comm_ref.topk(g, self.cr, self.method)
            idx[j] = torch.from_numpy(i.astype(np.int32))
            val[j] = torch.from_numpy(v).to(val.dtype)
            norms2[j, 0], norms2[j, 1] = s_full, s_topk
            decision[j], rho[j] = int(c), r
            if tile_off is not None:
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
                lo = int(row_ptr[j])
                hi = lo + int(tile_off[j, -1]) if tile_off is not None else int(row_ptr[j + 1])
                flat_i, flat_v = idx.reshape(-1), val.reshape(-1)
                payloads.append((dim, flat_i[lo:hi].numpy().astype(np.int64), flat_v[lo:hi].numpy().astype(np.float64)))
            else:
                payloads.append(dense[j, :dim].numpy().astype(np.float64))
        agg = comm_ref.aggregate(payloads, weights)
        if out is not None:
            out.copy_(torch.from_numpy(agg).to(out.dtype))
        if params is not None:
            p = params.numpy().astype(np.float64)
            b = None if first_step else momentum_buf.numpy().astype(np.float64)
            p, b = comm_ref.sgd_momentum(p, b, agg, lr, momentum, weight_decay)
            params.copy_(torch.from_numpy(p).to(params.dtype))
            momentum_buf.copy_(torch.from_numpy(b).to(momentum_buf.dtype))
        return out

    def sgd(self, params, buf, grad, lr, momentum, weight_decay, first):
        p = params.numpy().astype(np.float64)
        b = None if first else buf.numpy().astype(np.float64)
        p, b = comm_ref.sgd_momentum(p, b, grad.numpy().astype(np.float64), lr, momentum, weight_decay)
        params.copy_(torch.from_numpy(p).to(params.dtype))
        buf.copy_(torch.from_numpy(b).to(buf.dtype))


class NumpySamplerOps:
    """Stand-in for kernels.{resolve_stream_rows, inject_rows, gather_batch}."""

    @staticmethod
    def resolve_stream_rows(head, b, out_ptr, pool_ptr, pool_rows, total, out):
        for d in range(head.numel()):
            lo, n = int(pool_ptr[d]), int(pool_ptr[d + 1] - pool_ptr[d])
            for i in range(int(b[d])):
                out[int(out_ptr[d]) + i] = pool_rows[lo + (int(head[d]) + i) % n]

    @staticmethod
    def inject_rows(base_ptr, base_rows, senders, pick_ptr, picks, out_ptr, out_rows):
        n_dev = base_ptr.numel() - 1
        for d in range(n_dev):
            o = int(out_ptr[d])
            own = base_rows[int(base_ptr[d]):int(base_ptr[d + 1])]
            out_rows[o:o + own.numel()] = own
            o += own.numel()
            for k in range(senders.numel()):
                s = int(senders[k])
                if s == d:
                    continue
                for q in range(int(pick_ptr[k]), int(pick_ptr[k + 1])):
                    out_rows[o] = base_rows[int(base_ptr[s]) + int(picks[q])]
                    o += 1

    @staticmethod
    def gather_batch(train_x, augment, train_y, rows, x_out, y_out):
        r = rows.long()
        x_out.copy_(train_x[r] + augment[r] if augment is not None else train_x[r])
        if y_out is not None:
            y_out.copy_(train_y[r])
