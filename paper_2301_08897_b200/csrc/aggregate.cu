// Weighted aggregation with decompression (item 2 + sparse merge-densify) and momentum SGD.
//
// Replaces reference pkg/src/streamsgd/comm.py:67-78 (weighted_aggregate: acc = zeros(D);
// for each worker in order acc += w_j * densify(g_j)), comm.py:45-50 (densify) and
// nn.py:161-172 (sgd_momentum_step).
//
// Output-tile merge: every CTA owns one 4096-element output tile; each thread owns 16
// positions (four 16-byte groups, coalesced) and keeps their float64 accumulators in
// registers.  Workers are folded in ascending order:
//   dense worker   -> 128-bit streaming loads of its tile (next dense worker prefetched),
//                     acc = acc + w*x;
//   sparse worker  -> its (idx, val) pairs inside the tile (located by a per-worker tile
//                     offset table: from sg_topk_gate's writer or k_tile_offsets) are staged
//                     in shared memory for ALL sparse workers with one batched load, then
//                     scattered into a zeroed shared tile S, and every thread adds w*S[q] for
//                     its positions and re-zeroes them.
// Positions a sparse worker does not keep contribute w*(+0.0) in the reference: adding a
// zero to an accumulator that starts at +0.0 (and therefore is never -0.0) is the identity,
// so S = 0 there reproduces it bit-for-bit.  All arithmetic is binary64 round-to-nearest
// without contraction, i.e. numpy's `acc += weight * densify(g)` on the upcast inputs; the
// single rounding to the output type happens at the store.  With params/buf the momentum
// step runs in the epilogue on the unrounded float64 aggregate (nn.py:169-171 order), with
// p and buf loaded in the prologue so their latency overlaps the fold.  No atomics: the
// result is deterministic and identical on every rank.
#include "common.cuh"

namespace sg {

constexpr int AG_THREADS = 256;
constexpr int AG_TILE = 4096;
constexpr int AG_GROUPS = 4;  // 4 groups of 4 consecutive elements per thread

template <typename TI> struct AgTraits;
template <> struct AgTraits<float> { static constexpr int ECAP = 4096; };
template <> struct AgTraits<double> { static constexpr int ECAP = 1024; };

template <typename TI> SG_DEV void load4(const TI* p, double (&o)[4]);
template <> SG_DEV void load4<float>(const float* p, double (&o)[4]) {
    const float4 v = ld_stream(reinterpret_cast<const float4*>(p));
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}
template <> SG_DEV void load4<double>(const double* p, double (&o)[4]) {
    const double2 a = ld_stream(reinterpret_cast<const double2*>(p));
    const double2 b = ld_stream(reinterpret_cast<const double2*>(p) + 1);
    o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
}
template <typename TO> SG_DEV void load4_rw(const TO* p, double (&o)[4]);
template <> SG_DEV void load4_rw<float>(const float* p, double (&o)[4]) {
    const float4 v = *reinterpret_cast<const float4*>(p);
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}
template <> SG_DEV void load4_rw<double>(const double* p, double (&o)[4]) {
    const double2 a = reinterpret_cast<const double2*>(p)[0];
    const double2 b = reinterpret_cast<const double2*>(p)[1];
    o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
}
// Raw 4-element loads (no conversion): streaming for read-once inputs, cached for p/buf.
template <typename T> SG_DEV void stream4(const T* p, T (&o)[4]);
template <> SG_DEV void stream4<float>(const float* p, float (&o)[4]) {
    const float4 v = ld_stream(reinterpret_cast<const float4*>(p));
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}
template <> SG_DEV void stream4<double>(const double* p, double (&o)[4]) {
    const double2 a = ld_stream(reinterpret_cast<const double2*>(p));
    const double2 b = ld_stream(reinterpret_cast<const double2*>(p) + 1);
    o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
}
template <typename T> SG_DEV void raw4(const T* p, T (&o)[4]);
template <> SG_DEV void raw4<float>(const float* p, float (&o)[4]) {
    const float4 v = *reinterpret_cast<const float4*>(p);
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}
template <> SG_DEV void raw4<double>(const double* p, double (&o)[4]) {
    const double2 a = reinterpret_cast<const double2*>(p)[0];
    const double2 b = reinterpret_cast<const double2*>(p)[1];
    o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
}
template <typename TO> SG_DEV void store4(TO* p, const double (&o)[4]);
template <> SG_DEV void store4<float>(float* p, const double (&o)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4((float)o[0], (float)o[1], (float)o[2], (float)o[3]);
}
template <> SG_DEV void store4<double>(double* p, const double (&o)[4]) {
    reinterpret_cast<double2*>(p)[0] = make_double2(o[0], o[1]);
    reinterpret_cast<double2*>(p)[1] = make_double2(o[2], o[3]);
}

// Momentum SGD on one element, nn.py:167-171 operation order in binary64.
SG_DEV void sgd_elem(double g, double& p, double& b, double lr, double mu, double wd, bool first) {
    double buf = first ? 0.0 : b;
    buf = dmul(buf, mu);
    buf = dadd(buf, dadd(g, dmul(wd, p)));
    p = dsub(p, dmul(lr, buf));
    b = buf;
}

// off[j][t] = number of row-j entries with index < t*AG_TILE, t in [0, ntiles]; one thread
// per entry writes the boundaries between its predecessor's tile and its own.
__global__ void k_tile_offsets(const uint32_t* __restrict__ idx, const long long* __restrict__ row_ptr,
                               const uint8_t* __restrict__ comp, long long ntiles, int* __restrict__ off) {
    pdl_enter();
    constexpr int U = 4;  // entries per thread per iteration (independent loads in flight)
    const int j = blockIdx.y;
    if (comp && !comp[j]) return;
    const long long r0 = row_ptr[j], nnz = row_ptr[j + 1] - r0;
    int* o = off + (long long)j * (ntiles + 1);
    const uint32_t* ix = idx + r0;
    const long long stride = (long long)gridDim.x * blockDim.x * U;
    const long long first = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * U;
    if (nnz == 0) {
        for (long long t = first / U; t <= ntiles; t += stride / U) o[t] = 0;
        return;
    }
    for (long long p0 = first; p0 < nnz; p0 += stride) {
        long long tl[U + 1];
#pragma unroll
        for (int u = 0; u <= U; ++u) {
            const long long p = p0 + u - 1;
            tl[u] = p < 0 ? -1 : (p < nnz ? (long long)(ix[p] / AG_TILE) : -2);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long p = p0 + u;
            if (p >= nnz) break;
            for (long long t = tl[u] + 1; t <= tl[u + 1]; ++t) o[t] = (int)p;
            if (p == nnz - 1)
                for (long long t = tl[u + 1] + 1; t <= ntiles; ++t) o[t] = (int)nnz;
        }
    }
}

constexpr int PEER_MAXW = 16;  // workers whose payloads may sit in other GPUs' memory

template <typename TI, typename TO> struct AggArgs {
    double w[MAX_WORKERS];
    // peer mode (sg_weighted_aggregate_peers_f32): worker j's idx/val/tile offsets are read
    // through these device pointers (possibly another GPU's memory over NVLink) instead of
    // idx/val + row_ptr[j] and off + j*(ntiles+1)
    const uint32_t* idxw[PEER_MAXW];
    const TI* valw[PEER_MAXW];
    const int* offw[PEER_MAXW];
    int peer;
    const uint8_t* comp;
    const TI* dense;
    const uint32_t* idx;
    const TI* val;
    const long long* row_ptr;
    const int* off;
    TO* out;
    TO* p;
    TO* buf;
    long long ld, dim, ntiles;
    double lr, mu, wd;
    int nw, first, vec_ok;
    int pipe;  // k_merge_ws owns all-sparse calls: k_merge then exits
    // device-side guard on a decision array (multi-GPU steps enqueue both exchange paths):
    // guard_mode 1 = run only if every guard byte is non-zero, 2 = only if some byte is zero
    const uint8_t* guard;
    int guard_n, guard_mode;
    int balance;  // k_merge_ws: cost-balanced tile ranges (else equal ranges)
    int own;        // all-sparse merge kernel: -1 by density, 0 k_merge_ws, 1 k_merge_own
    int pf;         // k_merge_own: prefetch the next tile's p / buf into L2
    int cost_j0, cost_j1;  // workers whose offsets estimate the tile costs (local memory)
    int direct;     // k_merge_ws: chunks of multi-chunk tiles fold run by run (no lists)
};

template <typename TI, typename TO>
__global__ void __launch_bounds__(AG_THREADS, 2)
k_aggregate(const AggArgs<TI, TO> a) {
    pdl_enter();
    constexpr int ECAP = AgTraits<TI>::ECAP;
    __shared__ TI S[AG_TILE];
    __shared__ uint16_t ent_pos[ECAP];
    __shared__ TI ent_val[ECAP];
    __shared__ long long s_lo[MAX_WORKERS];
    __shared__ int s_cnt[MAX_WORKERS];
    __shared__ int s_pre[MAX_WORKERS + 1];
    __shared__ uint8_t s_comp[MAX_WORKERS];
    const int tid = threadIdx.x;
    const long long tile = blockIdx.x;
    const long long tb = tile * AG_TILE;
    const bool full = a.vec_ok && tb + AG_TILE <= a.dim;
    const bool first = a.first != 0;

    // prologue: optimizer state loads in flight first, then the sparse ranges
    TO pv[AG_GROUPS][4], bv[AG_GROUPS][4];
    if (a.p && full) {
#pragma unroll
        for (int r = 0; r < AG_GROUPS; ++r) {
            const long long e = tb + r * (AG_THREADS * 4) + tid * 4;
            raw4<TO>(a.p + e, pv[r]);
            if (!first) raw4<TO>(a.buf + e, bv[r]);
            else bv[r][0] = bv[r][1] = bv[r][2] = bv[r][3] = (TO)0;
        }
    }
    for (int j = tid; j < a.nw; j += AG_THREADS) {
        const uint8_t c = a.comp ? a.comp[j] : 0;
        s_comp[j] = c;
        int n = 0;
        if (c) {
            const int* o = a.off + (long long)j * (a.ntiles + 1);
            const int lo = o[tile], hi = o[tile + 1];
            s_lo[j] = a.row_ptr[j] + lo;
            n = hi - lo;
        }
        s_cnt[j] = n;
    }
#pragma unroll
    for (int r = 0; r < AG_GROUPS; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) S[r * (AG_THREADS * 4) + tid * 4 + c] = (TI)0;
    __syncthreads();
    if (tid == 0) {
        int acc = 0;
        for (int j = 0; j < a.nw; ++j) {
            s_pre[j] = acc;
            acc += s_cnt[j];
        }
        s_pre[a.nw] = acc;
    }
    __syncthreads();
    const int E = s_pre[a.nw];

    // stage entries [e0, e0 + n) of the flattened (worker-major) tile entry list
    auto stage = [&](int e0, int n) {
        for (int q = tid; q < n; q += AG_THREADS) {
            const int e = e0 + q;
            int lo = 0, hi = a.nw;  // s_pre[lo] <= e < s_pre[hi]
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (s_pre[mid] <= e) lo = mid;
                else hi = mid;
            }
            const long long gi = s_lo[lo] + (e - s_pre[lo]);
            ent_pos[q] = (uint16_t)(a.idx[gi] - (uint32_t)tb);
            ent_val[q] = a.val[gi];
        }
    };
    int st_lo = 0, st_hi = 0;
    if (E > 0) {
        st_hi = E < ECAP ? E : ECAP;
        stage(0, st_hi);
    }
    __syncthreads();

    double acc[AG_GROUPS][4];
#pragma unroll
    for (int r = 0; r < AG_GROUPS; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = 0.0;

    TI x[AG_GROUPS][4];
    auto load_dense = [&](int j) {
        const TI* row = a.dense + (long long)j * a.ld + tb;
#pragma unroll
        for (int r = 0; r < AG_GROUPS; ++r) {
            const int e = r * (AG_THREADS * 4) + tid * 4;
            if (full) {
                stream4<TI>(row + e, x[r]);
            } else {
#pragma unroll
                for (int c = 0; c < 4; ++c) x[r][c] = tb + e + c < a.dim ? row[e + c] : (TI)0;
            }
        }
    };
    int loaded = -1;
    for (int j = 0; j < a.nw; ++j) {
        const double wj = a.w[j];
        if (!s_comp[j]) {
            if (loaded != j) load_dense(j);
            TI xc[AG_GROUPS][4];
#pragma unroll
            for (int r = 0; r < AG_GROUPS; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) xc[r][c] = x[r][c];
            // prefetch the next dense worker while folding this one
            int nxt = j + 1;
            while (nxt < a.nw && s_comp[nxt] && s_cnt[nxt] == 0) ++nxt;
            if (nxt < a.nw && !s_comp[nxt]) {
                load_dense(nxt);
                loaded = nxt;
            }
#pragma unroll
            for (int r = 0; r < AG_GROUPS; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[r][c] = dadd(acc[r][c], dmul(wj, (double)xc[r][c]));
        } else if (s_cnt[j] > 0) {
            int e = s_pre[j];
            const int e_end = e + s_cnt[j];
            while (e < e_end) {
                if (e >= st_hi) {  // uniform: refill the staging buffer
                    __syncthreads();
                    st_lo = e;
                    st_hi = (E - e) < ECAP ? E : e + ECAP;
                    stage(st_lo, st_hi - st_lo);
                    __syncthreads();
                }
                const int piece = e_end < st_hi ? e_end : st_hi;
                for (int q = e + tid; q < piece; q += AG_THREADS) S[ent_pos[q - st_lo]] = ent_val[q - st_lo];
                e = piece;
            }
            __syncthreads();
#pragma unroll
            for (int r = 0; r < AG_GROUPS; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int q = r * (AG_THREADS * 4) + tid * 4 + c;
                    const TI s = S[q];
                    acc[r][c] = dadd(acc[r][c], dmul(wj, (double)s));
                    S[q] = (TI)0;
                }
            __syncthreads();
        }
    }

    // epilogue
#pragma unroll
    for (int r = 0; r < AG_GROUPS; ++r) {
        const int e = r * (AG_THREADS * 4) + tid * 4;
        if (full) {
            if (a.out) store4<TO>(a.out + tb + e, acc[r]);
            if (a.p) {
                double pd[4], bd[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    pd[c] = (double)pv[r][c];
                    bd[c] = (double)bv[r][c];
                    sgd_elem(acc[r][c], pd[c], bd[c], a.lr, a.mu, a.wd, first);
                }
                store4<TO>(a.p + tb + e, pd);
                store4<TO>(a.buf + tb + e, bd);
            }
        } else {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const long long q = tb + e + c;
                if (q >= a.dim) continue;
                if (a.out) a.out[q] = (TO)acc[r][c];
                if (a.p) {
                    double pq = a.p[q], bq = first ? 0.0 : (double)a.buf[q];
                    sgd_elem(acc[r][c], pq, bq, a.lr, a.mu, a.wd, first);
                    a.p[q] = (TO)pq;
                    a.buf[q] = (TO)bq;
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------------------
// k_merge: the float32 fast path of k_aggregate.  512 threads; thread t owns the 8
// contiguous positions [8t, 8t+8) of the 4096-element tile.  Dense workers are folded in
// float64 registers.  Sparse workers are folded entry-driven: all of them are staged into
// shared memory with one batched load (worker-major), the running float64 tile moves to
// shared memory for the run of sparse workers, and each staged entry updates its position
// (unique within a worker, so one barrier per worker keeps the ascending-worker fold order).
// p/buf for the fused momentum-SGD step are loaded first so their latency hides under the
// fold.
// ---------------------------------------------------------------------------------------
constexpr int MP_MAXW = PEER_MAXW;
constexpr int MG_THREADS = 512;
constexpr int MG_PER = 8;
constexpr int MG_ECAP = 4096;
constexpr size_t MG_SMEM = AG_TILE * sizeof(double) + MG_ECAP * (sizeof(float) + sizeof(uint16_t)) +
                           AG_TILE * sizeof(unsigned);

template <typename TO>
__global__ void __launch_bounds__(MG_THREADS, 2)
k_merge(const AggArgs<float, TO> a) {
    pdl_enter();
    SG_STAMP(1);
    extern __shared__ __align__(128) unsigned char mg_smem[];
    double* acc_s = reinterpret_cast<double*>(mg_smem);                   // [AG_TILE]
    float* ent_val = reinterpret_cast<float*>(acc_s + AG_TILE);            // [MG_ECAP]
    uint16_t* ent_pos = reinterpret_cast<uint16_t*>(ent_val + MG_ECAP);    // [MG_ECAP]
    __shared__ long long s_lo[MAX_WORKERS];
    __shared__ int s_cnt[MAX_WORKERS];
    __shared__ int s_pre[MAX_WORKERS + 1];
    __shared__ uint8_t s_comp[MAX_WORKERS];
    const int tid = threadIdx.x;
    __shared__ int s_skip;
    if (tid == 0) {
        int all = a.pipe && a.nw <= MP_MAXW;
        for (int j = 0; j < a.nw && all; ++j) all = a.comp && a.comp[j] != 0;
        if (a.guard_mode) {
            int any0 = 0;
            for (int j = 0; j < a.guard_n; ++j) any0 |= a.guard[j] == 0;
            all |= a.guard_mode == 2 ? !any0 : any0;  // guarded off
        }
        s_skip = all;
    }
    __syncthreads();
    if (s_skip) return;  // the pipelined kernel merged this call
    for (long long tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
    __syncthreads();  // shared memory of the previous tile is no longer read
    const long long tb = tile * AG_TILE;
    const int q0 = tid * MG_PER;
    const bool full = a.vec_ok && tb + AG_TILE <= a.dim;
    const bool first = a.first != 0;

    float pv[MG_PER], bv[MG_PER];
    if (a.p && full) {
        const float4* pp = reinterpret_cast<const float4*>(a.p + tb + q0);
        const float4* bp = reinterpret_cast<const float4*>(a.buf + tb + q0);
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const float4 u = pp[r];
            pv[4 * r] = u.x; pv[4 * r + 1] = u.y; pv[4 * r + 2] = u.z; pv[4 * r + 3] = u.w;
            if (!first) {
                const float4 z = bp[r];
                bv[4 * r] = z.x; bv[4 * r + 1] = z.y; bv[4 * r + 2] = z.z; bv[4 * r + 3] = z.w;
            } else {
                bv[4 * r] = bv[4 * r + 1] = bv[4 * r + 2] = bv[4 * r + 3] = 0.f;
            }
        }
    }
    for (int j = tid; j < a.nw; j += MG_THREADS) {
        const uint8_t c = a.comp ? a.comp[j] : 0;
        s_comp[j] = c;
        int n = 0;
        if (c) {
            const int* o = a.off + (long long)j * (a.ntiles + 1);
            const int lo = o[tile], hi = o[tile + 1];
            s_lo[j] = a.row_ptr[j] + lo;
            n = hi - lo;
        }
        s_cnt[j] = n;
    }
    __syncthreads();
    if (tid < 32) {  // exclusive scan of the per-worker entry counts (nw <= 64)
        const int lane = tid;
        const int c0 = lane < a.nw ? s_cnt[lane] : 0;
        const int c1 = lane + 32 < a.nw ? s_cnt[lane + 32] : 0;
        int i0 = c0, i1 = c1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y0 = __shfl_up_sync(FULL, i0, o), y1 = __shfl_up_sync(FULL, i1, o);
            if (lane >= o) {
                i0 += y0;
                i1 += y1;
            }
        }
        const int tot0 = __shfl_sync(FULL, i0, 31);
        if (lane < a.nw) s_pre[lane] = i0 - c0;
        if (lane + 32 < a.nw) s_pre[lane + 32] = tot0 + i1 - c1;
        if (lane == 31) s_pre[a.nw] = a.nw <= 32 ? tot0 : tot0 + i1;
    }
    __syncthreads();
    const int E = s_pre[a.nw];
    int st_lo = 0, st_hi = 0;  // staged entry window [st_lo, st_hi) (whole workers)
    auto fill = [&](int j0) {
        int j1 = j0;
        while (j1 < a.nw && s_pre[j1 + 1] - s_pre[j0] <= MG_ECAP) ++j1;
        if (j1 == j0) j1 = j0 + 1;  // cannot happen for f32 (<= 4096 entries per worker)
        const int e0 = s_pre[j0], e1 = s_pre[j1];
        for (int q = tid; q < e1 - e0; q += MG_THREADS) {
            const int e = e0 + q;
            int lo = j0, hi = j1;  // s_pre[lo] <= e < s_pre[hi]
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (s_pre[mid] <= e) lo = mid;
                else hi = mid;
            }
            const long long gi = s_lo[lo] + (e - s_pre[lo]);
            ent_pos[q] = (uint16_t)(a.idx[gi] - (uint32_t)tb);
            ent_val[q] = a.val[gi];
        }
        st_lo = e0;
        st_hi = e1;
    };
    if (E > 0) fill(0);

    double acc[MG_PER];
#pragma unroll
    for (int c = 0; c < MG_PER; ++c) acc[c] = 0.0;
    bool all_sparse = a.nw <= 32 && E <= MG_ECAP;
    for (int j = 0; j < a.nw && all_sparse; ++j) all_sparse = s_comp[j] != 0;
    if (all_sparse) {
        // Fast path (every worker sparse, whole tile staged): one pass records which workers
        // touch each position; positions with one contributor take +0 + w*v directly, the
        // rare collided ones are folded in ascending worker order by their lowest worker.
        // who[q]: bitmask of the workers keeping position q; acc_s[q] is written only for
        // touched positions and read only where the mask is non-zero.
        unsigned* who = reinterpret_cast<unsigned*>(ent_pos + MG_ECAP);
        *reinterpret_cast<uint4*>(who + q0) = make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4*>(who + q0 + 4) = make_uint4(0, 0, 0, 0);
        __syncthreads();
        for (int e = tid; e < E; e += MG_THREADS) {
            int lo = 0, hi = a.nw;
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (s_pre[mid] <= e) lo = mid;
                else hi = mid;
            }
            atomicOr(&who[ent_pos[e]], 1u << lo);
        }
        __syncthreads();
        for (int e = tid; e < E; e += MG_THREADS) {
            int lo = 0, hi = a.nw;
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (s_pre[mid] <= e) lo = mid;
                else hi = mid;
            }
            const int q = ent_pos[e];
            const unsigned m = who[q];
            double r;
            if ((m & (m - 1)) == 0) {
                r = dadd(0.0, dmul(a.w[lo], (double)ent_val[e]));
            } else {
                if (__ffs(m) - 1 != lo) continue;  // the lowest contributor folds the position
                r = 0.0;
                for (unsigned mm = m; mm; mm &= mm - 1) {
                    const int j = __ffs(mm) - 1;
                    int l = s_pre[j], h = s_pre[j + 1];  // entry of worker j at position q
                    while (l < h) {
                        const int mid = (l + h) >> 1;
                        if ((int)ent_pos[mid] < q) l = mid + 1;
                        else h = mid;
                    }
                    r = dadd(r, dmul(a.w[j], (double)ent_val[l]));
                }
            }
            acc_s[q] = r;
        }
        __syncthreads();
#pragma unroll
        for (int c = 0; c < MG_PER; ++c) {
            const int q = q0 + c;
            if (who[q]) acc[c] = acc_s[q];
        }
    }
    bool in_smem = false;  // uniform: the running tile lives in acc_s during a sparse run
    for (int j = 0; j < (all_sparse ? 0 : a.nw); ++j) {
        const double wj = a.w[j];
        if (!s_comp[j]) {
            float x[MG_PER];
            const float* row = a.dense + (long long)j * a.ld + tb + q0;
            if (full) {
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const float4 u = reinterpret_cast<const float4*>(row)[r];
                    x[4 * r] = u.x; x[4 * r + 1] = u.y; x[4 * r + 2] = u.z; x[4 * r + 3] = u.w;
                }
            } else {
#pragma unroll
                for (int c = 0; c < MG_PER; ++c) x[c] = tb + q0 + c < a.dim ? row[c] : 0.f;
            }
            if (in_smem) {
                __syncthreads();
#pragma unroll
                for (int c = 0; c < MG_PER; ++c) acc[c] = acc_s[q0 + c];
                in_smem = false;
            }
#pragma unroll
            for (int c = 0; c < MG_PER; ++c) acc[c] = dadd(acc[c], dmul(wj, (double)x[c]));
        } else if (s_cnt[j] > 0) {
            if (!in_smem) {
#pragma unroll
                for (int c = 0; c < MG_PER; ++c) acc_s[q0 + c] = acc[c];
                in_smem = true;
            }
            __syncthreads();  // previous worker's updates (and the staging) are complete
            if (s_pre[j] >= st_hi) {
                fill(j);
                __syncthreads();
            }
            const int e0 = s_pre[j] - st_lo, e1 = e0 + s_cnt[j];
            for (int e = e0 + tid; e < e1; e += MG_THREADS) {
                const int q = ent_pos[e];
                acc_s[q] = dadd(acc_s[q], dmul(wj, (double)ent_val[e]));
            }
        }
    }
    if (in_smem) {
        __syncthreads();
#pragma unroll
        for (int c = 0; c < MG_PER; ++c) acc[c] = acc_s[q0 + c];
    }
    if (full) {
        if (a.out) {
            float4* op = reinterpret_cast<float4*>(a.out + tb + q0);
#pragma unroll
            for (int r = 0; r < 2; ++r)
                op[r] = make_float4((float)acc[4 * r], (float)acc[4 * r + 1], (float)acc[4 * r + 2], (float)acc[4 * r + 3]);
        }
        if (a.p) {
            float4* pp = reinterpret_cast<float4*>(a.p + tb + q0);
            float4* bp = reinterpret_cast<float4*>(a.buf + tb + q0);
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                double pd[4], bd[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    pd[c] = (double)pv[4 * r + c];
                    bd[c] = (double)bv[4 * r + c];
                    sgd_elem(acc[4 * r + c], pd[c], bd[c], a.lr, a.mu, a.wd, first);
                }
                pp[r] = make_float4((float)pd[0], (float)pd[1], (float)pd[2], (float)pd[3]);
                bp[r] = make_float4((float)bd[0], (float)bd[1], (float)bd[2], (float)bd[3]);
            }
        }
    } else {
#pragma unroll
        for (int c = 0; c < MG_PER; ++c) {
            const long long q = tb + q0 + c;
            if (q >= a.dim) continue;
            if (a.out) a.out[q] = (TO)acc[c];
            if (a.p) {
                double pq = a.p[q], bq = first ? 0.0 : (double)a.buf[q];
                sgd_elem(acc[c], pq, bq, a.lr, a.mu, a.wd, first);
                a.p[q] = (TO)pq;
                a.buf[q] = (TO)bq;
            }
        }
    }
    }  // tile loop
}

// ---------------------------------------------------------------------------------------
// k_merge_ws: persistent, warp-specialised merge + fused momentum SGD for the case the hot
// path produces (every worker sparse, float32, <= 16 workers).  One CTA per SM owns the
// tiles b, b + G, b + 2G, ... (G = grid; round-robin, so concentrated regions of kept entries --
// real gradients put most of them in a few layers -- spread evenly over the CTAs); a tile's
// entries (worker-major, ascending index
// inside a worker) are processed in chunks of <= MW_ECAP entries (one unless oversized).
//   producer warps (12): warp w stages worker w's run (w < nw) of the next chunk with
//     cp.async (LDGSTS) while, for the current chunk, (1) each entry is pushed onto its
//     position's list, head[q] <- atomicExch(head[q], node), node = {value, worker, next};
//     (2) each list's head entry folds the list in ascending worker order -- the reference's
//     fold (comm.py:70-78): +0 (or the previous chunk's partial), then + w_j * v_j -- into
//     the tile's float64 value slot and marks the position.  A named-barrier arrive hands
//     the tile (values + byte marks, double-buffered) to the consumers.
//   consumer warps (16): p/buf tiles arrive by TMA bulk copies (cp.async.bulk, mbarrier
//     completion, L2 evict-first) into a 3-stage shared ring; thread t owns positions
//     {4t..4t+3} and {2048+4t..+3}: g = marked ? value : +0, momentum SGD (nn.py:167-171
//     order, binary64), 128-bit global stores; marks are cleared and the hand-off buffer
//     and ring stage released.
// The streaming SGD never waits on a CTA-wide barrier.
// ---------------------------------------------------------------------------------------
constexpr int MW_CONS = 512;
#ifndef SG_MW_PROD  // producer threads of k_merge_ws (diagnostic builds may override)
#define SG_MW_PROD 384
#endif
constexpr int MW_PROD = SG_MW_PROD;
constexpr int MW_PW = MW_PROD / 32;
constexpr int MW_THREADS = MW_CONS + MW_PROD;
constexpr int MW_ECAP = 1024;
constexpr int MW_STAGES = 3;
constexpr int MW_SLOTS = 3;  // entry staging: two chunks in flight ahead of the one processed
constexpr int MW_HALF = AG_TILE / 2;
constexpr unsigned MW_NIL = 0xffffu;
enum { BAR_FULL = 1, BAR_EMPTY = 3, BAR_PROD = 5, BAR_CONS = 6 };

constexpr unsigned long long MW_BASE = 1024;  // a tile's streaming cost, in entry-equivalents

inline size_t mw_smem_bytes() {
    return (size_t)MW_STAGES * 2 * AG_TILE * sizeof(float)             // p/buf ring [S][2][TILE]
           + 2 * AG_TILE * sizeof(double)                                // values [2][TILE]
           + (size_t)AG_TILE * sizeof(unsigned)                          // heads [TILE]
           + (size_t)MW_ECAP * sizeof(uint2)                             // nodes [ECAP]
           + MW_SLOTS * (size_t)MW_ECAP * (sizeof(uint32_t) + sizeof(float) + 1)  // staging + worker ids
           + 2 * AG_TILE;                                                // marks [2][TILE]
}

// All-sparse merges with >= MO_DENSITY kept entries per position on average (e.g. cr 0.1)
// take k_merge_own, the sparser ones k_merge_ws; both fold in the same order, so the choice
// (made on the device from the tile offsets of workers cost_j0..cost_j1, this GPU's own on the
// peer path) never changes a result.
constexpr double MO_DENSITY = 0.2;
// Warp-cooperative (call from a whole warp): 1 if every worker compressed and the sparse
// merge of this call belongs to the kernel that asked (want_dense: k_merge_own), else 0.
// One load per lane, so the test costs one round trip.
template <typename TO>
SG_DEV int sparse_merge_is_mine(const AggArgs<float, TO>& a, bool want_dense) {
    const int lane = threadIdx.x & 31, nw = a.nw;
    if (nw > MP_MAXW) return 0;
    const bool comp = lane >= nw || a.comp[lane] != 0;
    long long part = 0;
    if (a.own < 0 && lane >= a.cost_j0 && lane < a.cost_j1) {
        const long long ntl = a.ntiles;
        part = a.peer ? (long long)(a.offw[lane][ntl] - a.offw[lane][0])
                      : (long long)(a.off[(long long)lane * (ntl + 1) + ntl] - a.off[(long long)lane * (ntl + 1)]);
    }
    const bool all_comp = __all_sync(FULL, comp);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(FULL, part, o);
    bool dense;
    if (a.own >= 0) {
        dense = a.own != 0;
    } else {
        const int nl = a.cost_j1 - a.cost_j0;
        dense = nl > 0 && (double)part * (double)nw >= MO_DENSITY * (double)a.dim * (double)nl;
    }
    return all_comp && dense == want_dense;
}

inline int mw_direct() {  // SG_MW_DIRECT=0: every chunk through the position lists (A/B runs)
    static const int v = [] {
        const char* e = getenv("SG_MW_DIRECT");
        return (e && *e == '0') ? 0 : 1;
    }();
    return v;
}

// Cost-balanced merge tile ranges (always on; the equal-range split was the round-1 ablation).
inline int mw_balance() { return 1; }
inline int merge_mode(int m) { return m < 0 ? -1 : (m > 0 ? 1 : 0); }

// One CTA per SM over cost-balanced contiguous tile ranges.
inline int mw_grid(long long ntiles, int sms) { return (int)(ntiles < sms ? ntiles : sms); }

template <typename TO>
__global__ void __launch_bounds__(MW_THREADS, 1)
k_merge_ws(const AggArgs<float, TO> a) {
    pdl_enter();
    SG_STAMP(0);
    extern __shared__ __align__(128) unsigned char mw_smem[];
    float* ring = reinterpret_cast<float*>(mw_smem);                     // [S][2][TILE]
    double* acc = reinterpret_cast<double*>(ring + MW_STAGES * 2 * AG_TILE);  // [2][TILE]
    uint2* node = reinterpret_cast<uint2*>(acc + 2 * AG_TILE);           // [ECAP]
    uint32_t* sidx = reinterpret_cast<uint32_t*>(node + MW_ECAP);        // [SLOTS][ECAP]
    float* sval = reinterpret_cast<float*>(sidx + MW_SLOTS * MW_ECAP);   // [SLOTS][ECAP]
    unsigned* head = reinterpret_cast<unsigned*>(sval + MW_SLOTS * MW_ECAP);  // [TILE]
    uint8_t* mark = reinterpret_cast<uint8_t*>(head + AG_TILE);          // [2][TILE]
    uint8_t* swk = mark + 2 * AG_TILE;                                   // [SLOTS][ECAP] worker ids
    constexpr int OR = 8;                    // tile-offset ring: filled 4 tiles ahead of the cursor
    __shared__ int so_lo[OR][MP_MAXW];       // worker j's merge offsets at the tile's two edges
    __shared__ int so_hi[OR][MP_MAXW];
    __shared__ int4 s_hdr[MW_SLOTS];  // staged chunk: {tile, c0, entries, last}
    __shared__ int s_direct[MW_SLOTS];  // staged chunk folds run by run (long worker runs)
    __shared__ __align__(8) unsigned long long fullb[MW_STAGES];
    __shared__ const uint32_t* s_ib[MP_MAXW];  // worker j's entries (local, or a peer GPU's)
    __shared__ const float* s_vb[MP_MAXW];
    __shared__ int s_ok;
    const int tid = threadIdx.x;
    const int nw = a.nw;
    if (tid < 32) {
        const int mine = sparse_merge_is_mine(a, false);
        if (tid == 0) s_ok = mine;
    }
    __syncthreads();
    if (!s_ok) return;  // not all-sparse (k_merge), or dense payloads (k_merge_own)
    // ---- this CTA's contiguous tile range, balanced by cost ------------------------------
    // cost(tile) = MW_BASE + entries of all workers in the tile.  Real gradients put most kept
    // entries in a few layers; equal-cost contiguous ranges give those tiles to many CTAs
    // while each CTA still streams one contiguous region (the fastest order for the p/buf
    // stream).  Every CTA derives the same partition: a coarse prefix over blocks of CB tiles,
    // refined inside one block for its own two bounds.
    const long long G = gridDim.x, ntl = a.ntiles;
    const long long CB = ntl > 64LL * 1024 ? (ntl + 1023) / 1024 : 64;
    const int nblk = (int)((ntl + CB - 1) / CB);  // <= 1024
    // (scratch in the p/buf ring, which the TMA fills only after the partition is known)
    unsigned long long* s_cp = reinterpret_cast<unsigned long long*>(ring);  // [1025] cost of tiles [0, k*CB)
    unsigned long long* s_wsum = s_cp + 1032;                                 // [MW_THREADS / 32]
    __shared__ long long s_bound[2];
    auto off_at = [&](int j, long long t) -> long long {
        return a.peer ? a.offw[j][t] : a.off[(long long)j * (ntl + 1) + t];
    };
    // (the cost estimate reads the offsets of workers cost_j0..cost_j1 only -- on the peer path
    // this rank's own, so the partition needs no NVLink round trips; each rank's partition is
    // private, the tiles' results do not depend on it)
    const int cj0 = a.cost_j0, cj1 = a.cost_j1;
    const unsigned long long base = MW_BASE * (unsigned long long)(cj1 - cj0) / (unsigned long long)nw + 1;
    auto tile_cost = [&](long long t) -> unsigned long long {
        unsigned long long c = base;
        for (int j = cj0; j < cj1; ++j) c += (unsigned long long)(off_at(j, t + 1) - off_at(j, t));
        return c;
    };
    if (a.balance) {
        // coarse costs: thread t owns blocks 2t, 2t+1; block-wide inclusive scan
        unsigned long long v[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int k = 2 * tid + u;
            v[u] = 0;
            if (k < nblk) {
                const long long t0 = k * CB, t1 = t0 + CB < ntl ? t0 + CB : ntl;
                unsigned long long c = (unsigned long long)(t1 - t0) * base;
                for (int j = cj0; j < cj1; ++j) c += (unsigned long long)(off_at(j, t1) - off_at(j, t0));
                v[u] = c;
            }
        }
        const int lane = tid & 31, warp = tid >> 5;
        unsigned long long incl = v[0] + v[1];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) s_wsum[warp] = incl;
        __syncthreads();
        unsigned long long wb = 0;
        for (int i = 0; i < warp; ++i) wb += s_wsum[i];
        const unsigned long long ex = wb + incl - (v[0] + v[1]);
        if (2 * tid < nblk) s_cp[2 * tid + 1] = ex + v[0];
        if (2 * tid + 1 < nblk) s_cp[2 * tid + 2] = ex + v[0] + v[1];
        if (tid == 0) s_cp[0] = 0;
        __syncthreads();
    }
    const unsigned long long total = s_cp[nblk];
    auto coarse_of = [&](unsigned long long target) {  // s_cp[k] <= target < s_cp[k + 1]
        int lo = 0, hi = nblk;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (s_cp[mid] <= target) lo = mid;
            else hi = mid;
        }
        return lo;
    };
    long long t_begin, t_end;
    if (!a.balance) {  // equal contiguous ranges
        const long long share = (ntl + G - 1) / G;
        t_begin = blockIdx.x * share;
        t_end = t_begin + share < ntl ? t_begin + share : ntl;
    } else {
        // warps 0 and 1 refine bounds b and b + 1: the first tile whose preceding cost >= target
        const int warp = tid >> 5, lane = tid & 31;
        if (warp < 2) {
            const long long b = (long long)blockIdx.x + warp;
            long long res = ntl;
            if (b == 0) {
                res = 0;
            } else if (b < G) {
                const unsigned long long target = total * (unsigned long long)b / (unsigned long long)G;
                const int k = coarse_of(target);
                const long long t0 = k * CB, t1 = t0 + CB < ntl ? t0 + CB : ntl;
                unsigned long long run = s_cp[k];  // cost before tile t0 + (chunk start)
                res = t1;
                for (long long c0 = t0; c0 < t1; c0 += 32) {
                    const long long t = c0 + lane;
                    const unsigned long long c = t < t1 ? tile_cost(t) : 0ull;
                    unsigned long long inc = c;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const unsigned long long y = __shfl_up_sync(FULL, inc, o);
                        if (lane >= o) inc += y;
                    }
                    const unsigned long long before = run + inc - c;  // cost of tiles < t
                    const unsigned hit = __ballot_sync(FULL, t < t1 && before >= target);
                    if (hit) {
                        res = c0 + __ffs(hit) - 1;
                        break;
                    }
                    run += __shfl_sync(FULL, inc, 31);
                }
            }
            if (lane == 0) s_bound[warp] = res;
        }
        __syncthreads();
        t_begin = s_bound[0];
        t_end = s_bound[1];
    }
    if (t_begin >= t_end) return;
    const int nt = (int)(t_end - t_begin);
    auto tile_of = [&](int i) { return t_begin + i; };
    // ring stage s <- p/buf of tile i (full tiles only; a partial last tile is read directly)
    unsigned long long policy = 0;
    auto issue = [&](int i) {
        const long long tb = tile_of(i) * AG_TILE;
        const int s = i % MW_STAGES;
        if (tb + AG_TILE > a.dim) {  // the row's partial tile is read directly: just advance the phase
            mbar_arrive(&fullb[s]);
            return;
        }
        mbar_expect_tx(&fullb[s], 2 * AG_TILE * sizeof(float));
        bulk_g2s(ring + (s * 2) * AG_TILE, a.p + tb, AG_TILE * sizeof(float), &fullb[s], policy);
        bulk_g2s(ring + (s * 2 + 1) * AG_TILE, a.buf + tb, AG_TILE * sizeof(float), &fullb[s], policy);
    };
    __syncthreads();  // the partition scratch in the ring is dead
    if (tid == 0) {
        policy = policy_evict_first();
        for (int s = 0; s < MW_STAGES; ++s) mbar_init(&fullb[s], 1);
        fence_mbar_init();
        fence_proxy_async();  // generic writes to the ring before the first bulk copies into it
        for (int i = 0; i < MW_STAGES && i < nt; ++i) issue(i);
    }
    for (int q = tid; q < AG_TILE; q += MW_THREADS) head[q] = MW_NIL;
    for (int q = tid; q < 2 * AG_TILE / 4; q += MW_THREADS) reinterpret_cast<unsigned*>(mark)[q] = 0u;
    if (tid < nw) {
        s_ib[tid] = a.peer ? a.idxw[tid] : a.idx + a.row_ptr[tid];
        s_vb[tid] = a.peer ? a.valw[tid] : a.val + a.row_ptr[tid];
    }
    __syncthreads();

    if (tid >= MW_CONS) {
        // ------------------------------- producers -------------------------------
        const int pt = tid - MW_CONS, lane = pt & 31, pw = pt >> 5;
        // per-warp view of tile i: lane j < nw holds worker j's entry count and start
        // the cursor enters tile i: warp 0 fetches tile i + 4's per-worker offsets into the
        // ring (read 4 cursor advances -- and at least 4 producer barriers -- later)
        // (asynchronous: the copies join the current staging group, complete before that chunk is
        // processed and are read only when the cursor reaches the tile)
        auto prefetch_offsets = [&](int i) {
            if (pw == 0 && lane < nw && i < nt) {
                const long long t = tile_of(i);
                const int* o = a.peer ? a.offw[lane] : a.off + (long long)lane * (ntl + 1);
                cp_async4(&so_lo[i % OR][lane], o + t);
                cp_async4(&so_hi[i % OR][lane], o + t + 1);
            }
        };
        auto tile_runs = [&](int i, int& cnt, int& pre, int& tot) {
            cnt = lane < nw ? so_hi[i % OR][lane] - so_lo[i % OR][lane] : 0;
            int incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += y;
            }
            pre = incl - cnt;
            tot = __shfl_sync(FULL, incl, 31);
        };
        // Staging cursor: the next chunk to stage is entries [c0, min(E, c0 + ECAP)) of tile
        // ci (cnt/pre: the tile's per-worker runs); ci == nt marks the end.
        int ci = 0, cc0 = 0, cE, ccnt, cpre;
        for (int i = 0; i <= 4; ++i) prefetch_offsets(i);
        cp_async_commit();
        cp_async_wait<0>();
        bar_sync(BAR_PROD, MW_PROD);
        tile_runs(0, ccnt, cpre, cE);
        auto stage_next = [&](int slot) {  // stage the cursor's chunk into slot (async), advance
            if (ci < nt) {
                const int c1 = cE - cc0 < MW_ECAP ? cE : cc0 + MW_ECAP;
                for (int j = pw; j < nw; j += MW_PW) {
                    const int pj = __shfl_sync(FULL, cpre, j), nj = __shfl_sync(FULL, ccnt, j);
                    const int lo = pj > cc0 ? pj : cc0, hi = pj + nj < c1 ? pj + nj : c1;
                    const long long g0 = so_lo[ci % OR][j] - pj;
                    const uint32_t* ib = s_ib[j];
                    const float* vb = s_vb[j];
                    for (int e = lo + lane; e < hi; e += 32) {
                        SG_CHECK(e - cc0 >= 0 && e - cc0 < MW_ECAP);
                        cp_async4(sidx + slot * MW_ECAP + (e - cc0), ib + g0 + e);
                        cp_async4(sval + slot * MW_ECAP + (e - cc0), vb + g0 + e);
                        swk[slot * MW_ECAP + (e - cc0)] = (uint8_t)j;
                    }
                }
                // fold mode: tiles of more than one chunk (candidate-dense; their chunks hold a
                // few long worker runs) fold run by run.  (A per-chunk run-length test here cost
                // ~6 % of the sparse merge: it sits on the staging path of every chunk.)
                if (pt == 0) s_direct[slot] = a.direct && cE > MW_ECAP;
                if (pt == 0) s_hdr[slot] = make_int4(ci, cc0, c1 - cc0, c1 == cE);
                if (c1 < cE) {
                    cc0 = c1;
                } else {
                    ++ci;
                    cc0 = 0;
                    prefetch_offsets(ci + 4);
                    if (ci < nt) tile_runs(ci, ccnt, cpre, cE);
                }
            } else if (pt == 0) {
                s_hdr[slot] = make_int4(nt, 0, 0, 1);
            }
            cp_async_commit();  // one group per call (possibly empty) keeps the wait counts uniform
        };
        stage_next(0);
        stage_next(1);
        for (int s = 0;; ++s) {
            const int slot = s % MW_SLOTS;
            cp_async_wait<1>();
            // chunk s is visible; chunk s - 1's lists are consumed, so its slot (the one
            // restaged below), the nodes and the heads are free
            bar_sync(BAR_PROD, MW_PROD);
            const int4 hd = s_hdr[slot];
            const int i = hd.x, c0 = hd.y, ne = hd.z;
            if (i >= nt) break;
            stage_next((s + 2) % MW_SLOTS);
            const int b = i & 1;
            const uint32_t tb = (uint32_t)(tile_of(i) * AG_TILE);
            double* ab = acc + b * AG_TILE;
            uint8_t* mb = mark + b * AG_TILE;
            const uint32_t* si = sidx + slot * MW_ECAP;
            const float* sv = sval + slot * MW_ECAP;
            const uint8_t* sw8 = swk + slot * MW_ECAP;
            // Candidate-dense tiles (real gradients) give chunks of one or a few long worker
            // runs (entries [c0, c0 + ne) of the tile's worker-major order):
            // one worker's positions are distinct, so such a chunk folds run by run straight
            // into the tile (a producer barrier between runs keeps the ascending worker order)
            // -- no lists, the same operations in the same order as the list fold below.
            if (s_direct[slot]) {
                if (c0 == 0 && i >= 2) bar_sync(BAR_EMPTY + b, MW_CONS + MW_PROD);  // buffer b released
                int pre = 0, done = 0;
                for (int j = 0; j < nw; ++j) {
                    const int cnt = so_hi[i % OR][j] - so_lo[i % OR][j];
                    const int lo = pre > c0 ? pre : c0, hi = pre + cnt < c0 + ne ? pre + cnt : c0 + ne;
                    pre += cnt;
                    if (hi <= lo) continue;
                    if (done++) bar_sync(BAR_PROD, MW_PROD);  // the previous run's folds are visible
                    const double wj = a.w[j];
                    for (int n = lo - c0 + pt; n < hi - c0; n += MW_PROD) {
                        const unsigned q = si[n] - tb;
                        SG_CHECK(q < (unsigned)AG_TILE);
                        const double r = mb[q] ? ab[q] : 0.0;
                        ab[q] = dadd(r, dmul(wj, (double)sv[n]));
                        mb[q] = 1;
                    }
                }
                if (hd.w) bar_arrive(BAR_FULL + b, MW_CONS + MW_PROD);  // buffer b holds tile i's values
                continue;
            }
            // (1) push every entry onto its position's list
            for (int n = pt; n < ne; n += MW_PROD) {
                const unsigned q = si[n] - tb;
                SG_CHECK(q < (unsigned)AG_TILE);
                const float v = sv[n];
                const unsigned j = sw8[n];
                const unsigned old = atomicExch(head + q, (unsigned)n);
                node[n] = make_uint2(__float_as_uint(v), (j << 16) | (old & 0xffffu));
            }
            bar_sync(BAR_PROD, MW_PROD);
            if (c0 == 0 && i >= 2) bar_sync(BAR_EMPTY + b, MW_CONS + MW_PROD);  // buffer b released
            // (2) each list's head entry folds its position in ascending worker order
            for (int n = pt; n < ne; n += MW_PROD) {
                const unsigned q = si[n] - tb;
                const uint2 nd = node[n];
                if (head[q] != (unsigned)n) continue;
                double r = 0.0;
                if (c0 > 0 && mb[q]) r = ab[q];  // partial of an earlier chunk of this tile
                if ((nd.y & 0xffffu) == MW_NIL) {
                    r = dadd(r, dmul(a.w[nd.y >> 16], (double)__uint_as_float(nd.x)));
                } else {
                    int prev = -1;
                    for (;;) {
                        int best = MP_MAXW;
                        float bvv = 0.f;
                        for (unsigned p = (unsigned)n; p != MW_NIL;) {
                            const uint2 x = node[p];
                            const int j = (int)(x.y >> 16);
                            if (j > prev && j < best) {
                                best = j;
                                bvv = __uint_as_float(x.x);
                            }
                            p = x.y & 0xffffu;
                        }
                        if (best == MP_MAXW) break;
                        r = dadd(r, dmul(a.w[best], (double)bvv));
                        prev = best;
                    }
                }
                ab[q] = r;
                mb[q] = 1;
                head[q] = MW_NIL;
            }
            if (hd.w) bar_arrive(BAR_FULL + b, MW_CONS + MW_PROD);  // buffer b holds tile i's values
        }
        return;  // consumers release buffer b after tile i only when tile i + 2 exists
    }

    // ------------------------------- consumers -------------------------------
    const bool first = a.first != 0;
    const int q0 = 4 * tid;  // positions q0 + {0..3} and MW_HALF + q0 + {0..3}
    for (int i = 0; i < nt; ++i) {
        const long long tb = tile_of(i) * AG_TILE;
        const int b = i & 1, s = i % MW_STAGES;
        const bool full = tb + AG_TILE <= a.dim;
        // take the tile's aggregate values and release the hand-off buffer right away, so the
        // producers can build tile i + 2 while this tile's SGD runs
        bar_sync(BAR_FULL + b, MW_CONS + MW_PROD);
        const double* ab = acc + b * AG_TILE;
        uint8_t* mb = mark + b * AG_TILE;
        double g[8];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const int qh = hh * MW_HALF + q0;
            const unsigned mk = *reinterpret_cast<const unsigned*>(mb + qh);
            g[4 * hh] = (mk & 0xffu) ? ab[qh] : 0.0;
            g[4 * hh + 1] = (mk & 0xff00u) ? ab[qh + 1] : 0.0;
            g[4 * hh + 2] = (mk & 0xff0000u) ? ab[qh + 2] : 0.0;
            g[4 * hh + 3] = (mk & 0xff000000u) ? ab[qh + 3] : 0.0;
            if (mk) *reinterpret_cast<unsigned*>(mb + qh) = 0u;
        }
        if (i + 2 < nt) bar_arrive(BAR_EMPTY + b, MW_CONS + MW_PROD);  // the producer may refill buffer b
        if (full) mbar_wait(&fullb[s], (unsigned)(i / MW_STAGES) & 1u);
        const float* rp = ring + (s * 2) * AG_TILE;
        const float* rb = ring + (s * 2 + 1) * AG_TILE;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const int qh = hh * MW_HALF + q0;
            const long long e = tb + qh;
            float pv[4], bv[4];
            if (full) {
                const float4 u = *reinterpret_cast<const float4*>(rp + qh);
                const float4 z = *reinterpret_cast<const float4*>(rb + qh);
                pv[0] = u.x; pv[1] = u.y; pv[2] = u.z; pv[3] = u.w;
                bv[0] = z.x; bv[1] = z.y; bv[2] = z.z; bv[3] = z.w;
            } else {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const bool ok = e + c < a.dim;
                    pv[c] = ok ? a.p[e + c] : 0.f;
                    bv[c] = ok ? a.buf[e + c] : 0.f;
                }
            }
            double pd[4], bd[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                pd[c] = (double)pv[c];
                bd[c] = (double)bv[c];
                sgd_elem(g[4 * hh + c], pd[c], bd[c], a.lr, a.mu, a.wd, first);
            }
            if (full) {
                *reinterpret_cast<float4*>(a.p + e) = make_float4((float)pd[0], (float)pd[1], (float)pd[2], (float)pd[3]);
                *reinterpret_cast<float4*>(a.buf + e) = make_float4((float)bd[0], (float)bd[1], (float)bd[2], (float)bd[3]);
                if (a.out)
                    *reinterpret_cast<float4*>(a.out + e) = make_float4((float)g[4 * hh], (float)g[4 * hh + 1],
                                                                        (float)g[4 * hh + 2], (float)g[4 * hh + 3]);
            } else {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    if (e + c >= a.dim) continue;
                    a.p[e + c] = (float)pd[c];
                    a.buf[e + c] = (float)bd[c];
                    if (a.out) a.out[e + c] = (TO)g[4 * hh + c];
                }
            }
        }
        if (i + MW_STAGES < nt) {
            bar_sync(BAR_CONS, MW_CONS);  // ring stage s fully read
            if (tid == 0) {
                fence_proxy_async();
                issue(i + MW_STAGES);
            }
        }
    }
}


// ---------------------------------------------------------------------------------------
// k_merge_own: the all-sparse merge + fused momentum SGD for dense payloads (on average
// >= MO_DENSITY kept entries per position, e.g. cr 0.1), where k_merge_ws's per-chunk list
// building is latency-bound.  Per tile (4096 positions, 512 threads):
//   (1) every thread starts the p/buf loads of its 8 positions (consumed at the end, so the
//       HBM latency hides behind (2)-(3)); warp 0 loads the next tile's worker runs;
//   (2) the tile's entries (worker runs concatenated) are staged in shared memory, several
//       per thread with their loads in flight together;
//   (3) the float64 sums are folded worker by worker in ascending order -- the reference's
//       fold (comm.py:70-78): +0, then + w_j * v_j.  One worker's positions are distinct, so
//       its entries scatter without conflicts; a CTA barrier orders consecutive workers;
//   (4) momentum SGD (nn.py:167-171 order, binary64), 128-bit streaming stores.
// Tiles are dealt round-robin over a grid of 2 CTAs per SM.  Results are bit-identical to
// k_merge_ws (the same per-position fold order).
// ---------------------------------------------------------------------------------------
constexpr int MO_THREADS = 512;
constexpr int MO_PER = AG_TILE / MO_THREADS;  // 8 positions per thread
constexpr int MO_ECAP = 4096;  // entries staged per chunk (a whole tile's, unless oversized)
constexpr int MO_SMEM = MO_PER * MO_THREADS * (int)sizeof(double) + 2 * MO_ECAP * (int)(sizeof(float) + sizeof(uint32_t));
static_assert(MO_PER == 8, "two float4 per thread");

template <typename TO>
__global__ void __launch_bounds__(MO_THREADS, 2)
k_merge_own(const AggArgs<float, TO> a) {
    pdl_wait();  // no early trigger: the next kernel's CTAs must not take this grid's SM slots
    SG_STAMP(2);
    extern __shared__ __align__(16) unsigned char mo_smem[];
    double (*sacc)[MO_THREADS] = reinterpret_cast<double (*)[MO_THREADS]>(mo_smem);  // [MO_PER][MO_THREADS]
    float* st_v0 = reinterpret_cast<float*>(mo_smem + MO_PER * MO_THREADS * sizeof(double));  // [2][MO_ECAP]
    uint32_t* st_i0 = reinterpret_cast<uint32_t*>(st_v0 + 2 * MO_ECAP);                      // [2][MO_ECAP]
    __shared__ const uint32_t* s_ib[2][MP_MAXW];  // run sets, double-buffered by tile parity
    __shared__ const float* s_vb[2][MP_MAXW];
    __shared__ int s_pre[2][MP_MAXW + 1];
    __shared__ int s_ok;
    const int tid = threadIdx.x, lane = tid & 31;
    const int nw = a.nw;
    if (tid < 32) {
        const int mine = sparse_merge_is_mine(a, true);
        if (tid == 0) s_ok = mine;
    }
#pragma unroll
    for (int c = 0; c < MO_PER; ++c) sacc[c][tid] = 0.0;
    __syncthreads();
    if (!s_ok) return;  // not all-sparse (k_merge), or sparse payloads (k_merge_ws)
    const long long ntl = a.ntiles, G = gridDim.x;
    const bool first = a.first != 0;
    const int q0 = tid * MO_PER;
    // warp 0 lane j < nw: worker j's payload base, read once (not a global load per tile)
    const uint32_t* ib_base = nullptr;
    const float* vb_base = nullptr;
    if (tid < nw) {
        ib_base = a.peer ? a.idxw[lane] : a.idx + a.row_ptr[lane];
        vb_base = a.peer ? a.valw[lane] : a.val + a.row_ptr[lane];
    }
    // warp 0 lane j < nw: worker j's run [lo, lo + cnt) of a tile
    auto load_run = [&](long long t, int& lo, int& cnt) {
        lo = 0;
        cnt = 0;
        if (lane < nw && t < ntl) {
            if (a.peer) {
                lo = a.offw[lane][t];
                cnt = a.offw[lane][t + 1] - lo;
            } else {
                const int* o = a.off + (long long)lane * (ntl + 1);
                lo = o[t];
                cnt = o[t + 1] - lo;
            }
        }
    };
    auto publish_runs = [&](int b, int lo, int cnt) {  // warp 0: run set b <- (lo, cnt) per lane
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane < nw) {
            s_ib[b][lane] = ib_base + lo;
            s_vb[b][lane] = vb_base + lo;
            s_pre[b][lane] = incl - cnt;
        }
        if (lane == 31) s_pre[b][nw] = incl;
    };
    // entries [c0, c1) of run set b into stage b, asynchronously (cp.async, one group)
    auto stage = [&](int b, int c0, int c1) {
        for (int j = 0; j < nw; ++j) {  // run by run: no per-entry search for the worker
            const int pj = s_pre[b][j];
            const int lo = pj > c0 ? pj : c0, hi = s_pre[b][j + 1] < c1 ? s_pre[b][j + 1] : c1;
            const uint32_t* ib = s_ib[b][j] - pj;
            const float* vb = s_vb[b][j] - pj;
            for (int e = lo + tid; e < hi; e += MO_THREADS) {
                cp_async4(st_i0 + b * MO_ECAP + (e - c0), ib + e);
                cp_async4(st_v0 + b * MO_ECAP + (e - c0), vb + e);
            }
        }
        cp_async_commit();
    };
    // prologue: runs and first chunk of this CTA's first tile; runs of the second prefetched
    int nlo = 0, ncnt = 0;
    if (tid < 32) {
        int lo, cnt;
        load_run(blockIdx.x, lo, cnt);
        publish_runs(0, lo, cnt);
        load_run(blockIdx.x + G, nlo, ncnt);
    }
    __syncthreads();
    {
        const int E0 = s_pre[0][nw];
        stage(0, 0, E0 < MO_ECAP ? E0 : MO_ECAP);
    }
    int it = 0;
    for (long long t = blockIdx.x; t < ntl; t += G, ++it) {
        const int b = it & 1;
        const long long tb = t * AG_TILE;
        const bool full = tb + AG_TILE <= a.dim;
        // (1) the next tile's runs into set b ^ 1 and the next tile's chunk into stage b ^ 1
        // (both last read by the previous tile's fold, which every thread has left)
        __syncthreads();
        if (tid < 32) {
            publish_runs(b ^ 1, nlo, ncnt);
            load_run(t + 2 * G, nlo, ncnt);
        } else if (tid < 34 && a.pf && t + G < ntl) {
            // the next tile's p / buf into L2 now, so its loads in (2) are L2 hits while HBM
            // streams during this tile's fold
            const long long tn = (t + G) * AG_TILE;
            const long long n = a.dim - tn < AG_TILE ? a.dim - tn : AG_TILE;
            const unsigned bytes = (unsigned)(n * sizeof(float)) & ~15u;
            if (bytes) bulk_prefetch_l2((tid == 32 ? a.p : a.buf) + tn, bytes);
        }
        // (2) p/buf of this thread's positions (consumed by the SGD at the end)
        float pv[MO_PER], bv[MO_PER];
        if (full) {
            const float4* pp = reinterpret_cast<const float4*>(a.p + tb + q0);
            const float4* bp = reinterpret_cast<const float4*>(a.buf + tb + q0);
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const float4 u = __ldcs(pp + r), z = __ldcs(bp + r);
                pv[4 * r] = u.x; pv[4 * r + 1] = u.y; pv[4 * r + 2] = u.z; pv[4 * r + 3] = u.w;
                bv[4 * r] = z.x; bv[4 * r + 1] = z.y; bv[4 * r + 2] = z.z; bv[4 * r + 3] = z.w;
            }
        } else {
#pragma unroll
            for (int c = 0; c < MO_PER; ++c) {
                const bool ok = tb + q0 + c < a.dim;
                pv[c] = ok ? a.p[tb + q0 + c] : 0.f;
                bv[c] = ok ? a.buf[tb + q0 + c] : 0.f;
            }
        }
        __syncthreads();  // run set b ^ 1 published
        // (3) the next tile's first chunk goes in flight into stage b ^ 1 while this one folds
        if (t + G < ntl) {
            const int En = s_pre[b ^ 1][nw];
            stage(b ^ 1, 0, En < MO_ECAP ? En : MO_ECAP);
        } else {
            cp_async_commit();
        }
        cp_async_wait<1>();  // this thread's copies of this tile's first chunk have landed
        __syncthreads();     // everyone's
        // (4) fold worker by worker in ascending order (comm.py:70-78: +0, then + w_j * v_j);
        // a worker's positions are distinct, so its entries scatter without conflicts
        const int E = s_pre[b][nw];
        for (int c0 = 0; c0 < E; c0 += MO_ECAP) {
            const int c1 = E - c0 < MO_ECAP ? E : c0 + MO_ECAP;
            if (c0 > 0) {  // oversized tile: later chunks are staged synchronously into stage b
                stage(b, c0, c1);
                cp_async_wait<0>();
                __syncthreads();
            }
            const uint32_t* si = st_i0 + b * MO_ECAP;
            const float* sv = st_v0 + b * MO_ECAP;
            for (int j = 0; j < nw; ++j) {
                const int lo = s_pre[b][j] > c0 ? s_pre[b][j] : c0, hi = s_pre[b][j + 1] < c1 ? s_pre[b][j + 1] : c1;
                if (lo >= hi) continue;  // uniform
                const double wj = a.w[j];
                for (int e = lo + tid; e < hi; e += MO_THREADS) {
                    const unsigned q = si[e - c0] - (uint32_t)tb;
                    SG_CHECK(q < (unsigned)AG_TILE && e - c0 < MO_ECAP);
                    double* sa = &sacc[q % MO_PER][q / MO_PER];
                    *sa = dadd(*sa, dmul(wj, (double)sv[e - c0]));
                }
                __syncthreads();
            }
            if (c1 < E) __syncthreads();  // stage b is restaged for the next chunk
        }
        double acc[MO_PER];
#pragma unroll
        for (int c = 0; c < MO_PER; ++c) {
            acc[c] = sacc[c][tid];
            sacc[c][tid] = 0.0;
        }
        // (5) momentum SGD, stores
        double pd[MO_PER], bd[MO_PER];
#pragma unroll
        for (int c = 0; c < MO_PER; ++c) {
            pd[c] = (double)pv[c];
            bd[c] = (double)bv[c];
            sgd_elem(acc[c], pd[c], bd[c], a.lr, a.mu, a.wd, first);
        }
        if (full) {
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const long long e = tb + q0 + 4 * r;
                __stcs(reinterpret_cast<float4*>(a.p + e),
                       make_float4((float)pd[4 * r], (float)pd[4 * r + 1], (float)pd[4 * r + 2], (float)pd[4 * r + 3]));
                __stcs(reinterpret_cast<float4*>(a.buf + e),
                       make_float4((float)bd[4 * r], (float)bd[4 * r + 1], (float)bd[4 * r + 2], (float)bd[4 * r + 3]));
                if (a.out)
                    *reinterpret_cast<float4*>(a.out + e) = make_float4((float)acc[4 * r], (float)acc[4 * r + 1],
                                                                        (float)acc[4 * r + 2], (float)acc[4 * r + 3]);
            }
        } else {
#pragma unroll
            for (int c = 0; c < MO_PER; ++c) {
                const long long e = tb + q0 + c;
                if (e >= a.dim) continue;
                a.p[e] = (float)pd[c];
                a.buf[e] = (float)bd[c];
                if (a.out) a.out[e] = (TO)acc[c];
            }
        }
    }
    cp_async_wait<0>();
}


// The all-sparse merge pair: k_merge_ws then k_merge_own; each exits unless the device-side
// density test picks it (a.own forces one, and the other is not launched).
template <typename TO>
void launch_sparse_merge(const AggArgs<float, TO>& a, int grid, size_t sm, int sms, cudaStream_t stream) {
    if (a.own != 1) {
        AggArgs<float, TO> aw = a;
        aw.direct = mw_direct();
        smem_attr((const void*)k_merge_ws<TO>, (int)sm);
        launch_pdl(k_merge_ws<TO>, dim3((unsigned)grid), dim3(MW_THREADS), sm, stream, aw);
        debug_sync("k_merge_ws", stream);
    }
    if (a.own != 0) {
        AggArgs<float, TO> ao = a;
        ao.pf = 1;
        long long g2 = 2LL * sms;
        if (g2 > a.ntiles) g2 = a.ntiles;
        const int dsm = MO_SMEM;
        smem_attr((const void*)k_merge_own<TO>, dsm);
        launch_pdl(k_merge_own<TO>, dim3((unsigned)g2), dim3(MO_THREADS), (size_t)dsm, stream, ao);
        debug_sync("k_merge_own", stream);
    }
}

template <typename T>
__global__ void __launch_bounds__(256)
k_sgd(T* __restrict__ p, T* __restrict__ buf, const T* __restrict__ g, long long dim, double lr,
      double mu, double wd, int first, int vec_ok) {
    pdl_enter();
    const long long nvec = vec_ok ? dim / 4 : 0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += stride) {
        double gv[4], pv[4], bv[4] = {0.0, 0.0, 0.0, 0.0};
        load4<T>(g + 4 * i, gv);
        load4_rw<T>(p + 4 * i, pv);
        if (!first) load4_rw<T>(buf + 4 * i, bv);
#pragma unroll
        for (int c = 0; c < 4; ++c) sgd_elem(gv[c], pv[c], bv[c], lr, mu, wd, first != 0);
        store4<T>(p + 4 * i, pv);
        store4<T>(buf + 4 * i, bv);
    }
    for (long long q = nvec * 4 + (long long)blockIdx.x * blockDim.x + threadIdx.x; q < dim; q += stride) {
        double pv = p[q], bv = first ? 0.0 : (double)buf[q];
        sgd_elem((double)g[q], pv, bv, lr, mu, wd, first != 0);
        p[q] = (T)pv;
        buf[q] = (T)bv;
    }
}

struct WArr {
    double v[8];
};

inline long long ag_tiles(long long dim) { return (dim + AG_TILE - 1) / AG_TILE; }

// Dense rows only, no update (the dense workload's per-rank partial at P > 1):
// out = sum_j w_j * row_j in ascending j (float64, round-to-nearest), rounded once; float4
// loads of every row in flight per thread, grid-stride over the row.
template <int NWMAX>
__global__ void __launch_bounds__(256)
k_weighted_rows(const float* __restrict__ dense, long long ld, int nw, WArr w, long long dim, float* __restrict__ out,
                const uint8_t* __restrict__ guard, int gn) {
    pdl_enter();
    if (guard) {
        __shared__ int s_run;
        if (threadIdx.x == 0) {
            int any0 = 0;
            for (int j = 0; j < gn; ++j) any0 |= guard[j] == 0;
            s_run = any0;
        }
        __syncthreads();
        if (!s_run) return;
    }
    const long long n4 = dim / 4, stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        float4 x[NWMAX];
#pragma unroll
        for (int j = 0; j < NWMAX; ++j)
            if (j < nw) x[j] = ld_stream(reinterpret_cast<const float4*>(dense + j * ld) + i);
        double g[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int j = 0; j < NWMAX; ++j) {
            if (j >= nw) break;
            g[0] = dadd(g[0], dmul(w.v[j], (double)x[j].x));
            g[1] = dadd(g[1], dmul(w.v[j], (double)x[j].y));
            g[2] = dadd(g[2], dmul(w.v[j], (double)x[j].z));
            g[3] = dadd(g[3], dmul(w.v[j], (double)x[j].w));
        }
        reinterpret_cast<float4*>(out)[i] = make_float4((float)g[0], (float)g[1], (float)g[2], (float)g[3]);
    }
    for (long long q = n4 * 4 + (long long)blockIdx.x * blockDim.x + threadIdx.x; q < dim; q += stride) {
        double g = 0.0;
        for (int j = 0; j < nw; ++j) g = dadd(g, dmul(w.v[j], (double)dense[j * ld + q]));
        out[q] = (float)g;
    }
}

template <typename TI, typename TO>
int aggregate(int nw, const double* weights, const uint8_t* comp, const TI* dense, long long ld,
              const uint32_t* idx, const TI* val, const long long* row_ptr, const int* tile_off,
              long long dim, TO* out, TO* p, TO* buf, double lr, double mu, double wd, int first,
              void* ws, size_t ws_bytes, cudaStream_t stream, int sparse_merge = -1,
              const uint8_t* guard = nullptr, int guard_n = 0, int guard_mode = 0) {
    if (nw < 1 || dim < 1 || !weights || (!out && !p)) return SG_ERR_INVALID;
    if (nw > MAX_WORKERS || dim >= (1ll << 31)) return SG_ERR_UNSUPPORTED;
    if (p && !buf) return SG_ERR_INVALID;
    // Sparse workers need idx/val/row_ptr; dense workers need the dense rows.
    if (comp && (!idx || !val || !row_ptr)) return SG_ERR_INVALID;
    if (!dense && !comp) return SG_ERR_INVALID;
    if (dense && ld < dim) return SG_ERR_INVALID;
    const long long ntiles = ag_tiles(dim);
    const int* off = tile_off;
    if (comp && !off) {
        const size_t need = sizeof(int) * (size_t)nw * (size_t)(ntiles + 1);
        if (!ws || ws_bytes < need) return SG_ERR_WORKSPACE;
        int* o = reinterpret_cast<int*>(ws);
        // rows are sized on the device; a fixed grid strides over each row
        long long blocks = ((long long)num_sms() * 8 + nw - 1) / nw;
        launch_pdl(k_tile_offsets, dim3(dim3((unsigned)blocks, nw)), dim3(256), 0, stream, idx, row_ptr, comp, ntiles, o);
        off = o;
    }
    AggArgs<TI, TO> a;
    for (int j = 0; j < nw; ++j) a.w[j] = weights[j];
    a.comp = comp;
    a.dense = dense;
    a.idx = idx;
    a.val = val;
    a.row_ptr = row_ptr;
    a.off = off;
    a.out = out;
    a.p = p;
    a.buf = buf;
    a.ld = ld;
    a.dim = dim;
    a.ntiles = ntiles;
    a.lr = lr;
    a.mu = mu;
    a.wd = wd;
    a.nw = nw;
    a.first = first;
    a.pipe = 0;
    a.peer = 0;
    a.guard = guard;
    a.guard_n = guard_n;
    a.guard_mode = guard_mode;
    bool vec = true;
    if (dense) vec = vec && reinterpret_cast<size_t>(dense) % 16 == 0 && (ld * (long long)sizeof(TI)) % 16 == 0;
    if (out) vec = vec && reinterpret_cast<size_t>(out) % 16 == 0;
    if (p) vec = vec && reinterpret_cast<size_t>(p) % 16 == 0 && reinterpret_cast<size_t>(buf) % 16 == 0;
    a.vec_ok = vec;
    if constexpr (sizeof(TI) == 4 && sizeof(TO) == 4)
    {
        const int sms = num_sms();
        if (!comp && !p && vec && nw <= 8) {  // dense rows, no update: the streaming fold
            WArr wa;
            for (int j = 0; j < nw; ++j) wa.v[j] = weights[j];
            long long blocks = (dim / 4 + 255) / 256;
            if (blocks > (long long)sms * 8) blocks = (long long)sms * 8;
            if (blocks < 1) blocks = 1;
            launch_pdl(k_weighted_rows<8>, dim3((unsigned)blocks), dim3(256), 0, stream, reinterpret_cast<const float*>(dense),
                       ld, nw, wa, dim, reinterpret_cast<float*>(out), guard, guard_n);
            return cudaGetLastError() == cudaSuccess ? SG_OK : SG_ERR_CUDA;
        }
        a.pipe = comp && vec && p && nw <= MP_MAXW;
        if (a.pipe) {
            const int grid = mw_grid(ntiles, sms);
            const size_t sm = mw_smem_bytes();
            a.balance = mw_balance();
            a.cost_j0 = 0;
            a.cost_j1 = nw;
            a.own = merge_mode(sparse_merge);
            launch_sparse_merge(a, grid, sm, sms, stream);
        }
        smem_attr((const void*)k_merge<TO>, (int)MG_SMEM);
        long long grid = (long long)sms * 2;
        if (grid > ntiles) grid = ntiles;
        launch_pdl(k_merge<TO>, dim3((unsigned)grid), dim3(MG_THREADS), MG_SMEM, stream, a);
        debug_sync("k_merge", stream);
    }
    else
        launch_pdl(k_aggregate<TI, TO>, dim3((unsigned)ntiles), dim3(AG_THREADS), 0, stream, a);
    return cudaGetLastError() == cudaSuccess ? SG_OK : SG_ERR_CUDA;
}

template <typename T>
int sgd(T* p, T* buf, const T* g, long long dim, double lr, double mu, double wd, int first,
        cudaStream_t stream) {
    if (!p || !buf || !g || dim < 1) return SG_ERR_INVALID;
    const int vec_ok = reinterpret_cast<size_t>(p) % 16 == 0 && reinterpret_cast<size_t>(buf) % 16 == 0 &&
                       reinterpret_cast<size_t>(g) % 16 == 0;
    long long blocks = (dim / 4 + 255) / 256;
    const long long cap = (long long)num_sms() * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    launch_pdl(k_sgd<T>, dim3((unsigned)blocks), dim3(256), 0, stream, p, buf, g, dim, lr, mu, wd, first, vec_ok);
    return cudaGetLastError() == cudaSuccess ? SG_OK : SG_ERR_CUDA;
}

// Merge + fused SGD over workers whose payloads are addressed per worker (peer GPUs).
int aggregate_peers(int nw, const double* weights, const uint8_t* comp, const uint32_t* const* idx_ptrs,
                    const float* const* val_ptrs, const int32_t* const* off_ptrs, long long dim, float* out,
                    float* p, float* buf, double lr, double mu, double wd, int first, int local_lo, int local_n,
                    int sparse_merge, cudaStream_t stream) {
    if (nw < 1 || dim < 1 || !weights || !comp || !idx_ptrs || !val_ptrs || !off_ptrs || !p || !buf)
        return SG_ERR_INVALID;
    if (nw > PEER_MAXW || dim >= (1ll << 31)) return SG_ERR_UNSUPPORTED;
    if (reinterpret_cast<size_t>(p) % 16 || reinterpret_cast<size_t>(buf) % 16 ||
        (out && reinterpret_cast<size_t>(out) % 16))
        return SG_ERR_UNSUPPORTED;
    const long long ntiles = ag_tiles(dim);
    AggArgs<float, float> a = {};
    for (int j = 0; j < nw; ++j) {
        if (!idx_ptrs[j] || !val_ptrs[j] || !off_ptrs[j]) return SG_ERR_INVALID;
        a.w[j] = weights[j];
        a.idxw[j] = idx_ptrs[j];
        a.valw[j] = val_ptrs[j];
        a.offw[j] = off_ptrs[j];
    }
    a.peer = 1;
    a.comp = comp;
    a.out = out;
    a.p = p;
    a.buf = buf;
    a.dim = dim;
    a.ntiles = ntiles;
    a.lr = lr;
    a.mu = mu;
    a.wd = wd;
    a.nw = nw;
    a.first = first;
    a.vec_ok = 1;
    a.pipe = 1;
    const int sms = num_sms();
    const int grid = mw_grid(ntiles, sms);
    const size_t sm = mw_smem_bytes();
    a.balance = mw_balance();
    // the balanced ranges are costed from the workers whose payloads live on this device
    // (the caller names them: local reads are cheap to scan, remote ones are not)
    if (local_lo < 0 || local_n < 0 || local_lo + local_n > nw) return SG_ERR_INVALID;
    a.cost_j0 = local_n > 0 ? local_lo : 0;
    a.cost_j1 = local_n > 0 ? local_lo + local_n : nw;
    a.own = merge_mode(sparse_merge);
    launch_sparse_merge(a, grid, sm, sms, stream);
    return cudaGetLastError() == cudaSuccess ? SG_OK : SG_ERR_CUDA;
}

// The dense exchange of a mixed (or dense-workload) multi-GPU step without a collective
// library, O(D) NVLink bytes per rank: position-sharded reduce, then an all-gather fused with
// momentum SGD.  Rank r owns slice r = [r*L, min((r+1)*L, dim)) with L = peer_slice_len(dim, P)
// (a multiple of 4 elements, so slices stay 16-byte aligned).
//   k_peer_reduce_slice   g[slice r] = sum_q w_q * src_q[slice r] in ascending q (float64,
//                         IEEE round-to-nearest), rounded once to float32 and written to
//                         dst[slice r] (dst may be this rank's own source: slice r of a rank's
//                         partial is read by that rank only).  Reads (P-1)/P * 4D over NVLink.
//   k_peer_allgather_sgd  every rank reads element i's aggregate from its owner's buffer
//                         (P-1)/P * 4D over NVLink) and applies momentum SGD (nn.py:167-171
//                         order, binary64) to its full replica, so replicas stay bit-identical.
// Both are guarded: a no-op unless some worker in `guard` did not compress (guard NULL: always).
inline long long peer_slice_len(long long dim, int P) {
    const long long per = (dim + P - 1) / P;
    return (per + 3) / 4 * 4;
}

struct PeerRows {
    const float* p[MAX_WORKERS];
    double w[MAX_WORKERS];
};

SG_DEV bool peer_guard_run(const uint8_t* guard, int gn) {
    __shared__ int s_run;
    if (threadIdx.x == 0) {
        int any0 = guard == nullptr ? 1 : 0;
        for (int j = 0; j < gn; ++j) any0 |= guard[j] == 0;
        s_run = any0;
    }
    __syncthreads();
    return s_run != 0;
}

struct PeerDst {
    float* p[MAX_PEERS];
};

__global__ void __launch_bounds__(256)
k_peer_reduce_slice(PeerRows src, int P, int unit_w, long long lo, long long hi, const uint8_t* __restrict__ guard,
                    int gn, PeerDst dsts, int nd) {
    pdl_enter();
    if (!peer_guard_run(guard, gn)) return;
    const long long n4 = (hi - lo) / 4, stride = (long long)gridDim.x * blockDim.x;
    constexpr int U = 2;  // float4 groups per thread per iteration: P*U independent loads in flight
    for (long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; i0 < n4; i0 += stride * U) {
        float4 x[U][MAX_PEERS];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long i = i0 + u * stride;
            if (i < n4) {
#pragma unroll
                for (int r = 0; r < MAX_PEERS; ++r)
                    if (r < P) x[u][r] = __ldcv(reinterpret_cast<const float4*>(src.p[r] + lo) + i);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long i = i0 + u * stride;
            if (i >= n4) continue;
            double g[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int r = 0; r < MAX_PEERS; ++r) {
                if (r >= P) break;
                const double wr = src.w[r];
                const float4 v = x[u][r];
                if (unit_w) {
                    g[0] = dadd(g[0], (double)v.x);
                    g[1] = dadd(g[1], (double)v.y);
                    g[2] = dadd(g[2], (double)v.z);
                    g[3] = dadd(g[3], (double)v.w);
                } else {
                    g[0] = dadd(g[0], dmul(wr, (double)v.x));
                    g[1] = dadd(g[1], dmul(wr, (double)v.y));
                    g[2] = dadd(g[2], dmul(wr, (double)v.z));
                    g[3] = dadd(g[3], dmul(wr, (double)v.w));
                }
            }
            const float4 o = make_float4((float)g[0], (float)g[1], (float)g[2], (float)g[3]);
            // the reduced slice goes to every destination (this rank's buffer, or pushed into
            // every rank's aggregate buffer: posted NVLink writes instead of later pulls)
            for (int d = 0; d < nd; ++d) reinterpret_cast<float4*>(dsts.p[d] + lo)[i] = o;
        }
    }
    // ragged tail of the last slice (dim not a multiple of 4)
    for (long long q = lo + n4 * 4 + (long long)blockIdx.x * blockDim.x + threadIdx.x; q < hi; q += stride) {
        double g = 0.0;
        for (int r = 0; r < P; ++r) g = unit_w ? dadd(g, (double)src.p[r][q]) : dadd(g, dmul(src.w[r], (double)src.p[r][q]));
        for (int d = 0; d < nd; ++d) dsts.p[d][q] = (float)g;
    }
}

__global__ void __launch_bounds__(256)
k_peer_allgather_sgd(PeerRows src, int P, int rank, long long L, const uint8_t* __restrict__ guard, int gn,
                     long long dim, float* __restrict__ out, float* __restrict__ p, float* __restrict__ b, double lr,
                     double mu, double wd, int first) {
    pdl_enter();
    if (!peer_guard_run(guard, gn)) return;
    const long long n4 = dim / 4, stride = (long long)gridDim.x * blockDim.x;
    const long long L4 = L / 4;
    // rank r walks the slices starting at slice r + 1: at any moment the P ranks pull from P
    // different owners, so every GPU's NVLink egress serves one reader instead of all of them
    long long start = ((long long)(rank + 1) % P) * L4;
    if (start >= n4) start = 0;
    constexpr int U = 2;  // independent float4 groups per thread in flight
    for (long long j0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; j0 < n4; j0 += stride * U) {
        float4 gv[U], pv[U], bv[U];
        long long ii[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long j = j0 + u * stride;
            long long i = j + start;
            if (i >= n4) i -= n4;
            ii[u] = j < n4 ? i : -1;
            if (j < n4) {
                gv[u] = __ldcv(reinterpret_cast<const float4*>(src.p[(int)(i / L4)]) + i);
                pv[u] = reinterpret_cast<const float4*>(p)[i];
                bv[u] = first ? make_float4(0.f, 0.f, 0.f, 0.f) : reinterpret_cast<const float4*>(b)[i];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long i = ii[u];
            if (i < 0) continue;
            double g[4] = {gv[u].x, gv[u].y, gv[u].z, gv[u].w};
            double pd[4] = {pv[u].x, pv[u].y, pv[u].z, pv[u].w}, bd[4] = {bv[u].x, bv[u].y, bv[u].z, bv[u].w};
#pragma unroll
            for (int c = 0; c < 4; ++c) sgd_elem(g[c], pd[c], bd[c], lr, mu, wd, first != 0);
            reinterpret_cast<float4*>(p)[i] = make_float4((float)pd[0], (float)pd[1], (float)pd[2], (float)pd[3]);
            reinterpret_cast<float4*>(b)[i] = make_float4((float)bd[0], (float)bd[1], (float)bd[2], (float)bd[3]);
            if (out) reinterpret_cast<float4*>(out)[i] = gv[u];
        }
    }
    for (long long qd = n4 * 4 + (long long)blockIdx.x * blockDim.x + threadIdx.x; qd < dim; qd += stride) {
        const int q = (int)(qd / L);
        const double g = (double)__ldcv(src.p[q] + qd);
        double pq = p[qd], bq = first ? 0.0 : (double)b[qd];
        sgd_elem(g, pq, bq, lr, mu, wd, first != 0);
        p[qd] = (float)pq;
        b[qd] = (float)bq;
        if (out) out[qd] = (float)g;
    }
}

// ---- The pipelined dense exchange: partial -> reduce -> push -> update in ONE launch ---------
// The dense side of a multi-GPU step as a single cooperative kernel per rank whose three CTA
// roles overlap over chunks of XC elements, synchronised across GPUs by per-chunk epoch flags
// in peer-mapped memory instead of barriers between phases:
//   partial  (role 0)  this rank's weighted fold of its dense rows for chunk c (or, with the
//                      partial precomputed, nothing) -> raise pflag[owner(c)][c][rank]
//   reduce   (role 1)  for the chunks this rank owns (c % P == rank): wait until every rank's
//                      partial of c is up, sum them in ascending rank order (float64, pulled
//                      over NVLink), push the float32 result into every rank's aggregate
//                      buffer, raise aflag[q][c] on every rank q
//   update   (role 2)  for every chunk: wait for aflag[c] (local), momentum SGD (nn.py:167-171
//                      order, binary64) from the local copy of the aggregate
// HBM work (the fold, the update) overlaps the NVLink pulls and pushes of other chunks.  Flags
// carry the step's epoch (monotone), so no reset; a rank's buffers are reused only after the
// previous launch completed, which already implies every owner consumed them (the update role
// waits for every chunk's aggregate).  Guarded like the rest of the dense side.
constexpr int XC = 16384;  // chunk elements (64 KB of float32)

struct DxArgs {
    const float* dense;    // this rank's [k][ld] rows (role 0 folds them) or nullptr
    long long ld, dim;
    int k, P, rank, nchunk, roles_per;  // roles_per: CTAs per role
    WArr w;                // this rank's worker weights
    const float* partial_src[MAX_PEERS];  // every rank's partial buffer (peers' memory)
    float* partial_own;    // this rank's partial buffer (role 0 writes it)
    float* agg[MAX_PEERS];  // every rank's aggregate buffer (role 1 pushes into them)
    const float* agg_own;
    unsigned* pflag[MAX_PEERS];  // rank q's pflag array [nchunk][P]
    unsigned* aflag[MAX_PEERS];  // rank q's aflag array [nchunk]
    unsigned* pflag_own;
    unsigned* aflag_own;
    unsigned epoch;
    const uint8_t* guard;
    int gn;
    float* out;
    float* p;
    float* b;
    double lr, mu, wd;
    int first;
};

SG_DEV void st_release_sys(unsigned* p, unsigned v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
SG_DEV unsigned ld_acquire_sys(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
SG_DEV void wait_epoch(const unsigned* f, unsigned epoch) {
    while ((int)(ld_acquire_sys(f) - epoch) < 0) __nanosleep(100);
}

__global__ void __launch_bounds__(256)
k_dense_exchange(DxArgs a) {
    pdl_enter();
    {
        __shared__ int s_run;
        if (threadIdx.x == 0) {
            int any0 = a.guard == nullptr ? 1 : 0;
            for (int j = 0; j < a.gn; ++j) any0 |= a.guard[j] == 0;
            s_run = any0;
        }
        __syncthreads();
        if (!s_run) return;
    }
    const int role = blockIdx.x / a.roles_per, rb = blockIdx.x % a.roles_per, R = a.roles_per;
    const int tid = threadIdx.x;
    const int P = a.P;
    if (role == 0) {
        for (int c = rb; c < a.nchunk; c += R) {
            const long long lo = (long long)c * XC, hi = lo + XC < a.dim ? lo + XC : a.dim;
            if (a.dense) {
                const long long n4 = (hi - lo) / 4;
                for (long long i = tid; i < n4; i += 256) {
                    double g[4] = {0.0, 0.0, 0.0, 0.0};
                    for (int j = 0; j < a.k; ++j) {
                        const float4 x = ld_stream(reinterpret_cast<const float4*>(a.dense + j * a.ld + lo) + i);
                        g[0] = dadd(g[0], dmul(a.w.v[j], (double)x.x));
                        g[1] = dadd(g[1], dmul(a.w.v[j], (double)x.y));
                        g[2] = dadd(g[2], dmul(a.w.v[j], (double)x.z));
                        g[3] = dadd(g[3], dmul(a.w.v[j], (double)x.w));
                    }
                    reinterpret_cast<float4*>(a.partial_own + lo)[i] =
                        make_float4((float)g[0], (float)g[1], (float)g[2], (float)g[3]);
                }
                for (long long q = lo + n4 * 4 + tid; q < hi; q += 256) {
                    double g = 0.0;
                    for (int j = 0; j < a.k; ++j) g = dadd(g, dmul(a.w.v[j], (double)a.dense[j * a.ld + q]));
                    a.partial_own[q] = (float)g;
                }
            }
            __threadfence_system();
            __syncthreads();
            if (tid == 0) st_release_sys(a.pflag[c % P] + (long long)c * P + a.rank, a.epoch);
        }
    } else if (role == 1) {
        __shared__ int s_dummy;
        (void)s_dummy;
        for (int i0 = rb;; i0 += R) {
            const int c = a.rank + i0 * P;
            if (c >= a.nchunk) break;
            if (tid < P) wait_epoch(a.pflag_own + (long long)c * P + tid, a.epoch);
            __syncthreads();
            const long long lo = (long long)c * XC, hi = lo + XC < a.dim ? lo + XC : a.dim;
            const long long n4 = (hi - lo) / 4;
            for (long long i = tid; i < n4; i += 256) {
                float4 x[MAX_PEERS];
#pragma unroll
                for (int r = 0; r < MAX_PEERS; ++r)
                    if (r < P) x[r] = __ldcg(reinterpret_cast<const float4*>(a.partial_src[r] + lo) + i);
                double g[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                for (int r = 0; r < MAX_PEERS; ++r) {
                    if (r >= P) break;
                    g[0] = dadd(g[0], (double)x[r].x);
                    g[1] = dadd(g[1], (double)x[r].y);
                    g[2] = dadd(g[2], (double)x[r].z);
                    g[3] = dadd(g[3], (double)x[r].w);
                }
                const float4 o = make_float4((float)g[0], (float)g[1], (float)g[2], (float)g[3]);
                for (int d = 0; d < P; ++d) {
                    const int q = (a.rank + 1 + d) % P;  // stagger the push targets
                    reinterpret_cast<float4*>(a.agg[q] + lo)[i] = o;
                }
            }
            for (long long qd = lo + n4 * 4 + tid; qd < hi; qd += 256) {
                double g = 0.0;
                for (int r = 0; r < P; ++r) g = dadd(g, (double)__ldcg(a.partial_src[r] + qd));
                for (int q = 0; q < P; ++q) a.agg[q][qd] = (float)g;
            }
            __threadfence_system();
            __syncthreads();
            if (tid < P) st_release_sys(a.aflag[tid] + c, a.epoch);
        }
    } else {
        for (int c = rb; c < a.nchunk; c += R) {
            if (tid == 0) wait_epoch(a.aflag_own + c, a.epoch);
            __syncthreads();
            const long long lo = (long long)c * XC, hi = lo + XC < a.dim ? lo + XC : a.dim;
            const long long n4 = (hi - lo) / 4;
            for (long long i = tid; i < n4; i += 256) {
                const float4 gv = __ldcg(reinterpret_cast<const float4*>(a.agg_own + lo) + i);
                const float4 pv = reinterpret_cast<const float4*>(a.p + lo)[i];
                const float4 bv = a.first ? make_float4(0.f, 0.f, 0.f, 0.f) : reinterpret_cast<const float4*>(a.b + lo)[i];
                double g[4] = {gv.x, gv.y, gv.z, gv.w};
                double pd[4] = {pv.x, pv.y, pv.z, pv.w}, bd[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) sgd_elem(g[e], pd[e], bd[e], a.lr, a.mu, a.wd, a.first != 0);
                reinterpret_cast<float4*>(a.p + lo)[i] = make_float4((float)pd[0], (float)pd[1], (float)pd[2], (float)pd[3]);
                reinterpret_cast<float4*>(a.b + lo)[i] = make_float4((float)bd[0], (float)bd[1], (float)bd[2], (float)bd[3]);
                if (a.out) reinterpret_cast<float4*>(a.out + lo)[i] = gv;
            }
            for (long long qd = lo + n4 * 4 + tid; qd < hi; qd += 256) {
                const double g = (double)__ldcg(a.agg_own + qd);
                double pq = a.p[qd], bq = a.first ? 0.0 : (double)a.b[qd];
                sgd_elem(g, pq, bq, a.lr, a.mu, a.wd, a.first != 0);
                a.p[qd] = (float)pq;
                a.b[qd] = (float)bq;
                if (a.out) a.out[qd] = (float)g;
            }
            __syncthreads();
        }
    }
}

// ---- NVLink SHARP (NVLS) reduce + broadcast through the switch ---------------------------------
// Rank r's slice of the dense side in one pass over multicast addresses: each 16-byte group is
// summed IN THE SWITCH over every rank's partial (multimem.ld_reduce, float32 adds) and the sum
// is written back to every rank's aggregate buffer with one multicast store (multimem.st).
// Per rank and direction that moves 4D bytes over NVLink instead of the 2(P-1)/P * 4D of a
// ring or of the pull/push exchanges; the result is identical on every rank (each element is
// reduced once, by its owner).  Guarded like the rest of the dense side.
SG_DEV float4 mm_ld_reduce_add_v4(const float* mc) {
    float4 v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(mc) : "memory");
    return v;
}
SG_DEV void mm_st_v4(float* mc, float4 v) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};"
                 ::"l"(mc), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
SG_DEV float mm_ld_reduce_add(const float* mc) {
    float v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(v) : "l"(mc) : "memory");
    return v;
}
SG_DEV void mm_st(float* mc, float v) {
    asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(mc), "f"(v) : "memory");
}

__global__ void __launch_bounds__(256)
k_nvls_reduce_bcast(const float* mc_src, float* mc_dst, long long lo, long long hi, const uint8_t* __restrict__ guard,
                    int gn) {
    pdl_enter();
    if (!peer_guard_run(guard, gn)) return;
    const long long n4 = (hi - lo) / 4, stride = (long long)gridDim.x * blockDim.x;
    constexpr int U = 4;  // independent multicast reductions in flight per thread
    for (long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; i0 < n4; i0 += stride * U) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long i = i0 + u * stride;
            if (i < n4) v[u] = mm_ld_reduce_add_v4(mc_src + lo + 4 * i);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long i = i0 + u * stride;
            if (i < n4) mm_st_v4(mc_dst + lo + 4 * i, v[u]);
        }
    }
    for (long long q = lo + n4 * 4 + (long long)blockIdx.x * blockDim.x + threadIdx.x; q < hi; q += stride)
        mm_st(mc_dst + q, mm_ld_reduce_add(mc_src + q));
    __threadfence_system();  // the multicast stores are visible system-wide before the barrier
}

// Multicast copy of n4 16-byte vectors (the payload broadcast, sg_multicast_copy_u32): local
// HBM reads, multimem.st to every rank's copy through the switch, U vectors in flight per thread.
__global__ void __launch_bounds__(256)
k_mc_copy(const uint4* __restrict__ src, float* mc_dst, long long n4) {
    pdl_enter();
    const long long stride = (long long)gridDim.x * blockDim.x;
    constexpr int U = 4;
    for (long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; i0 < n4; i0 += stride * U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long i = i0 + u * stride;
            if (i < n4) v[u] = ld_stream(src + i);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long i = i0 + u * stride;
            if (i < n4)  // a plain store: the words' bits (NaN payloads, indices) pass unchanged (tested)
                mm_st_v4(mc_dst + 4 * i, make_float4(__uint_as_float(v[u].x), __uint_as_float(v[u].y),
                                                     __uint_as_float(v[u].z), __uint_as_float(v[u].w)));
        }
    }
    __threadfence_system();  // the multicast stores are visible system-wide before the barrier
}

inline long long peer_blocks(long long n4) {
    long long blocks = (n4 + 255) / 256;
    const long long cap = (long long)num_sms() * 8;
    if (blocks > cap) blocks = cap;
    return blocks < 1 ? 1 : blocks;
}

struct GatherSrc {
    const uint8_t* p[MAX_WORKERS];
};

struct FlagPtrs {
    unsigned* p[MAX_PEERS];
};

// Peer barrier over symmetric flag words (sg_peer_signal_wait): lane q < P writes this rank's
// epoch into rank q's flag word [slot * P + rank] (st.release.sys over NVLink) and waits until
// rank q's epoch in this rank's own words reaches it (ld.acquire.sys).  epoch == 0: the epoch is
// a device-side counter incremented per executed call (identical on every rank, since every rank
// skips or runs a guarded call alike: the guard is the gathered decisions).  Guarded calls return
// at once when every worker compressed (the dense side has nothing to exchange).  Optionally
// gathers the ranks' decision bytes afterwards (the opening barrier of a peer step).
__global__ void __launch_bounds__(32)
k_peer_signal_wait(FlagPtrs flags, int P, int rank, int slot, unsigned epoch, unsigned* counter,
                   const uint8_t* __restrict__ guard, int gn, GatherSrc src, long long each, uint8_t* __restrict__ dst) {
    pdl_enter();
    const int lane = threadIdx.x;
    if (guard && !peer_guard_run(guard, gn)) return;
    unsigned e = epoch;
    if (e == 0) {
        if (lane == 0) e = *counter + 1u, *counter = e;
        e = __shfl_sync(FULL, e, 0);
    }
    __threadfence_system();
    if (lane < P) st_release_sys(flags.p[lane] + slot * P + rank, e);
    if (lane < P) {
        const unsigned* mine = flags.p[rank] + slot * P + lane;
        while ((int)(ld_acquire_sys(mine) - e) < 0) __nanosleep(32);
    }
    __syncwarp();
    if (dst) {
        const long long n = (long long)P * each;
        for (long long i = lane; i < n; i += 32) dst[i] = src.p[i / each][i % each];
    }
}

__global__ void k_gather_bytes(GatherSrc src, int nsrc, long long each, uint8_t* __restrict__ dst) {
    pdl_enter();
    const long long n = (long long)nsrc * each;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        dst[i] = src.p[i / each][i % each];
}

}  // namespace sg

using namespace sg;

SG_STAMPS_EXPORT(sg_diag_stamps_agg)

extern "C" {

size_t sg_aggregate_workspace_bytes(int nw, int64_t dim) {
    if (nw < 1 || dim < 1) return 0;
    return sizeof(int) * (size_t)nw * (size_t)(ag_tiles(dim) + 1);
}

int sg_weighted_aggregate_f32(int nw, const double* weights, const uint8_t* compressed,
                              const float* dense, int64_t ld_dense, const uint32_t* idx,
                              const float* val, const int64_t* row_ptr, const int32_t* tile_off,
                              int64_t dim, float* out, float* params, float* momentum_buf,
                              double lr, double momentum, double weight_decay, int first_step,
                              int sparse_merge, void* workspace, size_t workspace_bytes, void* stream) {
    return aggregate<float, float>(nw, weights, compressed, dense, ld_dense, idx, val,
                                   reinterpret_cast<const long long*>(row_ptr), tile_off, dim, out,
                                   params, momentum_buf, lr, momentum, weight_decay, first_step,
                                   workspace, workspace_bytes, (cudaStream_t)stream, sparse_merge);
}

int sg_weighted_aggregate_f64(int nw, const double* weights, const uint8_t* compressed,
                              const double* dense, int64_t ld_dense, const uint32_t* idx,
                              const double* val, const int64_t* row_ptr, const int32_t* tile_off,
                              int64_t dim, double* out, double* params, double* momentum_buf,
                              double lr, double momentum, double weight_decay, int first_step,
                              void* workspace, size_t workspace_bytes, void* stream) {
    return aggregate<double, double>(nw, weights, compressed, dense, ld_dense, idx, val,
                                     reinterpret_cast<const long long*>(row_ptr), tile_off, dim, out,
                                     params, momentum_buf, lr, momentum, weight_decay, first_step,
                                     workspace, workspace_bytes, (cudaStream_t)stream);
}

int sg_sgd_momentum_f32(float* params, float* momentum_buf, const float* grad, int64_t dim,
                        double lr, double momentum, double weight_decay, int first_step,
                        void* stream) {
    return sgd<float>(params, momentum_buf, grad, dim, lr, momentum, weight_decay, first_step,
                      (cudaStream_t)stream);
}

int sg_sgd_momentum_f64(double* params, double* momentum_buf, const double* grad, int64_t dim,
                        double lr, double momentum, double weight_decay, int first_step,
                        void* stream) {
    return sgd<double>(params, momentum_buf, grad, dim, lr, momentum, weight_decay, first_step,
                       (cudaStream_t)stream);
}

int sg_weighted_aggregate_peers_f32(int nw, const double* weights, const uint8_t* compressed,
                                    const uint32_t* const* idx_ptrs, const float* const* val_ptrs,
                                    const int32_t* const* tile_off_ptrs, int64_t dim, float* out,
                                    float* params, float* momentum_buf, double lr, double momentum,
                                    double weight_decay, int first_step, int local_lo, int local_n,
                                    int sparse_merge, void* stream) {
    return aggregate_peers(nw, weights, compressed, idx_ptrs, val_ptrs, tile_off_ptrs, dim, out, params,
                           momentum_buf, lr, momentum, weight_decay, first_step, local_lo, local_n,
                           sparse_merge, (cudaStream_t)stream);
}

int sg_weighted_partial_f32(int nw, const double* weights, const uint8_t* compressed, const float* dense,
                            int64_t ld_dense, const uint32_t* idx, const float* val, const int64_t* row_ptr,
                            const int32_t* tile_off, int64_t dim, float* out, const uint8_t* guard,
                            int guard_n, void* workspace, size_t workspace_bytes, void* stream) {
    if (!out || !guard || guard_n < 1 || guard_n > MAX_WORKERS) return SG_ERR_INVALID;
    return aggregate<float, float>(nw, weights, compressed, dense, ld_dense, idx, val,
                                   reinterpret_cast<const long long*>(row_ptr), tile_off, dim, out, nullptr,
                                   nullptr, 0.0, 0.0, 0.0, 0, workspace, workspace_bytes, (cudaStream_t)stream,
                                   -1, guard, guard_n, 2);
}

int64_t sg_peer_slice_len(int64_t dim, int nranks) {
    if (dim < 1 || nranks < 1) return -1;
    return peer_slice_len(dim, nranks);
}

int sg_peer_reduce_slice_f32(int nranks, const float* const* src, const double* weights, int rank,
                             const uint8_t* guard, int guard_n, int64_t dim, float* dst, void* stream) {
    if (nranks < 1 || nranks > MAX_PEERS || !src || !dst || rank < 0 || rank >= nranks || dim < 1 ||
        guard_n < 0 || guard_n > MAX_WORKERS || (guard_n > 0 && !guard))
        return SG_ERR_INVALID;
    if (dim >= (1ll << 31)) return SG_ERR_UNSUPPORTED;
    PeerRows r = {};
    for (int i = 0; i < nranks; ++i) {
        if (!src[i] || reinterpret_cast<size_t>(src[i]) % 16) return SG_ERR_UNSUPPORTED;
        r.p[i] = src[i];
        r.w[i] = weights ? weights[i] : 1.0;
    }
    if (reinterpret_cast<size_t>(dst) % 16) return SG_ERR_UNSUPPORTED;
    const long long L = peer_slice_len(dim, nranks);
    long long lo = (long long)rank * L, hi = lo + L < dim ? lo + L : dim;
    if (lo > dim) lo = dim;
    if (hi < lo) hi = lo;
    PeerDst d = {};
    d.p[0] = dst;
    launch_pdl(k_peer_reduce_slice, dim3((unsigned)peer_blocks((hi - lo) / 4 / 2 + 1)), dim3(256), 0,
               (cudaStream_t)stream, r, nranks, weights ? 0 : 1, lo, hi, guard_n > 0 ? guard : nullptr, guard_n, d, 1);
    return cudaGetLastError() == cudaSuccess ? SG_OK : SG_ERR_CUDA;
}

int sg_peer_reduce_push_f32(int nranks, const float* const* src, const double* weights, int rank,
                            const uint8_t* guard, int guard_n, int64_t dim, float* const* dsts, void* stream) {
    if (nranks < 1 || nranks > MAX_PEERS || !src || !dsts || rank < 0 || rank >= nranks || dim < 1 ||
        guard_n < 0 || guard_n > MAX_WORKERS || (guard_n > 0 && !guard))
        return SG_ERR_INVALID;
    if (dim >= (1ll << 31)) return SG_ERR_UNSUPPORTED;
    PeerRows r = {};
    PeerDst d = {};
    for (int i = 0; i < nranks; ++i) {
        if (!src[i] || !dsts[i] || reinterpret_cast<size_t>(src[i]) % 16 || reinterpret_cast<size_t>(dsts[i]) % 16)
            return SG_ERR_UNSUPPORTED;
        r.p[i] = src[i];
        r.w[i] = weights ? weights[i] : 1.0;
        d.p[i] = dsts[(rank + 1 + i) % nranks];  // stagger the push targets over the ranks
    }
    const long long L = peer_slice_len(dim, nranks);
    long long lo = (long long)rank * L, hi = lo + L < dim ? lo + L : dim;
    if (lo > dim) lo = dim;
    if (hi < lo) hi = lo;
    launch_pdl(k_peer_reduce_slice, dim3((unsigned)peer_blocks((hi - lo) / 4 / 2 + 1)), dim3(256), 0,
               (cudaStream_t)stream, r, nranks, weights ? 0 : 1, lo, hi, guard_n > 0 ? guard : nullptr, guard_n, d,
               nranks);
    return cudaGetLastError() == cudaSuccess ? SG_OK : SG_ERR_CUDA;
}

int sg_nvls_reduce_bcast_f32(int nranks, int rank, const float* mc_src, float* mc_dst, int64_t dim,
                             const uint8_t* guard, int guard_n, void* stream) {
    if (nranks < 1 || rank < 0 || rank >= nranks || !mc_src || !mc_dst || dim < 1 || guard_n < 0 ||
        guard_n > MAX_WORKERS || (guard_n > 0 && !guard))
        return SG_ERR_INVALID;
    if (reinterpret_cast<size_t>(mc_src) % 16 || reinterpret_cast<size_t>(mc_dst) % 16) return SG_ERR_UNSUPPORTED;
    const long long L = peer_slice_len(dim, nranks);
    long long lo = (long long)rank * L, hi = lo + L < dim ? lo + L : dim;
    if (lo > dim) lo = dim;
    if (hi < lo) hi = lo;
    launch_pdl(k_nvls_reduce_bcast, dim3((unsigned)peer_blocks((hi - lo) / 4 / 4 + 1)), dim3(256), 0,
               (cudaStream_t)stream, mc_src, mc_dst, lo, hi, guard_n > 0 ? guard : nullptr, guard_n);
    return cudaGetLastError() == cudaSuccess ? SG_OK : SG_ERR_CUDA;
}

size_t sg_dense_exchange_flag_words(int64_t dim, int nranks) {
    if (dim < 1 || nranks < 1) return 0;
    const long long nchunk = (dim + XC - 1) / XC;
    return (size_t)nchunk * (size_t)nranks + (size_t)nchunk;
}

int sg_dense_exchange_f32(int nranks, int rank, int k, const double* weights, const float* dense, int64_t ld,
                          int64_t dim, const float* const* partials, float* const* aggs, unsigned* const* flags,
                          unsigned epoch, const uint8_t* guard, int guard_n, float* out, float* params,
                          float* momentum_buf, double lr, double momentum, double weight_decay, int first_step,
                          void* stream) {
    if (nranks < 1 || nranks > MAX_PEERS || rank < 0 || rank >= nranks || !partials || !aggs || !flags || dim < 1 ||
        !params || !momentum_buf || guard_n < 0 || guard_n > MAX_WORKERS || (guard_n > 0 && !guard) || epoch == 0)
        return SG_ERR_INVALID;
    if (dense && (k < 1 || k > 8 || !weights || ld < dim)) return SG_ERR_INVALID;
    if (dim >= (1ll << 31)) return SG_ERR_UNSUPPORTED;
    DxArgs a = {};
    a.dense = dense;
    a.ld = ld;
    a.dim = dim;
    a.k = dense ? k : 0;
    a.P = nranks;
    a.rank = rank;
    a.nchunk = (int)((dim + XC - 1) / XC);
    for (int j = 0; dense && j < k; ++j) a.w.v[j] = weights[j];
    const long long pw = (long long)a.nchunk * nranks;  // pflag words; aflag follows
    for (int q = 0; q < nranks; ++q) {
        if (!partials[q] || !aggs[q] || !flags[q] || reinterpret_cast<size_t>(partials[q]) % 16 ||
            reinterpret_cast<size_t>(aggs[q]) % 16)
            return SG_ERR_UNSUPPORTED;
        a.partial_src[q] = partials[q];
        a.agg[q] = aggs[q];
        a.pflag[q] = flags[q];
        a.aflag[q] = flags[q] + pw;
    }
    a.partial_own = const_cast<float*>(partials[rank]);
    a.agg_own = aggs[rank];
    a.pflag_own = flags[rank];
    a.aflag_own = flags[rank] + pw;
    a.epoch = epoch;
    a.guard = guard_n > 0 ? guard : nullptr;
    a.gn = guard_n;
    a.out = out;
    a.p = params;
    a.b = momentum_buf;
    a.lr = lr;
    a.mu = momentum;
    a.wd = weight_decay;
    a.first = first_step;
    if (reinterpret_cast<size_t>(params) % 16 || reinterpret_cast<size_t>(momentum_buf) % 16 ||
        (out && reinterpret_cast<size_t>(out) % 16) || (dense && (reinterpret_cast<size_t>(dense) % 16 || ld % 4)))
        return SG_ERR_UNSUPPORTED;
    a.roles_per = num_sms();  // one CTA per SM per role, all co-resident (cooperative launch)
    launch_coop(k_dense_exchange, dim3((unsigned)(3 * a.roles_per)), dim3(256), 0, (cudaStream_t)stream, a);
    return cudaGetLastError() == cudaSuccess ? SG_OK : SG_ERR_CUDA;
}

int sg_peer_allgather_sgd_f32(int nranks, const float* const* src, int rank, const uint8_t* guard, int guard_n,
                              int64_t dim, float* out, float* params, float* momentum_buf, double lr, double momentum,
                              double weight_decay, int first_step, void* stream) {
    if (nranks < 1 || nranks > MAX_PEERS || !src || dim < 1 || !params || !momentum_buf || guard_n < 0 ||
        rank < 0 || rank >= nranks ||
        guard_n > MAX_WORKERS || (guard_n > 0 && !guard))
        return SG_ERR_INVALID;
    if (dim >= (1ll << 31)) return SG_ERR_UNSUPPORTED;
    PeerRows r = {};
    for (int i = 0; i < nranks; ++i) {
        if (!src[i] || reinterpret_cast<size_t>(src[i]) % 16) return SG_ERR_UNSUPPORTED;
        r.p[i] = src[i];
    }
    if (reinterpret_cast<size_t>(params) % 16 || reinterpret_cast<size_t>(momentum_buf) % 16 ||
        (out && reinterpret_cast<size_t>(out) % 16))
        return SG_ERR_UNSUPPORTED;
    launch_pdl(k_peer_allgather_sgd, dim3((unsigned)peer_blocks(dim / 4 / 2 + 1)), dim3(256), 0, (cudaStream_t)stream,
               r, nranks, rank, (long long)peer_slice_len(dim, nranks), guard_n > 0 ? guard : nullptr, guard_n,
               (long long)dim,
               out, params, momentum_buf, lr, momentum, weight_decay, first_step);
    return cudaGetLastError() == cudaSuccess ? SG_OK : SG_ERR_CUDA;
}

int sg_multicast_copy_u32(const void* src, void* mc_dst, int64_t words, void* stream) {
    if (!src || !mc_dst || words < 4 || words % 4 || reinterpret_cast<size_t>(src) % 16 ||
        reinterpret_cast<size_t>(mc_dst) % 16)
        return SG_ERR_INVALID;
    const long long n4 = words / 4;
    launch_pdl(k_mc_copy, dim3((unsigned)peer_blocks(n4 / 4 + 1)), dim3(256), 0, (cudaStream_t)stream,
               reinterpret_cast<const uint4*>(src), reinterpret_cast<float*>(mc_dst), n4);
    return cudaGetLastError() == cudaSuccess ? SG_OK : SG_ERR_CUDA;
}

int sg_peer_signal_wait(int nranks, int rank, unsigned* const* flags, int slot, unsigned epoch, unsigned* counter,
                        const uint8_t* guard, int guard_n, const uint8_t* const* dec_src, int64_t dec_each,
                        uint8_t* dec_dst, void* stream) {
    if (nranks < 1 || nranks > MAX_PEERS || rank < 0 || rank >= nranks || !flags || slot < 0 || guard_n < 0 ||
        guard_n > MAX_WORKERS || (guard_n > 0 && !guard) || (epoch == 0 && !counter) || (dec_dst && (!dec_src || dec_each < 1)))
        return SG_ERR_INVALID;
    FlagPtrs f{};
    for (int i = 0; i < nranks; ++i) {
        if (!flags[i]) return SG_ERR_INVALID;
        f.p[i] = flags[i];
    }
    GatherSrc g{};
    if (dec_dst)
        for (int i = 0; i < nranks; ++i) {
            if (!dec_src[i]) return SG_ERR_INVALID;
            g.p[i] = dec_src[i];
        }
    launch_pdl(k_peer_signal_wait, dim3(1), dim3(32), 0, (cudaStream_t)stream, f, nranks, rank, slot, epoch, counter,
               guard_n > 0 ? guard : nullptr, guard_n, g, (long long)dec_each, dec_dst);
    return cudaGetLastError() == cudaSuccess ? SG_OK : SG_ERR_CUDA;
}

int sg_gather_bytes(int nsrc, const uint8_t* const* src, int64_t each, uint8_t* dst, void* stream) {
    if (nsrc < 1 || nsrc > MAX_WORKERS || each < 1 || !src || !dst) return SG_ERR_INVALID;
    GatherSrc g;
    for (int i = 0; i < nsrc; ++i) {
        if (!src[i]) return SG_ERR_INVALID;
        g.p[i] = src[i];
    }
    const long long n = (long long)nsrc * each;
    long long blocks = (n + 255) / 256;
    if (blocks > 1024) blocks = 1024;
    launch_pdl(k_gather_bytes, dim3((unsigned)blocks), dim3(256), 0, (cudaStream_t)stream, g, nsrc, (long long)each, dst);
    return cudaGetLastError() == cudaSuccess ? SG_OK : SG_ERR_CUDA;
}

}  // extern "C"
