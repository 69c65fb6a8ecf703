// Weighted aggregation with decompression (item 2 + sparse merge-densify) and momentum SGD.
//
// Replaces reference pkg/src/streamsgd/comm.py:67-78 (weighted_aggregate: acc = zeros(D);
// for each worker in order acc += w_j * densify(g_j)), comm.py:45-50 (densify) and
// nn.py:161-172 (sgd_momentum_step).
//
// Output-tile merge: every CTA owns one 4096-element output tile held as float64 in shared
// memory.  Workers are folded in ascending order (a __syncthreads between workers): a dense
// worker streams its tile with 128-bit loads, a sparse worker streams only the (idx, val)
// pairs that fall in the tile, located through a per-worker tile-offset table built by
// k_tile_offsets from the ascending indices.  No atomics, so the result is deterministic
// and identical on every rank.  Arithmetic is binary64 round-to-nearest without contraction
// (acc = acc + w*x), which is exactly numpy's `acc += weight * densify(g)` on the upcast
// inputs; the single rounding to the output type happens once, at the store.  Positions a
// sparse worker does not keep would add w*(+0.0) in the reference: a no-op on an accumulator
// that starts at +0.0, so they are skipped.  With params/buf the momentum-SGD step runs in
// the epilogue on the unrounded float64 aggregate (nn.py:169-171 operation order).
#include "common.cuh"

namespace sg {

constexpr int AG_THREADS = 256;
constexpr int AG_TILE = 4096;  // 16 elements per thread
constexpr int AG_PER_THREAD = AG_TILE / AG_THREADS;
static_assert(AG_PER_THREAD == 16, "4 groups of 4 consecutive elements per thread");

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

// off[j][t] = number of row-j entries with index < t*AG_TILE, t in [0, ntiles].
__global__ void k_tile_offsets(const uint32_t* __restrict__ idx, const long long* __restrict__ row_ptr,
                               const uint8_t* __restrict__ comp, long long ntiles, int* __restrict__ off) {
    const int j = blockIdx.y;
    if (comp && !comp[j]) return;
    const long long r0 = row_ptr[j], nnz = row_ptr[j + 1] - r0;
    int* o = off + (long long)j * (ntiles + 1);
    const uint32_t* ix = idx + r0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long first = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (nnz == 0) {
        for (long long t = first; t <= ntiles; t += stride) o[t] = 0;
        return;
    }
    for (long long p = first; p < nnz; p += stride) {
        const long long tc = ix[p] / AG_TILE;
        const long long tp = p ? (long long)(ix[p - 1] / AG_TILE) : -1;
        for (long long t = tp + 1; t <= tc; ++t) o[t] = (int)p;
        if (p == nnz - 1)
            for (long long t = tc + 1; t <= ntiles; ++t) o[t] = (int)nnz;
    }
}

template <typename TI, typename TO> struct AggArgs {
    double w[MAX_WORKERS];
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
};

template <typename TI, typename TO>
__global__ void __launch_bounds__(AG_THREADS)
k_aggregate(const AggArgs<TI, TO> a) {
    __shared__ double acc[AG_TILE];
    __shared__ uint8_t s_comp[MAX_WORKERS];
    __shared__ long long s_rp[MAX_WORKERS];
    const int tid = threadIdx.x;
    const long long tile = blockIdx.x;
    const long long tb = tile * AG_TILE;
    const bool full = a.vec_ok && tb + AG_TILE <= a.dim;
    for (int i = tid; i < a.nw; i += AG_THREADS) {
        s_comp[i] = a.comp ? a.comp[i] : 0;
        s_rp[i] = a.row_ptr ? a.row_ptr[i] : 0;
    }
#pragma unroll
    for (int q = 0; q < AG_PER_THREAD; ++q) acc[q * AG_THREADS + tid] = 0.0;
    __syncthreads();
    for (int j = 0; j < a.nw; ++j) {
        const double wj = a.w[j];
        if (!s_comp[j]) {
            const TI* row = a.dense + (long long)j * a.ld + tb;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int e = r * (AG_THREADS * 4) + tid * 4;
                double x[4];
                if (full) {
                    load4<TI>(row + e, x);
                } else {
#pragma unroll
                    for (int c = 0; c < 4; ++c) x[c] = tb + e + c < a.dim ? (double)row[e + c] : 0.0;
                }
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[e + c] = dadd(acc[e + c], dmul(wj, x[c]));
            }
        } else {
            const int* o = a.off + (long long)j * (a.ntiles + 1);
            const long long lo = s_rp[j] + o[tile], hi = s_rp[j] + o[tile + 1];
            for (long long i = lo + tid; i < hi; i += AG_THREADS) {
                const int pos = (int)(a.idx[i] - (uint32_t)tb);
                acc[pos] = dadd(acc[pos], dmul(wj, (double)a.val[i]));
            }
        }
        __syncthreads();
    }
    const bool first = a.first != 0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int e = r * (AG_THREADS * 4) + tid * 4;
        double g[4] = {acc[e], acc[e + 1], acc[e + 2], acc[e + 3]};
        if (full) {
            if (a.out) store4<TO>(a.out + tb + e, g);
            if (a.p) {
                double pv[4], bv[4] = {0.0, 0.0, 0.0, 0.0};
                load4_rw<TO>(a.p + tb + e, pv);
                if (!first) load4_rw<TO>(a.buf + tb + e, bv);
#pragma unroll
                for (int c = 0; c < 4; ++c) sgd_elem(g[c], pv[c], bv[c], a.lr, a.mu, a.wd, first);
                store4<TO>(a.p + tb + e, pv);
                store4<TO>(a.buf + tb + e, bv);
            }
        } else {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const long long q = tb + e + c;
                if (q >= a.dim) continue;
                if (a.out) a.out[q] = (TO)g[c];
                if (a.p) {
                    double pv = a.p[q], bv = first ? 0.0 : (double)a.buf[q];
                    sgd_elem(g[c], pv, bv, a.lr, a.mu, a.wd, first);
                    a.p[q] = (TO)pv;
                    a.buf[q] = (TO)bv;
                }
            }
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(256)
k_sgd(T* __restrict__ p, T* __restrict__ buf, const T* __restrict__ g, long long dim, double lr,
      double mu, double wd, int first, int vec_ok) {
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

inline long long ag_tiles(long long dim) { return (dim + AG_TILE - 1) / AG_TILE; }

template <typename TI, typename TO>
int aggregate(int nw, const double* weights, const uint8_t* comp, const TI* dense, long long ld,
              const uint32_t* idx, const TI* val, const long long* row_ptr, long long dim, TO* out,
              TO* p, TO* buf, double lr, double mu, double wd, int first, void* ws, size_t ws_bytes,
              cudaStream_t stream) {
    if (nw < 1 || dim < 1 || !weights || (!out && !p)) return SG_ERR_INVALID;
    if (nw > MAX_WORKERS || dim >= (1ll << 31)) return SG_ERR_UNSUPPORTED;
    if (p && !buf) return SG_ERR_INVALID;
    // Sparse workers need idx/val/row_ptr; dense workers need the dense rows.
    if (comp && (!idx || !val || !row_ptr)) return SG_ERR_INVALID;
    if (!dense && !comp) return SG_ERR_INVALID;
    if (dense && ld < dim) return SG_ERR_INVALID;
    const long long ntiles = ag_tiles(dim);
    int* off = nullptr;
    if (comp) {
        const size_t need = sizeof(int) * (size_t)nw * (size_t)(ntiles + 1);
        if (!ws || ws_bytes < need) return SG_ERR_WORKSPACE;
        off = reinterpret_cast<int*>(ws);
        k_tile_offsets<<<dim3(64, nw), 256, 0, stream>>>(idx, row_ptr, comp, ntiles, off);
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
    bool vec = true;
    if (dense) vec = vec && reinterpret_cast<size_t>(dense) % 16 == 0 && (ld * (long long)sizeof(TI)) % 16 == 0;
    if (out) vec = vec && reinterpret_cast<size_t>(out) % 16 == 0;
    if (p) vec = vec && reinterpret_cast<size_t>(p) % 16 == 0 && reinterpret_cast<size_t>(buf) % 16 == 0;
    a.vec_ok = vec;
    k_aggregate<TI, TO><<<(unsigned)ntiles, AG_THREADS, 0, stream>>>(a);
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
    k_sgd<T><<<(unsigned)blocks, 256, 0, stream>>>(p, buf, g, dim, lr, mu, wd, first, vec_ok);
    return cudaGetLastError() == cudaSuccess ? SG_OK : SG_ERR_CUDA;
}

}  // namespace sg

using namespace sg;

extern "C" {

size_t sg_aggregate_workspace_bytes(int nw, int64_t dim) {
    if (nw < 1 || dim < 1) return 0;
    return sizeof(int) * (size_t)nw * (size_t)(ag_tiles(dim) + 1);
}

int sg_weighted_aggregate_f32(int nw, const double* weights, const uint8_t* compressed,
                              const float* dense, int64_t ld_dense, const uint32_t* idx,
                              const float* val, const int64_t* row_ptr, int64_t dim, float* out,
                              float* params, float* momentum_buf, double lr, double momentum,
                              double weight_decay, int first_step, void* workspace,
                              size_t workspace_bytes, void* stream) {
    return aggregate<float, float>(nw, weights, compressed, dense, ld_dense, idx, val,
                                   reinterpret_cast<const long long*>(row_ptr), dim, out, params,
                                   momentum_buf, lr, momentum, weight_decay, first_step, workspace,
                                   workspace_bytes, (cudaStream_t)stream);
}

int sg_weighted_aggregate_f64(int nw, const double* weights, const uint8_t* compressed,
                              const double* dense, int64_t ld_dense, const uint32_t* idx,
                              const double* val, const int64_t* row_ptr, int64_t dim, double* out,
                              double* params, double* momentum_buf, double lr, double momentum,
                              double weight_decay, int first_step, void* workspace,
                              size_t workspace_bytes, void* stream) {
    return aggregate<double, double>(nw, weights, compressed, dense, ld_dense, idx, val,
                                     reinterpret_cast<const long long*>(row_ptr), dim, out, params,
                                     momentum_buf, lr, momentum, weight_decay, first_step, workspace,
                                     workspace_bytes, (cudaStream_t)stream);
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

}  // extern "C"
