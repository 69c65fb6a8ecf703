// Streaming sampler staged on device (item 5): stream id -> train row resolution, non-IID
// injection row lists, and the batch feature gather.
//
// Reference: engine.py:223-227 (batches = [[pools[d][a % len(pools[d])] for a in ids]]),
// datagen.py:182-210 (inject: each sender's picks appended to every other device's batch in
// plan order), engine.py:201-204 (_materialize: x = train_x[idx] + augment[idx]).
// The StreamBuffer's pending ids are always one contiguous range [head, next_id), so a
// draw of b ids is (head, b) and never materialises a Python list.  Random choices (the
// injection plan and picks) stay on the host with the reference's numpy calls and seeds;
// everything that touches sample payloads runs here.
#include "common.cuh"

namespace sg {

__global__ void k_resolve_rows(const long long* __restrict__ head, const long long* __restrict__ b,
                               const long long* __restrict__ out_ptr, const long long* __restrict__ pool_ptr,
                               const long long* __restrict__ pool_rows, long long* __restrict__ out) {
    const int d = blockIdx.y;
    const long long p0 = pool_ptr[d], plen = pool_ptr[d + 1] - p0;
    const long long h = head[d], n = b[d], o = out_ptr[d];
    SG_CHECK(n == 0 || plen > 0);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        out[o + i] = pool_rows[p0 + (h + i) % plen];
}

// Recipient d's augmented batch: own rows, then every other sender's picks in plan order.
__global__ void k_inject_rows(const long long* __restrict__ base_ptr, const long long* __restrict__ base_rows,
                              int n_send, const int* __restrict__ senders, const long long* __restrict__ pick_ptr,
                              const long long* __restrict__ picks, const long long* __restrict__ out_ptr,
                              long long* __restrict__ out_rows) {
    const int d = blockIdx.x;
    long long o = out_ptr[d];
    const long long b0 = base_ptr[d], nb = base_ptr[d + 1] - b0;
    for (long long i = threadIdx.x; i < nb; i += blockDim.x) out_rows[o + i] = base_rows[b0 + i];
    o += nb;
    for (int k = 0; k < n_send; ++k) {
        const int s = senders[k];
        const long long q0 = pick_ptr[k], nq = pick_ptr[k + 1] - q0;
        if (s == d) continue;
        const long long sb = base_ptr[s];
        for (long long i = threadIdx.x; i < nq; i += blockDim.x) out_rows[o + i] = base_rows[sb + picks[q0 + i]];
        o += nq;
    }
}

template <typename T>
__global__ void __launch_bounds__(256)
k_gather(const T* __restrict__ x, const T* __restrict__ aug, const long long* __restrict__ y,
         long long F, const long long* __restrict__ rows, long long n_rows, T* __restrict__ xo,
         long long* __restrict__ yo) {
    for (long long r = blockIdx.x; r < n_rows; r += gridDim.x) {
        const long long src = rows[r];
        const T* xs = x + src * F;
        const T* as = aug ? aug + src * F : nullptr;
        T* xd = xo + r * F;
        for (long long f = threadIdx.x; f < F; f += blockDim.x) {
            if (as) {
                if constexpr (sizeof(T) == 8) xd[f] = dadd(xs[f], as[f]);
                else xd[f] = __fadd_rn(xs[f], as[f]);
            } else {
                xd[f] = xs[f];
            }
        }
        if (threadIdx.x == 0 && yo) yo[r] = y[src];
    }
}

template <typename T>
int gather(const T* x, const T* aug, const long long* y, long long F, const long long* rows, long long n,
           T* xo, long long* yo, cudaStream_t stream) {
    if (!x || !rows || !xo || F < 1 || n < 0) return SG_ERR_INVALID;
    if (yo && !y) return SG_ERR_INVALID;
    if (n == 0) return SG_OK;
    long long grid = n < 65535 ? n : 65535;
    k_gather<T><<<(unsigned)grid, 256, 0, stream>>>(x, aug, y, F, rows, n, xo, yo);
    return cudaGetLastError() == cudaSuccess ? SG_OK : SG_ERR_CUDA;
}

}  // namespace sg

using namespace sg;

extern "C" {

int sg_gather_batch_f64(const double* train_x, const double* augment, const int64_t* train_y,
                        int64_t feature_dim, const int64_t* rows, int64_t n_rows, double* x_out,
                        int64_t* y_out, void* stream) {
    return gather<double>(train_x, augment, reinterpret_cast<const long long*>(train_y), feature_dim,
                          reinterpret_cast<const long long*>(rows), n_rows, x_out,
                          reinterpret_cast<long long*>(y_out), (cudaStream_t)stream);
}

int sg_gather_batch_f32(const float* train_x, const float* augment, const int64_t* train_y,
                        int64_t feature_dim, const int64_t* rows, int64_t n_rows, float* x_out,
                        int64_t* y_out, void* stream) {
    return gather<float>(train_x, augment, reinterpret_cast<const long long*>(train_y), feature_dim,
                         reinterpret_cast<const long long*>(rows), n_rows, x_out,
                         reinterpret_cast<long long*>(y_out), (cudaStream_t)stream);
}

int sg_resolve_stream_rows(int n_dev, const int64_t* head, const int64_t* b, const int64_t* out_ptr,
                           const int64_t* pool_ptr, const int64_t* pool_rows, int64_t total,
                           int64_t* out, void* stream) {
    if (n_dev < 1 || !head || !b || !out_ptr || !pool_ptr || !pool_rows || !out || total < 0)
        return SG_ERR_INVALID;
    if (total == 0) return SG_OK;
    long long per = (total / n_dev + 255) / 256;
    if (per < 1) per = 1;
    if (per > 1024) per = 1024;
    k_resolve_rows<<<dim3((unsigned)per, n_dev), 256, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const long long*>(head), reinterpret_cast<const long long*>(b),
        reinterpret_cast<const long long*>(out_ptr), reinterpret_cast<const long long*>(pool_ptr),
        reinterpret_cast<const long long*>(pool_rows), reinterpret_cast<long long*>(out));
    return cudaGetLastError() == cudaSuccess ? SG_OK : SG_ERR_CUDA;
}

int sg_inject_rows(int n_dev, const int64_t* base_ptr, const int64_t* base_rows, int n_send,
                   const int32_t* senders, const int64_t* pick_ptr, const int64_t* picks,
                   const int64_t* out_ptr, int64_t* out_rows, void* stream) {
    if (n_dev < 1 || !base_ptr || !base_rows || !out_ptr || !out_rows || n_send < 0) return SG_ERR_INVALID;
    if (n_send > 0 && (!senders || !pick_ptr || !picks)) return SG_ERR_INVALID;
    k_inject_rows<<<n_dev, 256, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const long long*>(base_ptr), reinterpret_cast<const long long*>(base_rows), n_send,
        senders, reinterpret_cast<const long long*>(pick_ptr), reinterpret_cast<const long long*>(picks),
        reinterpret_cast<const long long*>(out_ptr), reinterpret_cast<long long*>(out_rows));
    return cudaGetLastError() == cudaSuccess ? SG_OK : SG_ERR_CUDA;
}

}  // extern "C"
