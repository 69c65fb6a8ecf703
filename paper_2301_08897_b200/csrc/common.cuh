// Shared device helpers for the ScaDLES B200 hot path (sm_100a only).
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <mutex>
#include <tuple>
#include <vector>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "../../include/scadles_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "scadles_b200 is built for sm_100a only"
#endif

#define SG_DEV __device__ __forceinline__

namespace sg {

constexpr unsigned FULL = 0xffffffffu;
constexpr int MAX_WORKERS = 64;
constexpr int MAX_PEERS = 8;  // GPUs of one NVSwitch node in a peer-memory exchange

// ---------------------------------------------------------------------------------------
// Top-k ordering key.  The reference orders by np.lexsort((arange, -|g|)) (comm.py:94):
// descending |g|, NaN last (below every number), -0 == +0, ties to the lower index.
// key = isnan(x) ? 0 : bits(|x|) + 1 is monotone in |x| with those properties and never
// overflows because bits(|x|) <= bits(inf) for non-NaN x.
// ---------------------------------------------------------------------------------------
template <typename T> struct KeyOf;
template <> struct KeyOf<float> {
    using K = uint32_t;
    static constexpr K KMAX = 0x7f800001u;
    static constexpr int BITS = 32;
    static SG_DEV K key(float x) {
        uint32_t b = __float_as_uint(x) & 0x7fffffffu;
        return b > 0x7f800000u ? 0u : b + 1u;
    }
};
template <> struct KeyOf<double> {
    using K = unsigned long long;
    static constexpr K KMAX = 0x7ff0000000000001ull;
    static constexpr int BITS = 64;
    static SG_DEV K key(double x) {
        unsigned long long b = (unsigned long long)__double_as_longlong(x) & 0x7fffffffffffffffull;
        return b > 0x7ff0000000000000ull ? 0ull : b + 1ull;
    }
};

// 16-byte vectors (one 128-bit LDG per thread per round).
template <typename T> struct Vec16;
template <> struct Vec16<float> {
    using V = float4;
    using I = uint4;
    static constexpr int N = 4;
    static SG_DEV float get(const V& v, int c) { return c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w; }
};
template <> struct Vec16<double> {
    using V = double2;
    using I = uint2;
    static constexpr int N = 2;
    static SG_DEV double get(const V& v, int c) { return c == 0 ? v.x : v.y; }
};

// Streaming 128-bit loads: read-only path, no L1 allocation (each byte is read once).
SG_DEV float4 ld_stream(const float4* p) {
    float4 r;
    asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
        : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
}
SG_DEV double2 ld_stream(const double2* p) {
    double2 r;
    asm("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}
SG_DEV uint4 ld_stream(const uint4* p) {
    uint4 r;
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
SG_DEV uint2 ld_stream(const uint2* p) {
    uint2 r;
    asm("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}

// Relaxed gpu-scope 64-bit status words for decoupled look-back (flag and value share
// one word, so single-copy atomicity is all the ordering the protocol needs).
SG_DEV unsigned long long ld_relaxed(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
SG_DEV void st_relaxed(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

SG_DEV unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <typename K> SG_DEV K warp_max(K v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        K u = __shfl_xor_sync(FULL, v, o);
        v = u > v ? u : v;
    }
    return v;
}
template <typename K> SG_DEV K warp_min(K v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        K u = __shfl_xor_sync(FULL, v, o);
        v = u < v ? u : v;
    }
    return v;
}
// Fixed-order butterfly: every lane ends with the same bits regardless of scheduling.
SG_DEV double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(FULL, v, o));
    return v;
}
SG_DEV unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

template <typename K> SG_DEV int bitlen(K x) {
    if (sizeof(K) == 8) return 64 - __clzll((long long)x);
    return 32 - __clz((int)x);
}

// Look-back status word: [63:62] flag, [61:0] value.
constexpr unsigned long long ST_FLAG_AGG = 1ull << 62;
constexpr unsigned long long ST_FLAG_PRE = 2ull << 62;
constexpr unsigned long long ST_VALUE = (1ull << 62) - 1;

// Warp-cooperative decoupled look-back (Merrill & Garland).  Called by all 32 lanes of one
// warp; `status` points at this worker's tile array; returns the exclusive prefix of `tile`
// and publishes the inclusive one.  Values are summed as integers, so packed counters work
// as long as no field overflows.
SG_DEV unsigned long long lookback(unsigned long long* status, long long tile,
                                   unsigned long long agg) {
    const int lane = threadIdx.x & 31;
    if (tile == 0) {
        if (lane == 0) st_relaxed(status, ST_FLAG_PRE | agg);
        return 0;
    }
    if (lane == 0) st_relaxed(status + tile, ST_FLAG_AGG | agg);
    unsigned long long prefix = 0;
    long long look = tile - 1;
    for (;;) {
        long long i = look - lane;
        unsigned long long s = i >= 0 ? ld_relaxed(status + i) : ST_FLAG_PRE;
        while (__any_sync(FULL, (s >> 62) == 0)) {
            if ((s >> 62) == 0) {
                __nanosleep(20);
                s = ld_relaxed(status + i);
            }
        }
        unsigned pre = __ballot_sync(FULL, (s >> 62) == 2);
        if (pre) {
            int first = __ffs(pre) - 1;
            prefix += warp_sum_u64(lane <= first ? (s & ST_VALUE) : 0ull);
            break;
        }
        prefix += warp_sum_u64(s & ST_VALUE);
        look -= 32;
    }
    if (lane == 0) st_relaxed(status + tile, ST_FLAG_PRE | (prefix + agg));
    return prefix;
}

// IEEE binary64 round-to-nearest, never contracted into FMA: bit parity with numpy.
SG_DEV double dmul(double a, double b) { return __dmul_rn(a, b); }
SG_DEV double dadd(double a, double b) { return __dadd_rn(a, b); }
SG_DEV double dsub(double a, double b) { return __dsub_rn(a, b); }
SG_DEV double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// ---- TMA bulk copies + mbarriers (sm_90+ async proxy; SASS UBLKCP / SYNCS) ----------------
SG_DEV unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
SG_DEV void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
SG_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
SG_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
SG_DEV void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// global -> shared bulk copy (bytes % 16 == 0, both addresses 16-byte aligned), completion
// counted on `bar`; evict-first L2 policy since every byte is read exactly once.
SG_DEV void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar, unsigned long long policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy) : "memory");
}
SG_DEV unsigned long long policy_evict_first() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
SG_DEV void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
SG_DEV void mbar_wait(unsigned long long* bar, unsigned parity) {
    unsigned done = 0;
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    } while (!done);
}

// shared -> global bulk copy (TMA store, bulk-group completion).
SG_DEV void bulk_s2g(void* dst, const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 ::"l"(dst), "r"(smem_u32(src)), "r"(bytes) : "memory");
}
SG_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
SG_DEV void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
SG_DEV void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
SG_DEV void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// Bulk prefetch of [src, src + bytes) into L2 (no registers, no shared memory, no completion);
// src 16-byte aligned, bytes a multiple of 16.
SG_DEV void bulk_prefetch_l2(const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// 4-byte asynchronous global -> shared copy (LDGSTS) and its group fences.
SG_DEV void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
SG_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> SG_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Named CTA barriers (id 0 is __syncthreads): producer/consumer hand-offs between warp roles.
SG_DEV void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
SG_DEV void bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// Programmatic dependent launch: every kernel of the chain is launched with programmatic
// stream serialisation, lets its dependent grid launch as soon as all of its own CTAs are
// running (pdl_trigger) and waits for its prerequisite grid before touching its outputs
// (pdl_wait, a no-op without the launch attribute).  Every kernel calls both first thing,
// so completion stays transitive along the chain.  SG_PDL=0 turns the attribute off.
SG_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
SG_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
SG_DEV void pdl_enter() {
    pdl_trigger();
    pdl_wait();
}

inline bool pdl_on() {
    static const bool on = [] {
        const char* e = getenv("SG_PDL");
        return !(e && *e == '0');
    }();
    return on;
}

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_on() ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

SG_DEV unsigned ld_acquire_gpu(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Cooperative launch (every CTA co-resident, for an in-kernel grid barrier) with programmatic
// stream serialisation; without PDL support for the combination it launches cooperative only.
template <typename... KArgs, typename... Args>
inline void launch_coop(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                        Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_on() ? 2 : 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
    if (e != cudaSuccess && cfg.numAttrs == 2) {
        cudaGetLastError();
        if (getenv("SG_COOP_REPORT")) fprintf(stderr, "[scadles_b200] cooperative+PDL launch refused: %s\n", cudaGetErrorString(e));
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
    } else if (getenv("SG_COOP_REPORT")) {
        fprintf(stderr, "[scadles_b200] cooperative launch with %d attribute(s): %s\n", cfg.numAttrs, cudaGetErrorString(e));
    }
}

// SG_DEBUG_SYNC=1: synchronise after every launch and report the first failing kernel.
inline void debug_sync(const char* what, cudaStream_t stream) {
    static const bool on = [] {
        const char* e = getenv("SG_DEBUG_SYNC");
        return e && *e == '1';
    }();
    if (!on) return;
    const cudaError_t e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) fprintf(stderr, "[scadles_b200] %s: %s\n", what, cudaGetErrorString(e));
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device, size): the
// attribute is a per-context property, so the launchers do not pay the driver call per launch.
inline cudaError_t smem_attr(const void* kern, int bytes) {
    static std::mutex mu;
    static std::vector<std::tuple<const void*, int, int>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    for (auto& t : done)
        if (std::get<0>(t) == kern && std::get<1>(t) == dev && std::get<2>(t) >= bytes) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.emplace_back(kern, dev, bytes);
    return e;
}

// Diagnostic build only (-DSG_STAMPS via SG_NVCC_EXTRA): per-kernel first-CTA start and
// last-CTA end on %globaltimer, one slot pair per kernel id and translation unit, read and
// reset by sg_diag_stamps_<tu> (tools/stamps.py).  The product build compiles none of it.
#ifdef SG_STAMPS
SG_DEV unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
static __device__ unsigned long long g_stamp[2 * 16];
struct StampScope {
    int id;
    __device__ explicit StampScope(int i) : id(i) {
        if (threadIdx.x == 0) atomicMin(&g_stamp[2 * id], gtimer());
    }
    __device__ ~StampScope() {
        if (threadIdx.x == 0) atomicMax(&g_stamp[2 * id + 1], gtimer());
    }
};
#define SG_STAMP(id) ::sg::StampScope sg_stamp_scope_##id(id)
// first and last CTA (thread 0) to reach this point
#define SG_MARK(id)                                               \
    do {                                                          \
        if (threadIdx.x == 0) {                                   \
            const unsigned long long t_ = ::sg::gtimer();         \
            atomicMin(&::sg::g_stamp[2 * (id)], t_);              \
            atomicMax(&::sg::g_stamp[2 * (id) + 1], t_);          \
        }                                                         \
    } while (0)
#define SG_STAMPS_EXPORT(name)                                                             \
    extern "C" int name(unsigned long long* out) {                                        \
        if (cudaMemcpyFromSymbol(out, ::sg::g_stamp, sizeof(::sg::g_stamp)) != cudaSuccess) \
            return SG_ERR_CUDA;                                                            \
        unsigned long long init[2 * 16];                                                   \
        for (int i = 0; i < 16; ++i) {                                                     \
            init[2 * i] = ~0ull;                                                           \
            init[2 * i + 1] = 0ull;                                                        \
        }                                                                                  \
        return cudaMemcpyToSymbol(::sg::g_stamp, init, sizeof(init)) == cudaSuccess ? SG_OK : SG_ERR_CUDA; \
    }
#else
#define SG_STAMP(id) do { } while (0)
#define SG_MARK(id) do { } while (0)
#define SG_STAMPS_EXPORT(name)
#endif

// Diagnostic build only (-DSG_CHECKS): device-side bounds checks on the hot path's computed
// addresses (candidate slots, output slots, merge offsets, staged merge entries, sampler
// rows); a failed check prints the site and traps.  compute-sanitizer is closed on this GPU
// pool, so tools/checked_run.py runs the GPU tests and the race stress on this build instead.
#ifdef SG_CHECKS
#define SG_CHECK(cond)                                                                          \
    do {                                                                                        \
        if (!(cond)) {                                                                          \
            printf("[scadles_b200] check failed %s:%d: %s\n", __FILE__, __LINE__, #cond);      \
            __trap();                                                                           \
        }                                                                                       \
    } while (0)
#else
#define SG_CHECK(cond) do { } while (0)
#endif

inline int num_sms() {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
}

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace sg
