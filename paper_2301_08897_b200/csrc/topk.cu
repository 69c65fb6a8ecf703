// Top-k sparsification + squared norms + adaptive compression gate (items 3 and 4).
//
// Replaces reference pkg/src/streamsgd/comm.py:90-96 (topk_sparsify: lexsort on -|g| with
// index tie-break, kept indices re-sorted ascending) and comm.py:129-160 (compression_gate:
// s_full = g.g, s_topk = v.v, EWMA, rho, decision) for the k workers of one GPU at once.
//
// Pipeline per call (all on one stream, no host synchronisation):
//   k_estimate  one CTA per worker: zero the call's scratch, read a stratified random sample
//               of S keys from HBM and select the r_est-th largest -> a threshold `est`
//               that is below the true m-th largest key with overwhelming probability.
//   k_main      the single full read of the bucket: persistent CTAs take 16 KB tiles by
//               ticket, compute fp64 sum of squares per tile, and stably compact every
//               element with key >= est into a candidate buffer (~1.2-2 m entries) using a
//               decoupled look-back scan, so candidates stay in ascending index order.
//   k_select    2048-bin radix-select rounds over the candidates (L2-resident) with a
//               range-normalised digit; the last CTA of each round picks the bin.  If the
//               estimate undershot (fewer than m candidates) or the buffer overflowed (heavy
//               ties), the rounds run over the full row instead: same result, slower.
//   k_final     stable compaction of {key > T} U {first `need` keys == T} -> idx/val in
//               ascending index order, plus per-tile fp64 sum of kept squares.
//   k_gate      fixed-order reduction of the per-tile partials -> norms2, then the gate
//               update in IEEE round-to-nearest (comm.py:143-159 order of operations).
#include "common.cuh"

namespace sg {

constexpr int TK_THREADS = 256;
constexpr int TK_ROUNDS = 4;  // 16-byte vectors per thread per tile
constexpr int TK_NW = TK_THREADS / 32;
static_assert(TK_ROUNDS * TK_NW == 32, "one warp scans the per-(round, warp) totals");
constexpr int SEL_BITS = 11;
constexpr int SEL_BINS = 1 << SEL_BITS;
constexpr int EST_THREADS = 1024;

enum { MODE_CAND = 0, MODE_FULL = 1 };

template <typename T> struct TopkTraits;
template <> struct TopkTraits<float> {
    static constexpr int SAMPLE = 32768;  // keys in shared memory: 128 KB
    static constexpr int ROUNDS_MAX = 3;  // ceil(31 / 11)
};
template <> struct TopkTraits<double> {
    static constexpr int SAMPLE = 16384;
    static constexpr int ROUNDS_MAX = 6;  // ceil(63 / 11)
};

template <typename T> constexpr int tile_elems() { return TK_THREADS * TK_ROUNDS * Vec16<T>::N; }

template <typename K> struct SelState {
    K lo;                      // current key range [lo, lo + span]
    K span;
    K T;                       // final threshold key
    unsigned long long rank;   // remaining 1-based rank from the top inside the range
    unsigned long long gt;     // elements above the range (all kept)
    unsigned long long n_src;  // elements in the source (candidates or the full row)
    int shift;
    int done;
    int mode;
    int error;
};

// --------------------------------------------------------------------------------------
// Host-side layout of the caller workspace.
// --------------------------------------------------------------------------------------
struct TopkPlan {
    int k;
    long long dim, m;
    long long s_eff, stride, r_est, cap;
    long long nt_main, nt_fin;
    size_t off_status_main, off_status_fin, off_hist, off_ctr, off_count, off_maxkey, zero_end;
    size_t off_est, off_sel, off_sum_main, off_sum_fin, off_cidx, off_cval, total;
};

template <typename T> TopkPlan make_plan(int k, long long dim, long long m) {
    using K = typename KeyOf<T>::K;
    TopkPlan p{};
    p.k = k;
    p.dim = dim;
    p.m = m;
    const long long S = TopkTraits<T>::SAMPLE;
    p.s_eff = dim < S ? dim : S;
    p.stride = dim / (p.s_eff > 0 ? p.s_eff : 1);
    if (p.s_eff == dim) {
        p.r_est = m;  // exact sample: est is the true m-th largest key
        p.cap = dim;
    } else {
        // Keep enough sample ranks that count(key >= est) >= m fails with probability
        // ~1e-9 (6 sigma of the binomial sample count) plus a constant for tiny m.
        const double q = (double)m / (double)dim;
        const double mean = q * (double)p.s_eff;
        const double sd = __builtin_sqrt(mean * (1.0 - q) + 1.0);
        long long r = (long long)(mean + 6.0 * sd + 8.0) + 1;
        p.r_est = r;
        if (r >= p.s_eff) {
            p.cap = dim;
        } else {
            const double expect = (double)r * (double)dim / (double)p.s_eff;
            const double c = expect * 1.25 + 4096.0;
            p.cap = c >= (double)dim ? dim : (long long)c;
        }
    }
    p.cap = (p.cap + 3) / 4 * 4;
    const long long te = tile_elems<T>();
    p.nt_main = (dim + te - 1) / te;
    const long long src_max = p.cap > dim ? p.cap : dim;
    p.nt_fin = (src_max + te - 1) / te;
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + bytes, 256); return r; };
    p.off_status_main = take(sizeof(unsigned long long) * (size_t)k * p.nt_main);
    p.off_status_fin = take(sizeof(unsigned long long) * (size_t)k * p.nt_fin);
    p.off_hist = take(sizeof(unsigned) * (size_t)k * TopkTraits<T>::ROUNDS_MAX * SEL_BINS);
    p.off_ctr = take(sizeof(unsigned) * (2 + (size_t)k * TopkTraits<T>::ROUNDS_MAX));
    p.off_count = take(sizeof(unsigned long long) * (size_t)k);
    p.off_maxkey = take(sizeof(K) * (size_t)k);
    p.zero_end = o;
    p.off_est = take(sizeof(K) * (size_t)k);
    p.off_sel = take(sizeof(SelState<K>) * (size_t)k);
    p.off_sum_main = take(sizeof(double) * (size_t)k * p.nt_main);
    p.off_sum_fin = take(sizeof(double) * (size_t)k * p.nt_fin);
    p.off_cidx = take(sizeof(uint32_t) * (size_t)k * p.cap);
    p.off_cval = take(sizeof(T) * (size_t)k * p.cap);
    p.total = o + 256;  // slack for base alignment
    return p;
}

// --------------------------------------------------------------------------------------
// Shared select helper: warp 0 locates the bin holding the rank-th largest element.
// hist has SEL_BINS counters (bins past the range are zero).  Lane L owns the 64 bins
// [2047-64L-63, 2047-64L]; a warp scan from the top finds the owning lane, which walks
// its bins.  Returns (bin, count strictly above the bin); bin = -1 if rank > total.
// --------------------------------------------------------------------------------------
SG_DEV void find_bin_from_top(const unsigned* hist, unsigned long long rank, int& bin,
                              unsigned long long& above) {
    const int lane = threadIdx.x & 31;
    const int top = SEL_BINS - 1 - 64 * lane;
    unsigned long long s = 0;
    for (int i = 0; i < 64; ++i) s += hist[top - i];
    unsigned long long incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
    }
    const unsigned hit = __ballot_sync(FULL, incl >= rank);
    if (!hit) {
        bin = -1;
        above = 0;
        return;
    }
    const int f = __ffs(hit) - 1;
    int b = -1;
    unsigned long long a = 0;
    if (lane == f) {
        unsigned long long cum = incl - s;
        for (int i = 0; i < 64; ++i) {
            const unsigned h = hist[top - i];
            if (cum + h >= rank) {
                b = top - i;
                a = cum;
                break;
            }
            cum += h;
        }
    }
    bin = __shfl_sync(FULL, b, f);
    above = __shfl_sync(FULL, a, f);
}

template <typename K> SG_DEV int digit_shift(K span) {
    const int bl = bitlen<K>(span);
    return bl > SEL_BITS ? bl - SEL_BITS : 0;
}

// Advance a select state after the bin holding the remaining rank was found.
template <typename K> SG_DEV void advance(SelState<K>& s, int bin, unsigned long long above) {
    if (bin < 0) {
        s.error = 1;
        s.done = 1;
        s.T = 0;
        return;
    }
    const K off = (K)bin << s.shift;
    s.rank -= above;
    s.gt += above;
    s.lo += off;
    if (s.shift == 0) {
        s.span = 0;
        s.T = s.lo;
        s.done = 1;
        return;
    }
    const K width = ((K)1 << s.shift) - 1;
    const K rest = s.span - off;
    s.span = rest < width ? rest : width;
    s.shift = digit_shift<K>(s.span);
}

// --------------------------------------------------------------------------------------
// k_estimate: zero scratch, sample, select the r_est-th largest sample key.
// --------------------------------------------------------------------------------------
SG_DEV unsigned long long mix64(unsigned long long x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

template <typename T>
__global__ void __launch_bounds__(EST_THREADS)
k_estimate(const T* __restrict__ g, long long ld, long long s_eff, long long stride,
           long long r_est, typename KeyOf<T>::K* __restrict__ est,
           uint4* __restrict__ zero, long long zero_vec) {
    using KO = KeyOf<T>;
    using K = typename KO::K;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K* sk = reinterpret_cast<K*>(smem_raw);
    __shared__ unsigned hist[SEL_BINS];
    __shared__ SelState<K> st;
    const int w = blockIdx.x, tid = threadIdx.x;

    // Zero the per-call scratch (look-back status words, histograms, counters).
    for (long long i = (long long)w * EST_THREADS + tid; i < zero_vec; i += (long long)gridDim.x * EST_THREADS)
        zero[i] = make_uint4(0, 0, 0, 0);

    const T* row = g + (long long)w * ld;
    for (long long i = tid; i < s_eff; i += EST_THREADS) {
        long long pos = i * stride;
        if (stride > 1) pos += (long long)(mix64((unsigned long long)i * 0x9e3779b97f4a7c15ull + (unsigned long long)w) % (unsigned long long)stride);
        sk[i] = KO::key(row[pos]);
    }
    if (tid == 0) {
        st.lo = 0;
        st.span = KO::KMAX;
        st.rank = (unsigned long long)r_est;
        st.gt = 0;
        st.n_src = (unsigned long long)s_eff;
        st.shift = digit_shift<K>(st.span);
        st.done = 0;
        st.mode = MODE_FULL;
        st.error = 0;
        st.T = 0;
    }
    __syncthreads();
    if (r_est > s_eff) {
        if (tid == 0) est[w] = 0;
        return;
    }
    for (int round = 0; round < TopkTraits<T>::ROUNDS_MAX + 1; ++round) {
        for (int i = tid; i < SEL_BINS; i += EST_THREADS) hist[i] = 0;
        __syncthreads();
        const K lo = st.lo, span = st.span;
        const int shift = st.shift;
        for (long long i = tid; i < s_eff; i += EST_THREADS) {
            const K key = sk[i];
            if (key >= lo && key - lo <= span) atomicAdd(&hist[(unsigned)((key - lo) >> shift)], 1u);
        }
        __syncthreads();
        if (tid < 32) {
            int bin;
            unsigned long long above;
            find_bin_from_top(hist, st.rank, bin, above);
            if (tid == 0) advance<K>(st, bin, above);
        }
        __syncthreads();
        if (st.done) break;
    }
    if (tid == 0) est[w] = st.done && !st.error ? st.T : (K)0;
}

// --------------------------------------------------------------------------------------
// k_main: the single streaming pass over the bucket.
// --------------------------------------------------------------------------------------
template <typename T> struct MainArgs {
    const T* g;
    long long ld, dim, ntiles, cap;
    int k, vec_ok;
    const typename KeyOf<T>::K* est;
    uint32_t* cidx;
    T* cval;
    unsigned long long* status;
    unsigned* ticket;
    double* sumsq;
    unsigned long long* count;
    typename KeyOf<T>::K* maxkey;
};

// Per-lane exclusive prefix and warp total of a small count n (0..4) via 3 ballots.
SG_DEV void warp_scan_small(unsigned n, unsigned& excl, unsigned& total) {
    const unsigned b0 = __ballot_sync(FULL, n & 1u);
    const unsigned b1 = __ballot_sync(FULL, n & 2u);
    const unsigned b2 = __ballot_sync(FULL, n & 4u);
    const unsigned lt = lanemask_lt();
    excl = __popc(b0 & lt) + 2u * __popc(b1 & lt) + 4u * __popc(b2 & lt);
    total = __popc(b0) + 2u * __popc(b1) + 4u * __popc(b2);
}

template <typename T>
__global__ void __launch_bounds__(TK_THREADS)
k_main(MainArgs<T> a) {
    using KO = KeyOf<T>;
    using K = typename KO::K;
    using VT = Vec16<T>;
    constexpr int V = VT::N;
    constexpr int TILE = tile_elems<T>();
    __shared__ unsigned s_ticket;
    __shared__ unsigned s_wtot[32];
    __shared__ unsigned s_woff[32];
    __shared__ double s_wsum[TK_NW];
    __shared__ K s_wmax[TK_NW];
    __shared__ unsigned long long s_base;
    __shared__ K s_blkmax[MAX_WORKERS];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned long long total = (unsigned long long)a.k * (unsigned long long)a.ntiles;
    for (int i = tid; i < a.k; i += TK_THREADS) s_blkmax[i] = 0;

    for (;;) {
        if (tid == 0) s_ticket = atomicAdd(a.ticket, 1u);
        __syncthreads();
        const unsigned long long t = s_ticket;
        if (t >= total) break;
        const int w = (int)(t / (unsigned long long)a.ntiles);
        const long long tile = (long long)(t - (unsigned long long)w * a.ntiles);
        const T* row = a.g + (long long)w * a.ld;
        const long long base = tile * TILE;
        const K est = a.est[w];

        T v[TK_ROUNDS][V];
        unsigned cm[TK_ROUNDS];
        double ss = 0.0;
        K mx = 0;
        if (a.vec_ok && base + TILE <= a.dim) {
            typename VT::V x[TK_ROUNDS];
            const typename VT::V* src = reinterpret_cast<const typename VT::V*>(row + base);
#pragma unroll
            for (int r = 0; r < TK_ROUNDS; ++r) x[r] = ld_stream(src + r * TK_THREADS + tid);
#pragma unroll
            for (int r = 0; r < TK_ROUNDS; ++r) {
                cm[r] = 0;
#pragma unroll
                for (int c = 0; c < V; ++c) {
                    const T e = VT::get(x[r], c);
                    v[r][c] = e;
                    const K key = KO::key(e);
                    mx = key > mx ? key : mx;
                    cm[r] |= (key >= est ? 1u : 0u) << c;
                    ss = fma((double)e, (double)e, ss);
                }
            }
        } else {
#pragma unroll
            for (int r = 0; r < TK_ROUNDS; ++r) {
                cm[r] = 0;
#pragma unroll
                for (int c = 0; c < V; ++c) {
                    const long long e = base + (long long)(r * TK_THREADS + tid) * V + c;
                    const bool ok = e < a.dim;
                    const T x = ok ? row[e] : (T)0;
                    v[r][c] = x;
                    const K key = KO::key(x);
                    if (ok) {
                        mx = key > mx ? key : mx;
                        ss = fma((double)x, (double)x, ss);
                    }
                    cm[r] |= (ok && key >= est ? 1u : 0u) << c;
                }
            }
        }
        unsigned lp[TK_ROUNDS];
#pragma unroll
        for (int r = 0; r < TK_ROUNDS; ++r) {
            unsigned tot;
            warp_scan_small(__popc(cm[r]), lp[r], tot);
            if (lane == 0) s_wtot[r * TK_NW + warp] = tot;
        }
        ss = warp_sum(ss);
        mx = warp_max<K>(mx);
        if (lane == 0) {
            s_wsum[warp] = ss;
            s_wmax[warp] = mx;
        }
        __syncthreads();
        if (warp == 0) {
            const unsigned x = s_wtot[lane];
            unsigned incl = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += y;
            }
            s_woff[lane] = incl - x;
            const unsigned tot = __shfl_sync(FULL, incl, 31);
            const unsigned long long pre = lookback(a.status + (long long)w * a.ntiles, tile, tot);
            if (lane == 0) {
                s_base = pre;
                double tsum = 0.0;
                K tmax = 0;
                for (int i = 0; i < TK_NW; ++i) {
                    tsum = dadd(tsum, s_wsum[i]);
                    tmax = s_wmax[i] > tmax ? s_wmax[i] : tmax;
                }
                a.sumsq[(long long)w * a.ntiles + tile] = tsum;
                if (tmax > s_blkmax[w]) s_blkmax[w] = tmax;
                if (tile == a.ntiles - 1) a.count[w] = pre + tot;
            }
        }
        __syncthreads();
        const unsigned long long b = s_base;
        uint32_t* cidx = a.cidx + (long long)w * a.cap;
        T* cval = a.cval + (long long)w * a.cap;
#pragma unroll
        for (int r = 0; r < TK_ROUNDS; ++r) {
            if (!cm[r]) continue;
            unsigned long long pos = b + s_woff[r * TK_NW + warp] + lp[r];
#pragma unroll
            for (int c = 0; c < V; ++c) {
                if ((cm[r] >> c) & 1u) {
                    if (pos < (unsigned long long)a.cap) {
                        cidx[pos] = (uint32_t)(base + (long long)(r * TK_THREADS + tid) * V + c);
                        cval[pos] = v[r][c];
                    }
                    ++pos;
                }
            }
        }
    }
    __syncthreads();
    for (int i = tid; i < a.k; i += TK_THREADS)
        if (s_blkmax[i]) atomicMax(a.maxkey + i, s_blkmax[i]);
}

// --------------------------------------------------------------------------------------
// k_select: one radix-select round.  grid = (blocks_per_worker, k).
// --------------------------------------------------------------------------------------
template <typename T> struct SelArgs {
    const T* g;
    long long ld, dim, cap, m;
    const T* cval;
    const unsigned long long* count;
    const typename KeyOf<T>::K* est;
    const typename KeyOf<T>::K* maxkey;
    SelState<typename KeyOf<T>::K>* sel;
    unsigned* hist;   // [k][ROUNDS_MAX][SEL_BINS]
    unsigned* done;   // [k][ROUNDS_MAX]
};

template <typename T> SG_DEV SelState<typename KeyOf<T>::K> initial_state(const SelArgs<T>& a, int w) {
    using K = typename KeyOf<T>::K;
    SelState<K> s;
    const unsigned long long c = a.count[w];
    const K mk = a.maxkey[w];
    const bool cand = c >= (unsigned long long)a.m && c <= (unsigned long long)a.cap;
    s.mode = cand ? MODE_CAND : MODE_FULL;
    s.n_src = cand ? c : (unsigned long long)a.dim;
    s.lo = cand ? a.est[w] : (K)0;
    s.span = mk >= s.lo ? mk - s.lo : (K)0;
    s.shift = digit_shift<K>(s.span);
    s.rank = (unsigned long long)a.m;
    s.gt = 0;
    s.T = 0;
    s.done = 0;
    s.error = 0;
    return s;
}

template <typename T>
__global__ void __launch_bounds__(256)
k_select(SelArgs<T> a, int round) {
    using KO = KeyOf<T>;
    using K = typename KO::K;
    __shared__ unsigned hist[SEL_BINS];
    __shared__ SelState<K> st;
    __shared__ int s_last;
    const int w = blockIdx.y, tid = threadIdx.x;
    if (tid == 0) st = round == 0 ? initial_state<T>(a, w) : a.sel[w];
    for (int i = tid; i < SEL_BINS; i += 256) hist[i] = 0;
    __syncthreads();
    if (st.done) return;
    const K lo = st.lo, span = st.span;
    const int shift = st.shift;
    const long long n = (long long)st.n_src;
    const T* src = st.mode == MODE_CAND ? a.cval + (long long)w * a.cap : a.g + (long long)w * a.ld;
    for (long long i = (long long)blockIdx.x * 256 + tid; i < n; i += (long long)gridDim.x * 256) {
        const K key = KO::key(src[i]);
        if (key >= lo && key - lo <= span) atomicAdd(&hist[(unsigned)((key - lo) >> shift)], 1u);
    }
    __syncthreads();
    unsigned* gh = a.hist + ((long long)w * TopkTraits<T>::ROUNDS_MAX + round) * SEL_BINS;
    for (int i = tid; i < SEL_BINS; i += 256)
        if (hist[i]) atomicAdd(gh + i, hist[i]);
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        const unsigned prev = atomicAdd(a.done + w * TopkTraits<T>::ROUNDS_MAX + round, 1u);
        s_last = prev == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int i = tid; i < SEL_BINS; i += 256) hist[i] = __ldcg(gh + i);
    __syncthreads();
    if (tid < 32) {
        int bin;
        unsigned long long above;
        find_bin_from_top(hist, st.rank, bin, above);
        if (tid == 0) {
            SelState<K> s = st;
            advance<K>(s, bin, above);
            a.sel[w] = s;
        }
    }
}

// --------------------------------------------------------------------------------------
// k_final: stable compaction of the kept set into idx/val (ascending index order).
// --------------------------------------------------------------------------------------
template <typename T> struct FinArgs {
    const T* g;
    long long ld, dim, cap, m, nt_fin;
    int k, vec_ok;
    const uint32_t* cidx;
    const T* cval;
    const SelState<typename KeyOf<T>::K>* sel;
    unsigned long long* status;
    unsigned* ticket;
    uint32_t* idx;
    T* val;
    double* sumsq;
};

constexpr unsigned long long CNT_BITS = 31;
constexpr unsigned long long CNT_MASK = (1ull << CNT_BITS) - 1;

template <typename T>
__global__ void __launch_bounds__(TK_THREADS)
k_final(FinArgs<T> a) {
    using KO = KeyOf<T>;
    using K = typename KO::K;
    using VT = Vec16<T>;
    constexpr int V = VT::N;
    constexpr int TILE = tile_elems<T>();
    __shared__ long long s_tstart[MAX_WORKERS + 1];
    __shared__ K s_T[MAX_WORKERS];
    __shared__ unsigned long long s_need[MAX_WORKERS];
    __shared__ long long s_n[MAX_WORKERS];
    __shared__ int s_mode[MAX_WORKERS];
    __shared__ unsigned s_ticket;
    __shared__ unsigned s_gtot[32], s_etot[32], s_goff[32], s_eoff[32];
    __shared__ double s_wsum[TK_NW];
    __shared__ unsigned long long s_gb, s_eb;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        long long acc = 0;
        for (int w = 0; w < a.k; ++w) {
            const SelState<K> s = a.sel[w];
            s_tstart[w] = acc;
            s_T[w] = s.T;
            s_need[w] = s.rank;
            s_n[w] = (long long)s.n_src;
            s_mode[w] = s.mode;
            acc += ((long long)s.n_src + TILE - 1) / TILE;
        }
        s_tstart[a.k] = acc;
    }
    __syncthreads();
    const long long total = s_tstart[a.k];
    for (;;) {
        if (tid == 0) s_ticket = atomicAdd(a.ticket, 1u);
        __syncthreads();
        const long long t = s_ticket;
        if (t >= total) break;
        int w = 0;
        while (s_tstart[w + 1] <= t) ++w;
        const long long tile = t - s_tstart[w];
        const long long n = s_n[w];
        const long long base = tile * TILE;
        const K T_ = s_T[w];
        const unsigned long long need = s_need[w];
        const bool cand = s_mode[w] == MODE_CAND;
        const T* vsrc = cand ? a.cval + (long long)w * a.cap : a.g + (long long)w * a.ld;
        const uint32_t* isrc = a.cidx + (long long)w * a.cap;

        T v[TK_ROUNDS][V];
        uint32_t ix[TK_ROUNDS][V];
        unsigned gm[TK_ROUNDS], em[TK_ROUNDS];
        const bool vec = base + TILE <= n && (cand || a.vec_ok);
        if (vec) {
            typename VT::V x[TK_ROUNDS];
            typename VT::I xi[TK_ROUNDS];
            const typename VT::V* s = reinterpret_cast<const typename VT::V*>(vsrc + base);
#pragma unroll
            for (int r = 0; r < TK_ROUNDS; ++r) x[r] = ld_stream(s + r * TK_THREADS + tid);
            if (cand) {
                const typename VT::I* si = reinterpret_cast<const typename VT::I*>(isrc + base);
#pragma unroll
                for (int r = 0; r < TK_ROUNDS; ++r) xi[r] = ld_stream(si + r * TK_THREADS + tid);
            }
#pragma unroll
            for (int r = 0; r < TK_ROUNDS; ++r) {
                gm[r] = em[r] = 0;
#pragma unroll
                for (int c = 0; c < V; ++c) {
                    const T e = VT::get(x[r], c);
                    v[r][c] = e;
                    uint32_t id;
                    if (cand) {
                        if constexpr (V == 4) id = c == 0 ? xi[r].x : c == 1 ? xi[r].y : c == 2 ? xi[r].z : xi[r].w;
                        else id = c == 0 ? xi[r].x : xi[r].y;
                    } else {
                        id = (uint32_t)(base + (long long)(r * TK_THREADS + tid) * V + c);
                    }
                    ix[r][c] = id;
                    const K key = KO::key(e);
                    gm[r] |= (key > T_ ? 1u : 0u) << c;
                    em[r] |= (key == T_ ? 1u : 0u) << c;
                }
            }
        } else {
#pragma unroll
            for (int r = 0; r < TK_ROUNDS; ++r) {
                gm[r] = em[r] = 0;
#pragma unroll
                for (int c = 0; c < V; ++c) {
                    const long long e = base + (long long)(r * TK_THREADS + tid) * V + c;
                    const bool ok = e < n;
                    const T x = ok ? vsrc[e] : (T)0;
                    v[r][c] = x;
                    ix[r][c] = ok ? (cand ? isrc[e] : (uint32_t)e) : 0u;
                    const K key = KO::key(x);
                    gm[r] |= (ok && key > T_ ? 1u : 0u) << c;
                    em[r] |= (ok && key == T_ ? 1u : 0u) << c;
                }
            }
        }
        unsigned lg[TK_ROUNDS], le[TK_ROUNDS];
#pragma unroll
        for (int r = 0; r < TK_ROUNDS; ++r) {
            unsigned tg, te;
            warp_scan_small(__popc(gm[r]), lg[r], tg);
            warp_scan_small(__popc(em[r]), le[r], te);
            if (lane == 0) {
                s_gtot[r * TK_NW + warp] = tg;
                s_etot[r * TK_NW + warp] = te;
            }
        }
        __syncthreads();
        if (warp == 0) {
            const unsigned xg = s_gtot[lane], xe = s_etot[lane];
            unsigned ig = xg, ie = xe;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned yg = __shfl_up_sync(FULL, ig, o);
                const unsigned ye = __shfl_up_sync(FULL, ie, o);
                if (lane >= o) {
                    ig += yg;
                    ie += ye;
                }
            }
            s_goff[lane] = ig - xg;
            s_eoff[lane] = ie - xe;
            const unsigned long long tg = __shfl_sync(FULL, ig, 31), te = __shfl_sync(FULL, ie, 31);
            const unsigned long long pre =
                lookback(a.status + (long long)w * a.nt_fin, tile, (tg << CNT_BITS) | te);
            if (lane == 0) {
                s_gb = pre >> CNT_BITS;
                s_eb = pre & CNT_MASK;
            }
        }
        __syncthreads();
        const unsigned long long gb = s_gb, eb = s_eb;
        uint32_t* oi = a.idx + (long long)w * a.m;
        T* ov = a.val + (long long)w * a.m;
        double ss = 0.0;
#pragma unroll
        for (int r = 0; r < TK_ROUNDS; ++r) {
            unsigned long long g0 = gb + s_goff[r * TK_NW + warp] + lg[r];
            unsigned long long e0 = eb + s_eoff[r * TK_NW + warp] + le[r];
#pragma unroll
            for (int c = 0; c < V; ++c) {
                const bool isg = (gm[r] >> c) & 1u, ise = (em[r] >> c) & 1u;
                bool keep = false;
                unsigned long long pos = 0;
                if (isg) {
                    keep = true;
                    pos = g0 + (e0 < need ? e0 : need);
                } else if (ise && e0 < need) {
                    keep = true;
                    pos = g0 + e0;
                }
                if (keep && pos < (unsigned long long)a.m) {
                    oi[pos] = ix[r][c];
                    ov[pos] = v[r][c];
                    ss = fma((double)v[r][c], (double)v[r][c], ss);
                }
                g0 += isg;
                e0 += ise;
            }
        }
        ss = warp_sum(ss);
        if (lane == 0) s_wsum[warp] = ss;
        __syncthreads();
        if (tid == 0) {
            double tsum = 0.0;
            for (int i = 0; i < TK_NW; ++i) tsum = dadd(tsum, s_wsum[i]);
            a.sumsq[(long long)w * a.nt_fin + tile] = tsum;
        }
    }
}

// --------------------------------------------------------------------------------------
// Gate: EWMA update and decision exactly as comm.py:143-159.
// --------------------------------------------------------------------------------------
SG_DEV void gate_math(sg_gate_state& s, double s_full, double s_topk, uint8_t& dec, double& rho) {
    if (!s.initialized) {
        s.ewma_full = s_full;
        s.ewma_topk = s_topk;
        s.initialized = 1;
    } else {
        const double f = s.ewma_factor;
        const double one_m_f = dsub(1.0, f);
        s.ewma_full = dadd(dmul(f, s.ewma_full), dmul(one_m_f, s_full));
        s.ewma_topk = dadd(dmul(f, s.ewma_topk), dmul(one_m_f, s_topk));
    }
    const double full = s.raw_gate ? s_full : s.ewma_full;
    const double kept = s.raw_gate ? s_topk : s.ewma_topk;
    const double r = full == 0.0 ? 0.0 : ddiv(fabs(dsub(full, kept)), full);
    const bool compressed = r <= s.delta;  // NaN compares false -> dense, as in numpy
    if (compressed) s.n_compressed += 1;
    else s.n_uncompressed += 1;
    dec = compressed ? 1 : 0;
    rho = r;
}

SG_DEV double block_sum_fixed(const double* p, long long n, double* red) {
    const int tid = threadIdx.x;
    double acc = 0.0;
    for (long long i = tid; i < n; i += 256) acc = dadd(acc, p[i]);
    red[tid] = acc;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (tid < s) red[tid] = dadd(red[tid], red[tid + s]);
        __syncthreads();
    }
    const double r = red[0];
    __syncthreads();
    return r;
}

template <typename T>
__global__ void __launch_bounds__(256)
k_gate(const double* sum_main, long long nt_main, const double* sum_fin, long long nt_fin,
       const SelState<typename KeyOf<T>::K>* sel, double* norms2, sg_gate_state* states,
       uint8_t* decision, double* rho) {
    __shared__ double red[256];
    constexpr int TILE = tile_elems<T>();
    const int w = blockIdx.x;
    const double s_full = block_sum_fixed(sum_main + (long long)w * nt_main, nt_main, red);
    const long long nft = ((long long)sel[w].n_src + TILE - 1) / TILE;
    const double s_topk = block_sum_fixed(sum_fin + (long long)w * nt_fin, nft, red);
    if (threadIdx.x == 0) {
        norms2[2 * w] = s_full;
        norms2[2 * w + 1] = s_topk;
        if (states) {
            sg_gate_state s = states[w];
            uint8_t d;
            double r;
            gate_math(s, s_full, s_topk, d, r);
            states[w] = s;
            if (decision) decision[w] = d;
            if (rho) rho[w] = r;
        }
    }
}

__global__ void k_gate_update(const double* norms2, int k, sg_gate_state* states, uint8_t* decision,
                              double* rho) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= k) return;
    sg_gate_state s = states[w];
    uint8_t d;
    double r;
    gate_math(s, norms2[2 * w], norms2[2 * w + 1], d, r);
    states[w] = s;
    if (decision) decision[w] = d;
    if (rho) rho[w] = r;
}

// --------------------------------------------------------------------------------------
// Host launcher.
// --------------------------------------------------------------------------------------
template <typename T>
int topk_gate(const T* g, int k, long long ld, long long dim, long long m, uint32_t* idx, T* val,
              double* norms2, sg_gate_state* states, uint8_t* decision, double* rho, void* ws,
              size_t ws_bytes, cudaStream_t stream) {
    using K = typename KeyOf<T>::K;
    if (!g || !idx || !val || !norms2 || k < 1 || dim < 1 || m < 1 || m > dim || ld < dim)
        return SG_ERR_INVALID;
    if (k > MAX_WORKERS || dim >= (1ll << 31)) return SG_ERR_UNSUPPORTED;
    const TopkPlan p = make_plan<T>(k, dim, m);
    if (!ws || ws_bytes < p.total) return SG_ERR_WORKSPACE;
    unsigned char* base = reinterpret_cast<unsigned char*>(align_up(reinterpret_cast<size_t>(ws), 256));
    auto at = [&](size_t off) { return base + off; };
    unsigned long long* st_main = reinterpret_cast<unsigned long long*>(at(p.off_status_main));
    unsigned long long* st_fin = reinterpret_cast<unsigned long long*>(at(p.off_status_fin));
    unsigned* hist = reinterpret_cast<unsigned*>(at(p.off_hist));
    unsigned* ctr = reinterpret_cast<unsigned*>(at(p.off_ctr));
    unsigned long long* count = reinterpret_cast<unsigned long long*>(at(p.off_count));
    K* maxkey = reinterpret_cast<K*>(at(p.off_maxkey));
    K* est = reinterpret_cast<K*>(at(p.off_est));
    SelState<K>* sel = reinterpret_cast<SelState<K>*>(at(p.off_sel));
    double* sum_main = reinterpret_cast<double*>(at(p.off_sum_main));
    double* sum_fin = reinterpret_cast<double*>(at(p.off_sum_fin));
    uint32_t* cidx = reinterpret_cast<uint32_t*>(at(p.off_cidx));
    T* cval = reinterpret_cast<T*>(at(p.off_cval));

    const bool vec_ok = (reinterpret_cast<size_t>(g) % 16 == 0) && ((ld * (long long)sizeof(T)) % 16 == 0);
    const int sms = num_sms();

    // 1. estimate (+ zero the scratch)
    const size_t est_smem = sizeof(K) * (size_t)TopkTraits<T>::SAMPLE;
    cudaFuncSetAttribute(k_estimate<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)est_smem);
    k_estimate<T><<<k, EST_THREADS, est_smem, stream>>>(g, ld, p.s_eff, p.stride, p.r_est, est,
                                                         reinterpret_cast<uint4*>(base),
                                                         (long long)(p.zero_end / 16));
    // 2. main streaming pass
    MainArgs<T> ma;
    ma.g = g;
    ma.ld = ld;
    ma.dim = dim;
    ma.ntiles = p.nt_main;
    ma.cap = p.cap;
    ma.k = k;
    ma.vec_ok = vec_ok;
    ma.est = est;
    ma.cidx = cidx;
    ma.cval = cval;
    ma.status = st_main;
    ma.ticket = ctr;
    ma.sumsq = sum_main;
    ma.count = count;
    ma.maxkey = maxkey;
    long long tiles = (long long)k * p.nt_main;
    long long grid_main = (long long)sms * 8;
    if (grid_main > tiles) grid_main = tiles;
    k_main<T><<<(unsigned)grid_main, TK_THREADS, 0, stream>>>(ma);
    // 3. select rounds
    SelArgs<T> sa;
    sa.g = g;
    sa.ld = ld;
    sa.dim = dim;
    sa.cap = p.cap;
    sa.m = m;
    sa.cval = cval;
    sa.count = count;
    sa.est = est;
    sa.maxkey = maxkey;
    sa.sel = sel;
    sa.hist = hist;
    sa.done = ctr + 2;
    long long per_worker = (long long)sms * 4 / k;
    if (per_worker < 8) per_worker = 8;
    const long long need_blocks = (p.cap + 256 * 16 - 1) / (256 * 16);
    if (per_worker > need_blocks) per_worker = need_blocks < 8 ? 8 : need_blocks;
    dim3 sgrid((unsigned)per_worker, (unsigned)k);
    for (int r = 0; r < TopkTraits<T>::ROUNDS_MAX; ++r) k_select<T><<<sgrid, 256, 0, stream>>>(sa, r);
    // 4. final compaction
    FinArgs<T> fa;
    fa.g = g;
    fa.ld = ld;
    fa.dim = dim;
    fa.cap = p.cap;
    fa.m = m;
    fa.nt_fin = p.nt_fin;
    fa.k = k;
    fa.vec_ok = vec_ok;
    fa.cidx = cidx;
    fa.cval = cval;
    fa.sel = sel;
    fa.status = st_fin;
    fa.ticket = ctr + 1;
    fa.idx = idx;
    fa.val = val;
    fa.sumsq = sum_fin;
    long long grid_fin = (long long)sms * 8;
    const long long fin_need = (long long)k * ((p.cap + tile_elems<T>() - 1) / tile_elems<T>());
    if (grid_fin > fin_need) grid_fin = fin_need > 0 ? fin_need : 1;
    k_final<T><<<(unsigned)grid_fin, TK_THREADS, 0, stream>>>(fa);
    // 5. norms + gate
    k_gate<T><<<k, 256, 0, stream>>>(sum_main, p.nt_main, sum_fin, p.nt_fin, sel, norms2, states,
                                     decision, rho);
    return cudaGetLastError() == cudaSuccess ? SG_OK : SG_ERR_CUDA;
}

}  // namespace sg

using namespace sg;

extern "C" {

size_t sg_topk_workspace_bytes_f32(int k, int64_t dim, int64_t m) {
    if (k < 1 || dim < 1 || m < 1 || m > dim) return 0;
    return make_plan<float>(k, dim, m).total;
}
size_t sg_topk_workspace_bytes_f64(int k, int64_t dim, int64_t m) {
    if (k < 1 || dim < 1 || m < 1 || m > dim) return 0;
    return make_plan<double>(k, dim, m).total;
}

int sg_topk_gate_f32(const float* g, int k, int64_t ld, int64_t dim, int64_t m, uint32_t* idx,
                     float* val, double* norms2, sg_gate_state* states, uint8_t* decision,
                     double* rho, void* workspace, size_t workspace_bytes, void* stream) {
    return topk_gate<float>(g, k, ld, dim, m, idx, val, norms2, states, decision, rho, workspace,
                            workspace_bytes, (cudaStream_t)stream);
}
int sg_topk_gate_f64(const double* g, int k, int64_t ld, int64_t dim, int64_t m, uint32_t* idx,
                     double* val, double* norms2, sg_gate_state* states, uint8_t* decision,
                     double* rho, void* workspace, size_t workspace_bytes, void* stream) {
    return topk_gate<double>(g, k, ld, dim, m, idx, val, norms2, states, decision, rho, workspace,
                             workspace_bytes, (cudaStream_t)stream);
}

int sg_gate_update(const double* norms2, int k, sg_gate_state* states, uint8_t* decision,
                   double* rho, void* stream) {
    if (!norms2 || !states || k < 1) return SG_ERR_INVALID;
    k_gate_update<<<(k + 63) / 64, 64, 0, (cudaStream_t)stream>>>(norms2, k, states, decision, rho);
    return cudaGetLastError() == cudaSuccess ? SG_OK : SG_ERR_CUDA;
}

}  // extern "C"
