// Top-k sparsification + squared norms + adaptive compression gate (items 3 and 4).
//
// Replaces reference pkg/src/streamsgd/comm.py:90-96 (topk_sparsify: np.lexsort on -|g| with
// the index as tie-break, first m re-sorted ascending) and comm.py:129-160
// (compression_gate: s_full = g.g, s_topk = v.v, EWMA, rho, decision) for the k workers of
// one GPU in one launch sequence, with no host synchronisation.
//
//   k_estimate  one CTA per worker: zero the call's small scratch, read a stratified random
//               sample of S keys and radix-select its r_est-th largest -> `est`, below the
//               true m-th largest key with probability ~1 - 1e-9.
//   k_main      THE full read of the bucket (4 B/element).  grid = (B, k); CTA b owns a
//               contiguous range of 16 KB tiles ("segment") and walks it with the next
//               tile's 128-bit loads in flight, accumulating the fp64 sum of squares and
//               appending every element with key >= est to the segment's candidate list
//               (global index + value, ascending).  No inter-CTA dependency, so the pass
//               streams at HBM bandwidth; the candidate lists are ~1.2-2 m entries in total
//               and stay L2-resident.  It also builds the round-0 radix histogram of the
//               candidate keys (1024 bins over [est, sample max], top bin open-ended); the
//               last CTA of each worker finds the bin holding rank m.
//   k_main(fb)  only if fewer than m keys reached `est` (estimate undershot): the same pass
//               with est = 0.  Early-exits otherwise.
//   k_collect   one CTA per segment: counts the segment's candidates above the rank-m bin
//               and appends those inside it (key, index) to a boundary buffer.  Its last CTA
//               finishes the select in shared memory (T, the m-th largest key), resolves ties
//               at T by index (the first `need` indices among keys == T are kept), counts the
//               kept elements per segment and scans them into per-segment output bases.
//   k_resolve   only for oversized boundary sets (heavy ties): multi-CTA radix rounds.
//   k_write     one CTA per segment: kept = key > T or (key == T and idx <= idx_cut); an
//               in-CTA ordered scan places them at the segment's base -> idx/val ascending,
//               plus the fp64 sum of kept squares and the per-4096-element merge offsets.
//               (Oversized-tie mode: a decoupled look-back over segments with the exact
//               tie rank instead.)  Its last CTA reduces the norms in a fixed order and
//               applies the gate in IEEE round-to-nearest (comm.py:143-159 operation order).
#include "common.cuh"

namespace sg {

constexpr int TK_THREADS = 256;
constexpr int TK_ROUNDS = 4;  // 16-byte vectors per thread per tile
constexpr int TK_NW = TK_THREADS / 32;
static_assert(TK_ROUNDS * TK_NW == 32, "one warp scans the per-(round, warp) totals");
constexpr int H0_BITS = 12;
constexpr int H0_BINS = 1 << H0_BITS;
constexpr int SEL_BITS = 11;
constexpr int SEL_BINS = 1 << SEL_BITS;
constexpr int EST_THREADS = 1024;
constexpr int EST_G = 32;        // sampling CTAs per worker (k_sample)
constexpr int SE_GMAX = 128;     // sampling CTAs per worker (k_sample_est), at most
constexpr int BMAX = 1024;  // max segments (k_main CTAs) per worker
constexpr int MERGE_TILE = 4096;
constexpr int NSUB_MAX = 2048;      // collect/write sub-ranges per worker
constexpr int CW_PER_SM = 6;        // resident collect/write CTAs per SM (one wave)
constexpr int FB_CTAS = 32;         // fallback-pass CTAs per worker (striding over the segments)

enum { MODE_NORMAL = 0, MODE_FALLBACK = 1 };
enum { WR_FAST = 0, WR_SLOW = 1 };

template <typename T> struct TopkTraits;
template <> struct TopkTraits<float> {
    static constexpr int SAMPLE = 131072;
    static constexpr double Z = 4.0;      // sigmas of binomial slack (undershoot ~3e-5 per call)
    static constexpr int ROUNDS_MAX = 3;  // after round 0: <= 31 bits left (open top bin)
    static constexpr int RES = 15360;     // boundary entries resolved inside one CTA
};
template <> struct TopkTraits<double> {
    static constexpr int SAMPLE = 8192;
    static constexpr double Z = 6.0;
    static constexpr int ROUNDS_MAX = 6;  // after round 0: <= 63 bits left (open top bin)
    static constexpr int RES = 8192;
};

template <typename T> constexpr int tile_elems() { return TK_THREADS * TK_ROUNDS * Vec16<T>::N; }

template <typename K> struct SelState {
    K est, smax;               // from the estimate: smax bounds the round-0 histogram's fine range
    K lo, span;                // current key range [lo, lo + span]
    K T;                       // final threshold key
    unsigned long long rank;   // remaining 1-based rank from the top inside the range
    unsigned long long h;      // keys inside the range
    unsigned idx_cut;          // keys == T are kept iff index <= idx_cut (fast mode)
    int shift0, shift;         // round-0 / current digit shift
    int done;
    int mode;                  // MODE_NORMAL / MODE_FALLBACK
    int wmode;                 // WR_FAST / WR_SLOW
};

// --------------------------------------------------------------------------------------
// Host-side plan of the caller workspace.
// --------------------------------------------------------------------------------------
struct TopkPlan {
    int k, nseg, tps;  // segments per worker, tiles per segment
    int split, nsub;   // (unused) / collect-write grid per worker (>= Σ parts)
    int nsubt;         // target sub-range count apportioned over the segments by candidates
    long long dim, m;
    long long s_eff, stride, r_est;
    long long r_hi;  // float32 sample: rank whose level-1 bin bounds the main pass's fine histogram (0: none)
    long long ntiles, segcap;
    size_t off_se_h1, off_se_mm, off_se_done, state_end;  // zero state between calls (k_sample_est)
    size_t zero_begin, off_count, off_maxkey, off_ctr, off_bndn, off_hist0, off_hist0fb, off_histr, off_status, zero_end;
    size_t off_boff;
    size_t off_sel, off_samp, off_mm, off_cnt, off_tstart, off_segcnt, off_seggt, off_segbase, off_pmain, off_pwrite,
        off_cidx, off_cval, off_bkey, off_bidx, off_bpos, off_pp, off_submap, off_hs1, total;
};

template <typename T> TopkPlan make_plan(int k, long long dim, long long m, int segs_per_worker, long long cta_target) {
    using K = typename KeyOf<T>::K;
    TopkPlan p{};
    p.k = k;
    p.dim = dim;
    p.m = m;
    // sample: 131072 keys (f32) with 4 sigma slack keep C = count(key >= est) near m (C/m
    // ~1.04 at cr 0.1, ~1.1 at cr 0.01), which matters most on real gradients, whose kept
    // entries crowd into a few layers
    long long S = TopkTraits<T>::SAMPLE;  // a multiple of CHUNK
    p.s_eff = dim <= S ? dim : S;
    p.stride = dim / p.s_eff;
    if (p.s_eff == dim) {
        p.r_est = m;  // exact sample: est is the true m-th largest key
    } else {
        // count(key >= est) < m needs a 6-sigma binomial deviation of the sample (~1e-9).
        const double q = (double)m / (double)dim;
        const double mean = q * (double)p.s_eff;
        const double sd = __builtin_sqrt(mean * (1.0 - q) + 1.0);
        const double z = S == TopkTraits<T>::SAMPLE ? TopkTraits<T>::Z : 6.0;
        p.r_est = (long long)(mean + z * sd + 4.0) + 1;
        // the mirror bound: fewer than m keys lie above the r_hi-th largest sample key's level-1
        // bin (same odds), so the round-0 histogram of the candidates spans [est, that bin's
        // top] instead of [est, sample max] -- ~32x finer bins, a boundary bin far below RES
        const double r_hi = mean - z * sd - 4.0;
        p.r_hi = r_hi >= 1.0 ? (long long)r_hi : 0;
    }
    const long long te = tile_elems<T>();
    p.ntiles = (dim + te - 1) / te;
    long long segs = segs_per_worker < 1 ? 1 : segs_per_worker;
    if (segs > BMAX) segs = BMAX;
    if (segs > p.ntiles) segs = p.ntiles;
    p.tps = (int)((p.ntiles + segs - 1) / segs);
    p.nseg = (int)((p.ntiles + p.tps - 1) / p.tps);
    p.segcap = (long long)p.tps * te;
    {
        // collect/write: about one wave of CTAs (cta_target) over all sub-ranges, each CTA
        // streaming its sub-range with the next chunk's loads in flight
        // sub-ranges are apportioned to segments by candidate count on the device (adaptive
        // split: concentrated real gradients put most candidates in a few segments), so the
        // grid is the target plus one per segment (every segment gets at least one)
        // grid = one wave of CTAs per worker (cta_target / k, at least one per segment); the
        // apportioned target leaves one guaranteed part per segment inside it
        long long grid = cta_target / k;
        if (grid > NSUB_MAX) grid = NSUB_MAX;
        if (grid < 2LL * p.nseg) grid = 2LL * p.nseg;
        if (grid > NSUB_MAX) grid = NSUB_MAX;
        p.nsub = (int)grid;
        p.nsubt = p.nsub - p.nseg > 0 ? p.nsub - p.nseg : 1;
        p.split = 0;
    }
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + bytes, 256); return r; };
    // zero state: restored by k_sample_est's last CTA per worker (float32 chain)
    p.off_se_h1 = take(sizeof(unsigned) * (size_t)k * SEL_BINS);
    p.off_se_mm = take(sizeof(unsigned) * 2 * (size_t)k);
    p.off_se_done = take(sizeof(unsigned) * (size_t)k);
    p.state_end = o;
    // per-call scratch zeroed by the first kernel of the chain
    p.zero_begin = o;
    p.off_count = take(sizeof(unsigned long long) * 2 * k);  // [pass][k]
    p.off_maxkey = take(sizeof(K) * k);
    p.off_ctr = take(sizeof(unsigned) * (8 + 16 * (size_t)k));  // see the counter map in topk_gate
    p.off_bndn = take(sizeof(unsigned long long) * k);
    p.off_hist0 = take(sizeof(unsigned) * (size_t)k * H0_BINS);
    p.off_hist0fb = take(sizeof(unsigned) * (size_t)k * H0_BINS);
    p.off_histr = take(sizeof(unsigned) * (size_t)k * TopkTraits<T>::ROUNDS_MAX * SEL_BINS);
    p.off_status = take(sizeof(unsigned long long) * (size_t)k * p.nsub);
    p.zero_end = o;
    p.off_sel = take(sizeof(SelState<K>) * k);
    p.off_samp = take(sizeof(K) * (size_t)k * TopkTraits<T>::SAMPLE);
    p.off_mm = take(sizeof(K) * (size_t)k * EST_G * 2);
    p.off_cnt = take(sizeof(unsigned) * (size_t)k * p.ntiles);
    p.off_tstart = take(sizeof(unsigned) * (size_t)k * p.ntiles);
    p.off_segcnt = take(sizeof(unsigned) * (size_t)k * p.nseg);
    p.off_seggt = take(sizeof(unsigned) * (size_t)k * p.nsub);
    p.off_segbase = take(sizeof(unsigned) * (size_t)k * p.nsub);
    p.off_pmain = take(sizeof(double) * (size_t)k * p.nseg);
    p.off_pwrite = take(sizeof(double) * (size_t)k * p.nsub);
    p.off_pp = take(sizeof(unsigned) * (size_t)k * (BMAX + 1));
    p.off_submap = take(sizeof(uint4) * (size_t)k * NSUB_MAX);
    const size_t cap = (size_t)k * p.nseg * p.segcap;
    p.off_cidx = take(sizeof(uint32_t) * cap);
    p.off_cval = take(sizeof(T) * cap);
    // boundary lists: only the in-CTA resolve reads them, so RES entries per worker; a larger
    // boundary is counted, not stored, and resolved from the candidate lists (slow mode)
    const size_t bcap = (size_t)k * TopkTraits<T>::RES;
    p.off_bkey = take(sizeof(K) * bcap);
    p.off_bidx = take(sizeof(uint32_t) * bcap);
    p.off_bpos = take(sizeof(uint32_t) * bcap);
    // float32 level-1 sample histograms (key bits [30:20]): one dense row per sampling CTA,
    // written whole by k_sample (no atomics, no state between calls), summed by k_estimate
    p.off_hs1 = take(sizeof(unsigned) * (size_t)k * EST_G * SEL_BINS);
    p.off_boff = take(sizeof(uint16_t) * (size_t)k * SE_GMAX * (SEL_BINS + 1));
    p.total = o + 256;  // slack for base alignment
    return p;
}

// A block's copy of PER * NT global words into shared memory with all PER loads of a thread in
// flight before the first store: a last-CTA tail reading a histogram one round trip per
// iteration cost ~0.7 us per iteration.
template <int PER, int NT, typename U>
SG_DEV void ld_cg_rows(U* dst, const U* src, int tid) {
    U v[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) v[u] = __ldcg(src + tid + u * NT);
#pragma unroll
    for (int u = 0; u < PER; ++u) dst[tid + u * NT] = v[u];
}

// --------------------------------------------------------------------------------------
// Radix-select helpers.
// --------------------------------------------------------------------------------------
// Warp-cooperative: locate the bin holding the rank-th largest element of an NB-bin
// histogram.  Lane L owns the PER bins ending at top_L = NB-1-PER*L; it reads them in a
// lane-rotated order so the 32 lanes never hit the same shared-memory bank.
template <int NB>
SG_DEV void find_bin_from_top(const unsigned* hist, unsigned long long rank, int& bin,
                              unsigned long long& above) {
    constexpr int PER = NB / 32;
    const int lane = threadIdx.x & 31;
    const int top = NB - 1 - PER * lane;
    unsigned long long s = 0;
    for (int i = 0; i < PER; ++i) s += hist[top - ((i + lane) & (PER - 1))];
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
        for (int i = 0; i < PER; ++i) {
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

// Block-cooperative version (every thread calls it; the result is broadcast): thread t owns
// the NB/THREADS bins below NB-1-(NB/THREADS)*t; one block scan of the per-thread sums from
// the top locates the bin, two barriers instead of a one-warp serial walk.
template <int NB, int THREADS>
SG_DEV void block_find_bin_from_top(const unsigned* hist, unsigned long long rank, int& bin,
                                    unsigned long long& above) {
    constexpr int PER = NB / THREADS;
    static_assert(PER >= 1 && NB % THREADS == 0, "bins per thread");
    __shared__ unsigned long long s_wsum[THREADS / 32];
    __shared__ int s_bin;
    __shared__ unsigned long long s_above;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int top = NB - 1 - PER * tid;
    unsigned long long s = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) s += hist[top - i];
    unsigned long long incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_wsum[warp] = incl;
    if (tid == 0) s_bin = -1;
    __syncthreads();
    unsigned long long wb = 0;
    for (int i = 0; i < warp; ++i) wb += s_wsum[i];
    incl += wb;
    const unsigned long long ex = incl - s;
    if (ex < rank && incl >= rank) {  // exactly one thread holds the rank
        unsigned long long cum = ex;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const unsigned h = hist[top - i];
            if (cum + h >= rank) {
                s_bin = top - i;
                s_above = cum;
                break;
            }
            cum += h;
        }
    }
    __syncthreads();
    bin = s_bin;
    above = s_above;
}

// Two ranks from one block scan (the estimate's r_est and its mirror r_hi); rank 0: none (-1).
template <int NB, int THREADS>
SG_DEV void block_find_two_bins_from_top(const unsigned* hist, unsigned long long r1, int& bin1, unsigned long long& above1,
                                         unsigned long long r2, int& bin2, unsigned long long& above2) {
    constexpr int PER = NB / THREADS;
    static_assert(PER >= 1 && NB % THREADS == 0, "bins per thread");
    __shared__ unsigned long long s_wsum2[THREADS / 32];
    __shared__ int s_b[2];
    __shared__ unsigned long long s_a[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int top = NB - 1 - PER * tid;
    unsigned long long s = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) s += hist[top - i];
    unsigned long long incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_wsum2[warp] = incl;
    if (tid == 0) s_b[0] = s_b[1] = -1;
    __syncthreads();
    unsigned long long wb = 0;
    for (int i = 0; i < warp; ++i) wb += s_wsum2[i];
    incl += wb;
    const unsigned long long ex = incl - s;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const unsigned long long rank = r == 0 ? r1 : r2;
        if (rank >= 1 && ex < rank && incl >= rank) {  // exactly one thread holds the rank
            unsigned long long cum = ex;
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                const unsigned h = hist[top - i];
                if (cum + h >= rank) {
                    s_b[r] = top - i;
                    s_a[r] = cum;
                    break;
                }
                cum += h;
            }
        }
    }
    __syncthreads();
    bin1 = s_b[0];
    above1 = s_a[0];
    bin2 = s_b[1];
    above2 = s_a[1];
}

template <typename K> SG_DEV int digit_shift(K span, int bits) {
    const int bl = bitlen<K>(span);
    return bl > bits ? bl - bits : 0;
}

// Digit of `key` in a range starting at lo with shift s and an open-ended top bin.
template <typename K> SG_DEV unsigned digit(K key, K lo, int shift, unsigned nb) {
    const K d = (key - lo) >> shift;
    return d >= (K)(nb - 1) ? nb - 1 : (unsigned)d;
}

// Narrow the state to bin `bin` of an nb-bin round whose top bin is open-ended.
template <typename K>
SG_DEV void narrow(SelState<K>& s, int bin, unsigned long long above, unsigned long long h,
                   unsigned nb, int next_bits) {
    const K off = (K)bin << s.shift;
    s.rank -= above;
    s.h = h;
    const K lo = s.lo + off;
    const K rest = s.span - off;
    K span = rest;
    if ((unsigned)bin != nb - 1) {
        const K width = ((K)1 << s.shift) - 1;
        span = rest < width ? rest : width;
    }
    s.lo = lo;
    s.span = span;
    if (span == 0) {
        s.T = lo;
        s.done = 1;
        return;
    }
    s.shift = digit_shift<K>(span, next_bits);
}

SG_DEV unsigned long long mix64(unsigned long long x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

// In-block radix select of the rank-th largest of n keys (shared memory) inside st's range.
template <typename K, int THREADS>
SG_DEV void block_select(const K* keys, long long n, SelState<K>& st, unsigned* hist) {
    const int tid = threadIdx.x;
    for (int round = 0; round < 8; ++round) {
        __syncthreads();
        if (st.done) break;
        for (int i = tid; i < SEL_BINS; i += THREADS) hist[i] = 0;
        __syncthreads();
        const K lo = st.lo, span = st.span;
        const int shift = st.shift;
        for (long long i = tid; i < n; i += THREADS) {
            const K key = keys[i];
            if (key >= lo && key - lo <= span) atomicAdd(&hist[digit<K>(key, lo, shift, SEL_BINS)], 1u);
        }
        __syncthreads();
        int bin;
        unsigned long long above;
        block_find_bin_from_top<SEL_BINS, THREADS>(hist, st.rank, bin, above);
        if (tid == 0) {
            if (bin < 0) {
                st.done = 1;  // inconsistent counts (cannot happen): keep the lowest key
                st.T = st.lo;
            } else {
                narrow<K>(st, bin, above, hist[bin], SEL_BINS, SEL_BITS);
            }
        }
    }
    __syncthreads();
}

// In-block: the r-th SMALLEST (1-based) of the u32 values v[i] with flag[i] set; three
// radix rounds (11, 11, 10 bits), each bin located by a warp scan from the top with the
// rank mirrored (r-th smallest of N = (N - r + 1)-th largest).
template <int THREADS>
SG_DEV unsigned block_select_small_u32(const unsigned* v, const uint8_t* flag, long long n,
                                       unsigned long long r, unsigned* hist, unsigned* s_res) {
    const int tid = threadIdx.x;
    unsigned lo = 0;
    unsigned long long rank = r;
    const int shifts[3] = {21, 10, 0};
    for (int round = 0; round < 3; ++round) {
        const int shift = shifts[round];
        const unsigned nb = round == 2 ? 1024u : 2048u;
        for (int i = tid; i < SEL_BINS; i += THREADS) hist[i] = 0;
        __syncthreads();
        for (long long i = tid; i < n; i += THREADS) {
            if (!flag[i]) continue;
            const unsigned x = v[i];
            if (x < lo) continue;
            const unsigned long long d = ((unsigned long long)(x - lo)) >> shift;
            if (d < nb) atomicAdd(&hist[d], 1u);
        }
        __syncthreads();
        if (tid < 32) {
            unsigned long long tot = 0;
            for (int i = tid; i < SEL_BINS; i += 32) tot += hist[i];
            for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(FULL, tot, o);
            int bin;
            unsigned long long above;
            find_bin_from_top<SEL_BINS>(hist, tot - rank + 1, bin, above);
            if (tid == 0) {
                const unsigned long long below = tot - above - hist[bin];
                s_res[0] = lo + ((unsigned)bin << shift);
                s_res[1] = (unsigned)(rank - below);
            }
        }
        __syncthreads();
        lo = s_res[0];
        rank = s_res[1];
        __syncthreads();
    }
    return lo;
}

// --------------------------------------------------------------------------------------
// Candidate threshold estimate.  The sample is S/32 randomly placed 32-element chunks (one
// per stratum of the row, so every warp load is one coalesced 128-byte line for f32).
// --------------------------------------------------------------------------------------
constexpr int CHUNK = 32;

// k_sample: EST_G CTAs per worker gather the sample in parallel (one random 32-element chunk
// per stratum; a warp's chunk loads all in flight) into the workspace, with per-CTA key
// ranges; they also clear the small scratch (incl. the slow-mode look-back words).
template <typename T>
__global__ void __launch_bounds__(256)
k_sample(const T* __restrict__ g, long long ld, long long dim, long long s_eff,
         typename KeyOf<T>::K* __restrict__ samp, typename KeyOf<T>::K* __restrict__ mm,
         uint4* __restrict__ zero, long long zero_vec, unsigned* __restrict__ hs1) {
    pdl_enter();
    using KO = KeyOf<T>;
    using K = typename KO::K;
    constexpr bool H1 = sizeof(K) == 4;  // float32: level-1 histogram of the sample here
    __shared__ K s_min[8], s_max[8];
    __shared__ __align__(16) unsigned s_h1[H1 ? SEL_BINS : 1];
    const int x = blockIdx.x, w = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if constexpr (H1) {
        for (int i = tid; i < SEL_BINS; i += 256) s_h1[i] = 0;
        __syncthreads();
    }
    const long long cta = (long long)w * gridDim.x + x;
    for (long long i = cta * 256 + tid; i < zero_vec; i += (long long)gridDim.x * gridDim.y * 256)
        zero[i] = make_uint4(0, 0, 0, 0);
    const T* row = g + (long long)w * ld;
    K* sk = samp + (long long)w * TopkTraits<T>::SAMPLE;
    K mn = KO::KMAX, mx = 0;
    if (s_eff == dim) {  // the sample is the whole row
        const long long slice = (dim + gridDim.x - 1) / gridDim.x;
        const long long lo = x * slice, hi = lo + slice < dim ? lo + slice : dim;
        for (long long i = lo + tid; i < hi; i += 256) {
            const K key = KO::key(row[i]);
            sk[i] = key;
            if constexpr (H1) atomicAdd(&s_h1[(unsigned)(key >> 20)], 1u);
            mn = key < mn ? key : mn;
            mx = key > mx ? key : mx;
        }
    } else {
        const long long nch = s_eff / CHUNK;
        const long long stratum = dim / nch;  // >= CHUNK because dim > s_eff
        const int gw = x * 8 + warp, nwarps = gridDim.x * 8;
        constexpr int BATCH = 8;
        for (long long c0 = gw; c0 < nch; c0 += (long long)nwarps * BATCH) {
            T v[BATCH];
#pragma unroll
            for (int u = 0; u < BATCH; ++u) {
                const long long c = c0 + (long long)u * nwarps;
                v[u] = (T)0;
                if (c < nch) {
                    const unsigned h = (unsigned)mix64((unsigned long long)c * 0x9e3779b97f4a7c15ull + (unsigned long long)w);
                    const long long off = (long long)(((unsigned long long)h * (unsigned long long)(stratum - CHUNK + 1)) >> 32);
                    v[u] = __ldg(row + c * stratum + off + lane);
                }
            }
#pragma unroll
            for (int u = 0; u < BATCH; ++u) {
                const long long c = c0 + (long long)u * nwarps;
                if (c < nch) {
                    const K key = KO::key(v[u]);
                    sk[c * CHUNK + lane] = key;
                    if constexpr (H1) atomicAdd(&s_h1[(unsigned)(key >> 20)], 1u);
                    mn = key < mn ? key : mn;
                    mx = key > mx ? key : mx;
                }
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const K a = __shfl_xor_sync(FULL, mn, o), b = __shfl_xor_sync(FULL, mx, o);
        mn = a < mn ? a : mn;
        mx = b > mx ? b : mx;
    }
    if (lane == 0) {
        s_min[warp] = mn;
        s_max[warp] = mx;
    }
    __syncthreads();
    if (tid == 0) {
        K a = KO::KMAX, b = 0;
        for (int i = 0; i < 8; ++i) {
            a = s_min[i] < a ? s_min[i] : a;
            b = s_max[i] > b ? s_max[i] : b;
        }
        mm[cta * 2] = a;
        mm[cta * 2 + 1] = b;
    }
    if constexpr (H1) {  // this CTA's row, written whole (coalesced 16-byte stores)
        uint4* gh = reinterpret_cast<uint4*>(hs1 + cta * SEL_BINS);
        const uint4* sh = reinterpret_cast<const uint4*>(s_h1);
        for (int i = tid; i < SEL_BINS / 4; i += 256) gh[i] = sh[i];
    }
}

// k_estimate: one CTA per worker; est = the lower edge of the 2048-bin histogram bin (over the
// sample's key range) that holds the r_est-th largest sample key -- never above that key, so
// count(key >= est) >= m keeps its ~1 - 1e-9 odds.  With dim <= S the "sample" is the whole
// row and est is a lower bound of the true T.
template <typename T>
__global__ void __launch_bounds__(EST_THREADS)
k_estimate(long long dim, long long s_eff, long long r_est, const typename KeyOf<T>::K* __restrict__ samp,
           const typename KeyOf<T>::K* __restrict__ mm, int G, SelState<typename KeyOf<T>::K>* __restrict__ sel,
           unsigned* __restrict__ hs1) {
    pdl_enter();
    using KO = KeyOf<T>;
    using K = typename KO::K;
    __shared__ unsigned hist[SEL_BINS];
    __shared__ K s_lo, s_span;
    __shared__ int s_shift;
    const int w = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < SEL_BINS; i += EST_THREADS) hist[i] = 0;
    if (warp == 0) {
        K a = KO::KMAX, b = 0;
        for (int i = lane; i < G; i += 32) {
            const K x = mm[((long long)w * G + i) * 2], y = mm[((long long)w * G + i) * 2 + 1];
            a = x < a ? x : a;
            b = y > b ? y : b;
        }
        for (int o = 16; o > 0; o >>= 1) {
            const K x = __shfl_xor_sync(FULL, a, o), y = __shfl_xor_sync(FULL, b, o);
            a = x < a ? x : a;
            b = y > b ? y : b;
        }
        if (lane == 0) {
            s_lo = a;
            s_span = b - a;
            s_shift = digit_shift<K>(b - a, SEL_BITS);
        }
    }
    __syncthreads();
    const K lo = s_lo;
    const int shift = s_shift;
    const long long ns = (s_eff / CHUNK) * CHUNK == s_eff || s_eff == dim ? s_eff : (s_eff / CHUNK) * CHUNK;
    const K* sk = samp + (long long)w * TopkTraits<T>::SAMPLE;
    K est = 0;
    if constexpr (sizeof(K) == 4) {
        // float32: two fixed-digit rounds -- the sampling CTAs already histogrammed key bits
        // [30:20] (level 1, no contended atomics here); level 2 (bits [19:9]) only over the
        // sample keys inside the chosen level-1 bin.  est is the 512-key bin edge at or below
        // the r_est-th largest sample key.
        (void)lo;
        (void)shift;
        const unsigned* gh = hs1 + (long long)w * G * SEL_BINS;
        for (int i = tid; i < SEL_BINS; i += EST_THREADS) {
            unsigned v = 0;
            for (int r = 0; r < G; ++r) v += __ldcg(gh + (long long)r * SEL_BINS + i);
            hist[i] = v;
        }
        __syncthreads();
        if (r_est <= ns) {
            int b1;
            unsigned long long a1;
            block_find_bin_from_top<SEL_BINS, EST_THREADS>(hist, (unsigned long long)r_est, b1, a1);
            if (b1 >= 0) {
                for (int i = tid; i < SEL_BINS; i += EST_THREADS) hist[i] = 0;
                __syncthreads();
                // level 2 over the keys of bin b1: 16-byte loads, several in flight
                const long long n4 = ns / 4;
                const uint4* s4 = reinterpret_cast<const uint4*>(sk);
                constexpr int U = 8;
                for (long long i0 = tid; i0 < n4; i0 += (long long)EST_THREADS * U) {
                    uint4 v[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const long long i = i0 + (long long)u * EST_THREADS;
                        v[u] = i < n4 ? __ldcg(s4 + i) : make_uint4(0u, 0u, 0u, 0u);
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        if (i0 + (long long)u * EST_THREADS >= n4) break;
                        const unsigned kk[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                        for (int c = 0; c < 4; ++c)
                            if ((int)(kk[c] >> 20) == b1) atomicAdd(&hist[(kk[c] >> 9) & (SEL_BINS - 1)], 1u);
                    }
                }
                for (long long i = n4 * 4 + tid; i < ns; i += EST_THREADS) {
                    const K key = sk[i];
                    if ((int)(key >> 20) == b1) atomicAdd(&hist[(key >> 9) & (SEL_BINS - 1)], 1u);
                }
                __syncthreads();
                int b2;
                unsigned long long a2;
                block_find_bin_from_top<SEL_BINS, EST_THREADS>(hist, (unsigned long long)r_est - a1, b2, a2);
                est = ((K)b1 << 20) | (b2 >= 0 ? ((K)b2 << 9) : (K)0);
            }
        }
    } else {
        if (r_est <= ns) {
            for (long long i = tid; i < ns; i += EST_THREADS) atomicAdd(&hist[digit<K>(sk[i], lo, shift, SEL_BINS)], 1u);
        }
        __syncthreads();
        if (r_est <= ns) {  // uniform
            int bin;
            unsigned long long above;
            block_find_bin_from_top<SEL_BINS, EST_THREADS>(hist, (unsigned long long)r_est, bin, above);
            est = bin < 0 ? (K)0 : lo + ((K)bin << shift);
        }
    }
    {
        if (tid == 0) {
            SelState<K> o{};
            o.smax = s_lo + s_span;
            o.est = est;
            o.shift0 = digit_shift<K>(o.smax > est ? o.smax - est : (K)0, H0_BITS);
            o.done = 0;
            o.mode = MODE_NORMAL;
            o.wmode = WR_FAST;
            o.idx_cut = 0xffffffffu;
            sel[w] = o;
        }
    }
}

// --------------------------------------------------------------------------------------
// k_sample_est (float32): sample + estimate in ONE launch, spread over many SMs.
// The sample: S = 131072 keys per worker as 512 chunks of 256 elements (1 KB, one DRAM row),
// one at a hashed offset inside each of 512 strata of the row.  The reads are random, so their
// cost is DRAM row activations (128-byte chunks, 8x the activations, measured 25 us at k = 8).
// G CTAs per worker (G = se_ctas(k): 64 at k = 1, 32 otherwise) each take 512/G chunks, key
// them in shared memory, histogram key bits [30:20] (level 1), add the non-zero bins to the
// worker's global level-1 histogram and write the keys BUCKETED by level-1 bin (a counting
// sort in shared memory) with the bucket offsets.  The worker's last CTA to finish picks the
// level-1 bin b1 holding the r_est-th largest sample key, reads only the keys of bin b1 from
// every CTA's bucket (a few % of the sample), picks the level-2 bin (bits [19:9]), publishes
// est = (b1 << 20) | (b2 << 9) and restores the zero state it used (global histogram, key
// range, arrival counter).  (One 8-CTA cluster per worker with the sample in distributed
// shared memory measured 26 us at k = 1: the sampling rate is per SM.)
// --------------------------------------------------------------------------------------
// SG_SAMPLE_EST=0 selects the two-launch k_sample + k_estimate (A/B runs)
inline bool sample_est_fused() {
    static const bool on = [] {
        const char* e = getenv("SG_SAMPLE_EST");
        return !(e && *e == '0');
    }();
    return on;
}
constexpr int SE_THREADS = 256;
constexpr int SE_GMIN = 8;
constexpr int SE_CHUNK = 256;  // sample chunk (elements): one 1 KB DRAM row
inline int se_ctas(int k) {  // a power of two: the 512 sample chunks split evenly
    static const int cap = [] {  // SG_SE_G: at most this many sampling CTAs per worker (A/B runs)
        const char* e = getenv("SG_SE_G");
        const int v = e && *e ? atoi(e) : SE_GMAX;
        return v >= SE_GMIN && v <= SE_GMAX ? v : SE_GMAX;
    }();
    // measured (tools/stamps.py, D = R): k = 1: G = 128 / 64 / 32 -> 14.6 / 12.8 / 13.1 us;
    // k = 2: 128 / 64 / 32 -> 16.8 / 12.8 / 12.3; k = 8: 32 / 16 / 8 -> 15.2 / 15.1 / 18.1
    int g = k == 1 ? 64 : 32;
    while (g > SE_GMIN && g > cap) g >>= 1;
    return g;
}
inline size_t se_smem(int G) { return 2 * sizeof(uint32_t) * (size_t)(TopkTraits<float>::SAMPLE / G); }

struct SampleEstArgs {
    const float* g;
    long long ld, dim, s_eff, r_est, r_hi;
    int vec;                // 16-byte aligned rows and strata of >= SE_CHUNK + 4 elements
    SelState<uint32_t>* sel;
    uint4* zero;            // per-call scratch zeroed here (the later kernels' counters)
    long long zero_vec;
    uint32_t* bkeys;        // [k][SAMPLE] keys bucketed by level-1 bin, CTA-major
    uint16_t* boff;         // [k][G][SEL_BINS + 1] bucket offsets of each CTA
    unsigned* h1g;          // [k][SEL_BINS] zero state: level-1 histogram
    unsigned* mmg;          // [k][2] zero state: ~min key, max key
    unsigned* doneg;        // [k] zero state: arrivals
};

__global__ void __launch_bounds__(SE_THREADS)
k_sample_est_f32(SampleEstArgs a) {
    pdl_enter();
    SG_STAMP(0);
    using KO = KeyOf<float>;
    using K = uint32_t;
    extern __shared__ __align__(16) K se_smem_raw[];
    __shared__ unsigned h1[SEL_BINS];      // this CTA's level-1 histogram, then bucket cursors
    __shared__ unsigned s_wsum[SE_THREADS / 32];
    __shared__ K s_mn[SE_THREADS / 32], s_mx[SE_THREADS / 32];
    __shared__ int s_last;
    const int x = blockIdx.x, G = gridDim.x, w = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = SE_THREADS / 32;
    const int per = TopkTraits<float>::SAMPLE / G;  // keys per CTA (sampled case)
    K* keys = se_smem_raw;                          // [per]
    K* buck = se_smem_raw + per;                    // [per]
    for (int i = tid; i < SEL_BINS; i += SE_THREADS) h1[i] = 0;
    {
        const long long cta = (long long)w * G + x, ncta = (long long)G * gridDim.y;
        for (long long i = cta * SE_THREADS + tid; i < a.zero_vec; i += ncta * SE_THREADS) a.zero[i] = make_uint4(0, 0, 0, 0);
    }
    __syncthreads();
    SG_MARK(8);
    const float* row = a.g + (long long)w * a.ld;
    K mn = KO::KMAX, mx = 0;
    int nk = 0;
    if (a.s_eff == a.dim) {  // the sample is the whole row (dim <= SAMPLE)
        const long long slice = (a.dim + G - 1) / G;
        const long long lo = x * slice, hi = lo + slice < a.dim ? lo + slice : a.dim;
        nk = hi > lo ? (int)(hi - lo) : 0;
        for (int i = tid; i < nk; i += SE_THREADS) {
            const K key = KO::key(row[lo + i]);
            keys[i] = key;
            atomicAdd(&h1[key >> 20], 1u);
            mn = key < mn ? key : mn;
            mx = key > mx ? key : mx;
        }
    } else {
        // chunks [x * nc, (x + 1) * nc) of the worker's nch = s_eff / SE_CHUNK, one 1 KB chunk
        // at a hashed offset inside each stratum: the random reads are DRAM-row bound, so a
        // whole row per chunk (not 128-byte chunks) keeps the activations 8x fewer
        const long long nch = a.s_eff / SE_CHUNK;  // 512
        const long long stratum = a.dim / nch;
        const int nc = (int)(nch / G);
        const long long c_lo = (long long)x * nc;
        nk = nc * SE_CHUNK;
        constexpr int BATCH = 4;
        constexpr int PL = SE_CHUNK / 32;  // 8 elements per lane per chunk
        for (int c0 = warp; c0 < nc; c0 += NW * BATCH) {
            float v[BATCH][PL];
#pragma unroll
            for (int u = 0; u < BATCH; ++u) {
                const int cl = c0 + u * NW;
#pragma unroll
                for (int j = 0; j < PL; ++j) v[u][j] = 0.f;
                if (cl < nc) {
                    const long long c = c_lo + cl;
                    const unsigned h = (unsigned)mix64((unsigned long long)c * 0x9e3779b97f4a7c15ull + (unsigned long long)w);
                    if (a.vec) {  // 16-byte aligned start inside the stratum, two float4 per lane
                        const long long off = (long long)(((unsigned long long)h * (unsigned long long)(stratum - SE_CHUNK - 3 + 1)) >> 32);
                        const float4* src = reinterpret_cast<const float4*>(row + ((c * stratum + 3) & ~3LL) + (off & ~3LL));
                        const float4 p0 = __ldg(src + lane), p1 = __ldg(src + 32 + lane);
                        v[u][0] = p0.x; v[u][1] = p0.y; v[u][2] = p0.z; v[u][3] = p0.w;
                        v[u][4] = p1.x; v[u][5] = p1.y; v[u][6] = p1.z; v[u][7] = p1.w;
                    } else {
                        const long long off = (long long)(((unsigned long long)h * (unsigned long long)(stratum - SE_CHUNK + 1)) >> 32);
                        const float* src = row + c * stratum + off;
#pragma unroll
                        for (int j = 0; j < PL; ++j) v[u][j] = __ldg(src + j * 32 + lane);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < BATCH; ++u) {
                const int cl = c0 + u * NW;
                if (cl < nc) {
#pragma unroll
                    for (int j = 0; j < PL; ++j) {
                        const K key = KO::key(v[u][j]);
                        SG_CHECK(cl * SE_CHUNK + j * 32 + lane < per);
                        keys[cl * SE_CHUNK + j * 32 + lane] = key;
                        atomicAdd(&h1[key >> 20], 1u);
                        mn = key < mn ? key : mn;
                        mx = key > mx ? key : mx;
                    }
                }
            }
        }
    }
    mn = warp_min<K>(mn);
    mx = warp_max<K>(mx);
    if (lane == 0) {
        s_mn[warp] = mn;
        s_mx[warp] = mx;
    }
    __syncthreads();
    SG_MARK(9);
    // publish: the non-zero level-1 bins, the key range; then the exclusive bucket offsets
    constexpr int PB = SEL_BINS / SE_THREADS;  // 8 bins per thread
    unsigned hv[PB], hs = 0;
    unsigned* h1w = a.h1g + (long long)w * SEL_BINS;
#pragma unroll
    for (int u = 0; u < PB; ++u) {
        hv[u] = h1[tid * PB + u];
        if (hv[u]) atomicAdd(h1w + tid * PB + u, hv[u]);
        hs += hv[u];
    }
    if (tid == 0) {
        K mn2 = KO::KMAX, mx2 = 0;
        for (int i = 0; i < NW; ++i) {
            mn2 = s_mn[i] < mn2 ? s_mn[i] : mn2;
            mx2 = s_mx[i] > mx2 ? s_mx[i] : mx2;
        }
        atomicMax(a.mmg + 2 * w, ~mn2);  // zero state 0 == ~KMAX
        atomicMax(a.mmg + 2 * w + 1, mx2);
    }
    unsigned incl = hs;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    unsigned run = incl - hs;
    for (int i = 0; i < warp; ++i) run += s_wsum[i];
    uint16_t* bo = a.boff + ((long long)w * G + x) * (SEL_BINS + 1);
#pragma unroll
    for (int u = 0; u < PB; ++u) {
        h1[tid * PB + u] = run;  // bucket cursor
        bo[tid * PB + u] = (uint16_t)run;
        run += hv[u];
    }
    if (tid == SE_THREADS - 1) bo[SEL_BINS] = (uint16_t)run;
    __syncthreads();
    for (int i = tid; i < nk; i += SE_THREADS) {
        const K key = keys[i];
        buck[atomicAdd(&h1[key >> 20], 1u)] = key;
    }
    __syncthreads();
    K* bk = a.bkeys + (long long)w * TopkTraits<float>::SAMPLE + (long long)x * per;
    for (int i = tid; i < nk; i += SE_THREADS) bk[i] = buck[i];
    // the worker's last CTA estimates
    __threadfence();
    __syncthreads();
    SG_MARK(10);
    if (tid == 0) s_last = atomicAdd(a.doneg + w, 1u) == (unsigned)G - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    ld_cg_rows<SEL_BINS / SE_THREADS, SE_THREADS>(h1, h1w, tid);
    __syncthreads();
    SG_MARK(11);
    K est = 0;
    int b1 = -1;
    unsigned long long a1 = 0;
    K ucap = KO::KMAX;  // upper end of the main pass's fine histogram range (see make_plan)
    if (a.r_est <= a.s_eff) {
        // both ranks (r_est, and the mirror r_hi: 0 = none) from one block scan
        int bh;
        unsigned long long ah;
        block_find_two_bins_from_top<SEL_BINS, SE_THREADS>(h1, (unsigned long long)a.r_est, b1, a1,
                                                           (unsigned long long)(a.r_hi >= 1 ? a.r_hi : 0), bh, ah);
        if (b1 >= 0 && a.r_hi >= 1 && bh >= 0 && bh < SEL_BINS - 1) ucap = (K)(bh + 1) << 20;
    }
    __syncthreads();  // h1 is reused for level 2
    for (int i = tid; i < SEL_BINS; i += SE_THREADS) h1[i] = 0;
    __syncthreads();
    if (b1 >= 0) {
        // level 2 over bin b1 of every CTA's bucketed keys: thread c < G fetches CTA c's bucket
        // bounds (all in one round trip), a scan of the bucket sizes, then every thread takes
        // keys of the concatenated buckets (independent loads)
        __shared__ int s_o0[SE_GMAX], s_pre[SE_GMAX + 1];
        int cnt = 0;
        if (tid < G) {
            const uint16_t* bc = a.boff + ((long long)w * G + tid) * (SEL_BINS + 1);
            const int o0 = __ldcg(bc + b1);
            cnt = __ldcg(bc + b1 + 1) - o0;
            s_o0[tid] = o0;
        }
        static_assert(SE_GMAX <= SE_THREADS, "one bucket per thread");
        int inc = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) s_wsum[warp] = (unsigned)inc;
        __syncthreads();
        int wb = 0;
        for (int i = 0; i < warp; ++i) wb += (int)s_wsum[i];
        if (tid < G) s_pre[tid] = wb + inc - cnt;
        if (tid == 0) {
            int t = 0;
            for (int i = 0; i < NW; ++i) t += (int)s_wsum[i];
            s_pre[G] = t;
        }
        __syncthreads();
        const int total = s_pre[G];
        SG_MARK(12);
        const K* kw = a.bkeys + (long long)w * TopkTraits<float>::SAMPLE;
        for (int i = tid; i < total; i += SE_THREADS) {
            int l = 0, h = G;  // the bucket c with s_pre[c] <= i < s_pre[c + 1]
            while (h - l > 1) {
                const int mid = (l + h) >> 1;
                if (s_pre[mid] <= i) l = mid;
                else h = mid;
            }
            const K key = __ldcg(kw + (long long)l * per + s_o0[l] + (i - s_pre[l]));
            atomicAdd(&h1[(key >> 9) & (SEL_BINS - 1)], 1u);
        }
        __syncthreads();
        SG_MARK(13);
        int b2;
        unsigned long long a2;
        block_find_bin_from_top<SEL_BINS, SE_THREADS>(h1, (unsigned long long)a.r_est - a1, b2, a2);
        est = ((K)b1 << 20) | (b2 >= 0 ? ((K)b2 << 9) : (K)0);
    }
    if (tid == 0) {
        SelState<K> o{};
        const K smax = __ldcg(a.mmg + 2 * w + 1);
        o.smax = smax < ucap ? smax : ucap;
        o.est = est;
        o.shift0 = digit_shift<K>(o.smax > est ? o.smax - est : (K)0, H0_BITS);
        o.done = 0;
        o.mode = MODE_NORMAL;
        o.wmode = WR_FAST;
        o.idx_cut = 0xffffffffu;
        a.sel[w] = o;
        // restore the zero state
        a.mmg[2 * w] = 0;
        a.mmg[2 * w + 1] = 0;
        a.doneg[w] = 0;
    }
    for (int i = tid; i < SEL_BINS; i += SE_THREADS) h1w[i] = 0;
}

// --------------------------------------------------------------------------------------
// k_main: the streaming pass (pass 0) or the fallback pass (pass 1).
// --------------------------------------------------------------------------------------
template <typename T> struct MainArgs {
    const T* g;
    long long ld, dim, ntiles, m, segcap;
    int k, vec_ok, pass, nseg, tps;
    SelState<typename KeyOf<T>::K>* sel;
    unsigned* cnt;      // [k][ntiles]
    unsigned* tstart;   // [k][ntiles] offset of the tile's first candidate in its segment
    unsigned* segcnt;   // [k][nseg]
    uint32_t* cidx;     // [k][nseg][segcap]
    T* cval;
    double* pmain;      // [k][nseg]
    unsigned long long* count;  // [2][k]
    typename KeyOf<T>::K* maxkey;
    unsigned* hist0;    // [k][H0_BINS] (pass-specific)
    unsigned* done;     // [k] (pass-specific)
    int nsubt, nsub;
    unsigned* pp;       // [k][BMAX + 1] sub-range prefix per segment (adaptive split)
    uint4* submap;      // [k][NSUB_MAX] sub-range -> (segment, part | parts << 16, lo, hi); x = ~0u unused
    unsigned dense_thr; // k_main_tma: candidates per tile above which placement is staged
    int split_late;     // fallback launch: build the split of pass 0 when the fallback is not taken
};

// Per-lane exclusive prefix and warp total of a small count n (0..7) via 3 ballots.
SG_DEV void warp_scan_small(unsigned n, unsigned& excl, unsigned& total) {
    const unsigned b0 = __ballot_sync(FULL, n & 1u);
    const unsigned b1 = __ballot_sync(FULL, n & 2u);
    const unsigned b2 = __ballot_sync(FULL, n & 4u);
    const unsigned lt = lanemask_lt();
    excl = __popc(b0 & lt) + 2u * __popc(b1 & lt) + 4u * __popc(b2 & lt);
    total = __popc(b0) + 2u * __popc(b1) + 4u * __popc(b2);
}

template <typename T>
SG_DEV void load_tile(const T* row, long long base, long long dim, bool vec, typename Vec16<T>::V (&x)[TK_ROUNDS]) {
    using VT = Vec16<T>;
    constexpr int V = VT::N;
    const int tid = threadIdx.x;
    if (vec && base + tile_elems<T>() <= dim) {
        const typename VT::V* src = reinterpret_cast<const typename VT::V*>(row + base);
#pragma unroll
        for (int r = 0; r < TK_ROUNDS; ++r) x[r] = ld_stream(src + r * TK_THREADS + tid);
    } else {
#pragma unroll
        for (int r = 0; r < TK_ROUNDS; ++r) {
            T t[V];
#pragma unroll
            for (int c = 0; c < V; ++c) {
                const long long e = base + (long long)(r * TK_THREADS + tid) * V + c;
                t[c] = e < dim ? row[e] : (T)0;
            }
            if constexpr (V == 4) x[r] = make_float4(t[0], t[1], t[2], t[3]);
            else x[r] = make_double2(t[0], t[1]);
        }
    }
}

// Sub-range i of a segment's n candidates for the split collect/write passes: starts are
// 4-aligned so the writer's 16-byte loads stay aligned.
SG_DEV long long sub_lo(long long n, int i, int split) {
    // floor(n * i / split) in 32-bit: n = q * split + r  =>  q * i + (r * i) / split
    const unsigned nn = (unsigned)n, sp = (unsigned)split;
    const unsigned q = nn / sp, r = nn - q * sp;
    return i == 0 ? 0 : (long long)((q * (unsigned)i + (r * (unsigned)i) / sp) & ~3u);
}
SG_DEV int sub_of(long long n, long long off, int split) {
    // the largest i with sub_lo(n, i) <= off: a proportional guess, then a short walk
    int i = n > 0 ? (int)(((unsigned long long)off * (unsigned)split) / (unsigned long long)n) : 0;
    if (i > split - 1) i = split - 1;
    while (i > 0 && sub_lo(n, i, split) > off) --i;
    while (i + 1 < split && sub_lo(n, i + 1, split) <= off) ++i;
    return i;
}

// Adaptive split: segment s of a worker gets parts_s = max(1, ceil(n_s * nsubt / C)) sub-ranges
// (C = the worker's candidates), so the collect/write CTAs are balanced by candidate count, not
// by position; sub-ranges are numbered in index order (segment, then part).
SG_DEV unsigned parts_of(unsigned n, unsigned long long C, int nsubt) {
    if (C == 0) return 1u;
    const unsigned long long q = ((unsigned long long)n * (unsigned long long)nsubt + C - 1) / C;
    return q < 1 ? 1u : (unsigned)q;
}

// The adaptive collect/write split of worker w: parts per segment by candidate count
// (parts_of), their prefix and the sub-range map with each sub-range's candidate bounds.
// Block-uniform; C = the worker's candidate count.
template <typename T>
SG_DEV void build_submap(const MainArgs<T>& a, int w, unsigned long long C) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    {
        const unsigned* sc = a.segcnt + (long long)w * a.nseg;
        constexpr int PER = BMAX / TK_THREADS;
        unsigned pv[PER], nv[PER], sum = 0;
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int q = tid * PER + u;
            nv[u] = q < a.nseg ? __ldcg(sc + q) : 0u;
            pv[u] = q < a.nseg ? parts_of(nv[u], C, a.nsubt) : 0u;
            sum += pv[u];
        }
        __shared__ unsigned s_ps[TK_NW];
        unsigned incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) s_ps[warp] = incl;
        __syncthreads();
        unsigned run = incl - sum;
        for (int i = 0; i < warp; ++i) run += s_ps[i];
        unsigned* pp = a.pp + (long long)w * (BMAX + 1);
        uint4* sm = a.submap + (long long)w * NSUB_MAX;
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int q = tid * PER + u;
            if (q < a.nseg) {
                pp[q] = run;
                unsigned lo = 0;
                for (unsigned t = 0; t < pv[u] && run + t < (unsigned)a.nsub; ++t) {
                    const unsigned hi = t + 1 == pv[u] ? nv[u] : (unsigned)sub_lo(nv[u], (int)t + 1, (int)pv[u]);
                    sm[run + t] = make_uint4((unsigned)q, t | (pv[u] << 16), lo, hi);
                    lo = hi;
                }
            }
            run += pv[u];
        }
        __shared__ unsigned s_tot;
        if (tid == TK_THREADS - 1) s_tot = run;
        __syncthreads();
        if (tid == 0) pp[a.nseg] = s_tot;
        for (int i = (int)s_tot + tid; i < a.nsub; i += TK_THREADS) sm[i] = make_uint4(0xffffffffu, 0u, 0u, 0u);
    }
}

// Segment epilogue shared by both main-pass kernels: fixed-tree partial norm, segment count,
// max key, round-0 histogram flush; the last CTA of each worker picks the rank-m bin (or
// flags the fallback pass when fewer than m keys reached est).
template <typename T, bool SPLIT>
SG_DEV void main_finish(const MainArgs<T>& a, int w, int seg, double ss, typename KeyOf<T>::K mx, unsigned run,
                        unsigned* hist, typename KeyOf<T>::K est, int shift0) {
    using K = typename KeyOf<T>::K;
    __shared__ double s_red[32];
    __shared__ K s_kmax[32];
    __shared__ int s_last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    SelState<K>* stp = a.sel + w;
    ss = warp_sum(ss);
    mx = warp_max<K>(mx);
    if (lane == 0) {
        s_red[warp] = ss;
        s_kmax[warp] = mx;
    }
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        K km = 0;
        for (int i = 0; i < nw; ++i) {
            t = dadd(t, s_red[i]);
            km = s_kmax[i] > km ? s_kmax[i] : km;
        }
        a.pmain[(long long)w * a.nseg + seg] = t;
        a.segcnt[(long long)w * a.nseg + seg] = run;
        if (km) atomicMax(a.maxkey + w, km);
        if (run) atomicAdd(a.count + (long long)a.pass * a.k + w, (unsigned long long)run);
    }
    unsigned* gh = a.hist0 + (long long)w * H0_BINS;
    for (int i = tid; i < H0_BINS; i += blockDim.x)
        if (hist[i]) atomicAdd(gh + i, hist[i]);
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(a.done + w, 1u) == (unsigned)a.nseg - 1;  // one arrival per segment
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    ld_cg_rows<H0_BINS / TK_THREADS, TK_THREADS>(hist, gh, tid);
    __syncthreads();
    const unsigned long long C = __ldcg(a.count + (long long)a.pass * a.k + w);
    if (C < (unsigned long long)a.m) {
        if (tid == 0) {  // estimate undershot (pass 0 only): run the fallback pass
            SelState<K> s = *stp;
            s.mode = MODE_FALLBACK;
            *stp = s;
        }
        return;
    }
    // the adaptive collect/write split (k_main's: the TMA pass leaves it to the fallback
    // launch, which always runs, so the streaming kernel carries none of its code)
    if constexpr (SPLIT) build_submap<T>(a, w, C);
    int bin;
    unsigned long long above;
    block_find_bin_from_top<H0_BINS, TK_THREADS>(hist, (unsigned long long)a.m, bin, above);
    if (tid == 0) {
        SelState<K> s = *stp;
        s.lo = est;
        s.span = __ldcg(a.maxkey + w) - est;
        s.shift = shift0;
        s.rank = (unsigned long long)a.m;
        s.done = 0;
        if (a.pass == 1) s.est = 0;
        if (bin < 0) {
            s.done = 1;
            s.T = est;
        } else {
            narrow<K>(s, bin, above, hist[bin], H0_BINS, SEL_BITS);
        }
        *stp = s;
    }
}

// --------------------------------------------------------------------------------------
// k_main_tma: float32 main pass fed by TMA bulk copies.  One elected thread keeps
// MN_STAGES 16 KB tiles of the segment in flight (cp.async.bulk -> shared memory ring,
// mbarrier completion, L2 evict-first); each thread owns 16 contiguous elements of a tile,
// read from shared memory in a lane-rotated order that is bank-conflict free.  Per float4:
// 4 fp64 FMAs for the sum of squares and one |max| test against the candidate threshold;
// the rare candidates are placed with one warp scan per tile (index order preserved).
// --------------------------------------------------------------------------------------
constexpr int MN_STAGES = 3;
constexpr int MN_TILE = 4096;
constexpr unsigned MN_DENSE = 256;  // candidates per tile above which placement is staged
inline unsigned mn_dense() {  // SG_MN_DENSE overrides (A/B runs)
    static const unsigned v = [] {
        const char* e = getenv("SG_MN_DENSE");
        return e && *e ? (unsigned)strtoul(e, nullptr, 10) : MN_DENSE;
    }();
    return v;
}

__global__ void __launch_bounds__(TK_THREADS, 3)
k_main_tma(MainArgs<float> a) {
    SG_STAMP(1);
    // The prologue does not depend on the estimate: the ring starts filling while k_sample_est
    // may still be running (PDL).  (Prefetching further tiles of the segment into L2 here as
    // well measured 1-3% slower at k = 1..8.)
    pdl_trigger();
    using K = uint32_t;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* ring = reinterpret_cast<float*>(smem_raw);
    __shared__ __align__(8) unsigned long long full[MN_STAGES];
    __shared__ unsigned hist[H0_BINS];
    __shared__ unsigned s_wtot[TK_NW];
    __shared__ unsigned short s_stage[MN_TILE];  // dense tiles: candidate offsets in index order
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int w = blockIdx.y, seg = blockIdx.x;
    const float* row = a.g + (long long)w * a.ld;
    const long long t_begin = (long long)seg * a.tps;
    const long long t_end = t_begin + a.tps < a.ntiles ? t_begin + a.tps : a.ntiles;
    const int ntl = (int)(t_end - t_begin);
    unsigned long long policy = 0;
    auto issue = [&](int i) {  // tile t_begin + i -> stage i % MN_STAGES (full tiles only)
        const long long base = (t_begin + i) * MN_TILE;
        if (base + MN_TILE > a.dim) return;
        const int s = i % MN_STAGES;
        mbar_expect_tx(&full[s], MN_TILE * 4);
        bulk_g2s(ring + s * MN_TILE, row + base, MN_TILE * 4, &full[s], policy);
    };
    if (tid == 0) {
        policy = policy_evict_first();
        for (int s = 0; s < MN_STAGES; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
        for (int i = 0; i < MN_STAGES && i < ntl; ++i) issue(i);
    }
    for (int i = tid; i < H0_BINS; i += TK_THREADS) hist[i] = 0;
    pdl_wait();
    SG_STAMP(6);
    SelState<K>* stp = a.sel + w;  // pass 0 only (the fallback pass is k_main)
    const K est = stp->est;
    const int shift0 = stp->shift0;
    const bool take_all = est == 0;
    const float thr = take_all ? 0.f : __uint_as_float(est - 1u);  // key >= est <=> |x| >= thr
    uint32_t* ci = a.cidx + ((long long)w * a.nseg + seg) * a.segcap;
    float* cv = a.cval + ((long long)w * a.nseg + seg) * a.segcap;
    __syncthreads();
    double ss = 0.0, ss1 = 0.0;
    K mx = 0;
    unsigned run = 0;
    const int rot = (lane >> 1) & 3;
    // full tiles come from the TMA ring; a partial last tile (only ever the row's last) is
    // read directly after the loop, so the hot loop carries no bounds logic
    const int nfull = (t_end * MN_TILE <= a.dim) ? ntl : ntl - 1;
    auto place = [&](unsigned M, long long base, const float* src, unsigned n, unsigned incl, unsigned woff) {
        // lane-local ordered writes of this thread's candidates (usually 0-2 of them)
        unsigned pos = run + woff + incl - n;
        while (M) {
            const int b = __ffs(M) - 1;
            M &= M - 1;
            const int off = tid * 16 + b;
            const float val = src[off];
            const K key = KeyOf<float>::key(val);
            mx = key > mx ? key : mx;
            atomicAdd(&hist[digit<K>(key, est, shift0, H0_BINS)], 1u);
SG_CHECK(pos < (unsigned)a.segcap);
            ci[pos] = (uint32_t)(base + off);
            cv[pos] = val;
            ++pos;
        }
    };
    auto scan_and_place = [&](unsigned M, long long base, long long tile, const float* src) {
        const unsigned n = __popc(M);
        unsigned incl = n;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) s_wtot[warp] = incl;
        __syncthreads();
        // this warp's offset and the tile total: a shuffle scan over the TK_NW warp totals
        const unsigned wt = lane < TK_NW ? s_wtot[lane] : 0u;
        unsigned wi = wt;
#pragma unroll
        for (int o = 1; o < TK_NW; o <<= 1) {
            const unsigned y = __shfl_up_sync(FULL, wi, o);
            if (lane >= o) wi += y;
        }
        const unsigned woff = __shfl_sync(FULL, wi - wt, warp);
        const unsigned total = __shfl_sync(FULL, wi, TK_NW - 1);
        if (total > a.dense_thr) {
            // candidate-dense tile (real gradients crowd their large entries into a few layers):
            // stage the offsets in index order, then write them coalesced, one candidate per
            // thread per round (the lane-local path would issue 16 scattered stores per thread).
            // (A warp-aggregated histogram via __match_any_sync measured 1.4x slower here.)
            unsigned pos = woff + incl - n;
            for (unsigned R = M; R; R &= R - 1) s_stage[pos++] = (unsigned short)(tid * 16 + __ffs(R) - 1);
            __syncthreads();
            for (unsigned j0 = 0; j0 < total; j0 += TK_THREADS) {
                const unsigned j = j0 + tid;
                if (j < total) {
                    const int off = s_stage[j];
                    const float val = src[off];
                    const K key = KeyOf<float>::key(val);
                    mx = key > mx ? key : mx;
SG_CHECK(run + j < (unsigned)a.segcap);
                    ci[run + j] = (uint32_t)(base + off);
                    cv[run + j] = val;
                    atomicAdd(&hist[digit<K>(key, est, shift0, H0_BINS)], 1u);
                }
            }
        } else if (M) {
            place(M, base, src, n, incl, woff);
        }
        if (tid == 0) {
            const long long ti = (long long)w * a.ntiles + tile;
            a.cnt[ti] = total;
            a.tstart[ti] = run;
        }
        run += total;
    };
    int s = 0;
    unsigned phase = 0;  // ring stage of tile i and its mbarrier parity, advanced incrementally
    for (int i = 0; i < nfull; ++i) {
        const long long tile = t_begin + i;
        const long long base = tile * MN_TILE;
        const float* tb = ring + s * MN_TILE;
        mbar_wait(&full[s], phase);
        const float4* t4 = reinterpret_cast<const float4*>(tb);
        float4 y[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) y[r] = t4[tid * 4 + ((r + rot) & 3)];
        // candidate mask over this thread's 16 contiguous elements (bit b <-> element 16*tid+b)
        unsigned M = 0;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const float4 v = y[r];
            double& sr = (r & 1) ? ss1 : ss;  // two chains: half the DFMA dependency depth
            sr = fma((double)v.x, (double)v.x, sr);
            sr = fma((double)v.y, (double)v.y, sr);
            sr = fma((double)v.z, (double)v.z, sr);
            sr = fma((double)v.w, (double)v.w, sr);
            const unsigned m4 = (fabsf(v.x) >= thr ? 1u : 0u) | (fabsf(v.y) >= thr ? 2u : 0u) |
                                (fabsf(v.z) >= thr ? 4u : 0u) | (fabsf(v.w) >= thr ? 8u : 0u);
            M |= m4 << (((r + rot) & 3) * 4);
        }
        if (take_all) M = 0xffffu;  // fallback pass: every element (NaN included) is a candidate
        scan_and_place(M, base, tile, tb);
        __syncthreads();  // stage s fully consumed (and s_wtot free) before it is refilled
        if (tid == 0 && i + MN_STAGES < ntl) {
            fence_proxy_async();
            issue(i + MN_STAGES);
        }
        if (++s == MN_STAGES) {
            s = 0;
            phase ^= 1u;
        }
    }
    if (nfull < ntl) {  // partial last tile of the row: direct loads, bounds-checked
        const long long tile = t_begin + nfull;
        const long long base = tile * MN_TILE;
        const long long left = a.dim - base - tid * 16;
        const float* src = row + base;
        unsigned M = 0;
        for (int b = 0; b < 16; ++b) {
            if (b >= left) break;
            const float x = src[tid * 16 + b];
            double& sr = (b & 1) ? ss1 : ss;
            sr = fma((double)x, (double)x, sr);
            if (take_all || fabsf(x) >= thr) M |= 1u << b;
        }
        scan_and_place(M, base, tile, src);
        __syncthreads();
    }
    main_finish<float, false>(a, w, seg, dadd(ss, ss1), mx, run, hist, est, shift0);
}

template <typename T>
__global__ void __launch_bounds__(TK_THREADS, 4)
k_main(MainArgs<T> a) {
    pdl_enter();
    SG_STAMP(2);
    using KO = KeyOf<T>;
    using K = typename KO::K;
    using VT = Vec16<T>;
    constexpr int V = VT::N;
    constexpr int TILE = tile_elems<T>();
    __shared__ unsigned hist[H0_BINS];
    __shared__ unsigned s_wtot[32];
    __shared__ unsigned s_woff[32];
    __shared__ unsigned s_run, s_tbase;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int w = blockIdx.y;
    SelState<K>* stp = a.sel + w;
    if (a.pass == 1 && stp->mode != MODE_FALLBACK) {
        // not taken: the split of the (TMA) main pass, by the worker's first CTA
        if (a.split_late && blockIdx.x == 0) build_submap<T>(a, w, __ldcg(a.count + w));
        return;
    }
    const K est = a.pass == 1 ? (K)0 : stp->est;
    const int shift0 = a.pass == 1 ? digit_shift<K>(KO::KMAX, H0_BITS) : stp->shift0;
    // one segment per CTA for the main pass; the (rare) fallback pass runs on a small grid
    // that strides over the segments
    for (int seg = blockIdx.x; seg < a.nseg; seg += gridDim.x) {
    __syncthreads();  // the previous segment's histogram flush is done
    for (int i = tid; i < H0_BINS; i += TK_THREADS) hist[i] = 0;
    if (tid == 0) s_run = 0;
    const T* row = a.g + (long long)w * a.ld;
    const bool vec = a.vec_ok;
    const long long t_begin = (long long)seg * a.tps;
    const long long t_end = t_begin + a.tps < a.ntiles ? t_begin + a.tps : a.ntiles;
    uint32_t* ci = a.cidx + ((long long)w * a.nseg + seg) * a.segcap;
    T* cv = a.cval + ((long long)w * a.nseg + seg) * a.segcap;
    double ss = 0.0;
    K mx = 0;
    typename VT::V x[TK_ROUNDS];
    if (t_begin < t_end) load_tile<T>(row, t_begin * TILE, a.dim, vec, x);
    __syncthreads();
    for (long long tile = t_begin; tile < t_end; ++tile) {
        const long long base = tile * TILE;
        T v[TK_ROUNDS][V];
#pragma unroll
        for (int r = 0; r < TK_ROUNDS; ++r)
#pragma unroll
            for (int c = 0; c < V; ++c) v[r][c] = VT::get(x[r], c);
        if (tile + 1 < t_end) load_tile<T>(row, base + TILE, a.dim, vec, x);  // next tile in flight
        unsigned cm[TK_ROUNDS];
        const bool full = base + TILE <= a.dim;
#pragma unroll
        for (int r = 0; r < TK_ROUNDS; ++r) {
            cm[r] = 0;
#pragma unroll
            for (int c = 0; c < V; ++c) {
                const bool ok = full || base + (long long)(r * TK_THREADS + tid) * V + c < a.dim;
                const T e = v[r][c];
                const K key = KO::key(e);
                if (ok) {
                    mx = key > mx ? key : mx;
                    ss = fma((double)e, (double)e, ss);
                    if (key >= est) {
                        cm[r] |= 1u << c;
                        atomicAdd(&hist[digit<K>(key, est, shift0, H0_BINS)], 1u);
                    }
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
        __syncthreads();
        if (warp == 0) {
            const unsigned xw = s_wtot[lane];
            unsigned incl = xw;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += y;
            }
            s_woff[lane] = incl - xw;
            if (lane == 31) {
                const long long ti = (long long)w * a.ntiles + tile;
                a.cnt[ti] = incl;
                a.tstart[ti] = s_run;
                s_tbase = s_run;
                s_run += incl;
            }
        }
        __syncthreads();
        const unsigned tb = s_tbase;
#pragma unroll
        for (int r = 0; r < TK_ROUNDS; ++r) {
            if (!cm[r]) continue;
            unsigned pos = tb + s_woff[r * TK_NW + warp] + lp[r];
#pragma unroll
            for (int c = 0; c < V; ++c) {
                if ((cm[r] >> c) & 1u) {
SG_CHECK(pos < (unsigned long long)a.segcap);
                    ci[pos] = (uint32_t)(base + (long long)(r * TK_THREADS + tid) * V + c);
                    cv[pos] = v[r][c];
                    ++pos;
                }
            }
        }
    }
    main_finish<T, true>(a, w, seg, ss, mx, s_run, hist, est, shift0);
    }
}

// --------------------------------------------------------------------------------------
// k_collect: per-segment counts above the rank-m bin + boundary entries; last CTA resolves.
// --------------------------------------------------------------------------------------
template <typename T> struct CollectArgs {
    long long segcap, cap;         // cap: boundary entries stored per worker (RES)
    int nseg, tps, split, nsub, nsubt;
    const unsigned* pp;            // [k][BMAX + 1] (from the main pass's last CTA)
    const uint4* submap;           // [k][NSUB_MAX]
    uint32_t* bpos;                // [k][cap] boundary entry's position in its segment list
    SelState<typename KeyOf<T>::K>* sel;
    const unsigned* segcnt;
    const uint32_t* cidx;
    const T* cval;
    unsigned* seggt;               // [k][nseg]
    unsigned* segbase;             // [k][nseg]
    typename KeyOf<T>::K* bkey;    // [k][cap]
    uint32_t* bidx;
    unsigned long long* bndn;      // [k]
    unsigned* done;                // [k]
};

// Load the N consecutive candidate entries [e0, e0 + N) of a segment list (clipped at hi):
// 16-byte loads when the run is whole (segment bases and sub-range starts are 4-aligned).
template <typename T, int N>
SG_DEV void load16(const T* cv, int e0, int hi, T (&v)[N]) {
    if (e0 + N <= hi) {
        if constexpr (sizeof(T) == 4) {
#pragma unroll
            for (int r = 0; r < N / 4; ++r) {
                const float4 x = *reinterpret_cast<const float4*>(cv + e0 + 4 * r);
                v[4 * r] = x.x; v[4 * r + 1] = x.y; v[4 * r + 2] = x.z; v[4 * r + 3] = x.w;
            }
        } else {
#pragma unroll
            for (int r = 0; r < N / 2; ++r) {
                const double2 x = *reinterpret_cast<const double2*>(cv + e0 + 2 * r);
                v[2 * r] = x.x; v[2 * r + 1] = x.y;
            }
        }
    } else {
#pragma unroll
        for (int u = 0; u < N; ++u) v[u] = e0 + u < hi ? cv[e0 + u] : (T)0;
    }
}
template <int N>
SG_DEV void load16_idx(const uint32_t* ci, int e0, int hi, uint32_t (&x)[N]) {
    if (e0 + N <= hi) {
#pragma unroll
        for (int r = 0; r < N / 4; ++r) {
            const uint4 y = *reinterpret_cast<const uint4*>(ci + e0 + 4 * r);
            x[4 * r] = y.x; x[4 * r + 1] = y.y; x[4 * r + 2] = y.z; x[4 * r + 3] = y.w;
        }
    } else {
#pragma unroll
        for (int u = 0; u < N; ++u) x[u] = e0 + u < hi ? ci[e0 + u] : 0u;
    }
}
constexpr int CL_EPT = 8;                       // consecutive entries per thread
constexpr int CL_SPAN = TK_THREADS * CL_EPT;    // 2048 entries per CTA pass

template <typename T>
__global__ void __launch_bounds__(TK_THREADS, CW_PER_SM)
k_collect(CollectArgs<T> a) {
    pdl_enter();
    SG_STAMP(3);
    using KO = KeyOf<T>;
    using K = typename KO::K;
    __shared__ unsigned s_gt[TK_NW];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int w = blockIdx.y, sub = blockIdx.x;
    const uint4 e = a.submap[(long long)w * NSUB_MAX + sub];  // (uniform: every thread loads it)
    const int seg = e.x == 0xffffffffu ? -1 : (int)e.x;
    if (seg < 0) {  // beyond the worker's sub-ranges
        if (tid == 0) a.seggt[(long long)w * a.nsub + sub] = 0;
        return;
    }
    const SelState<K> st = a.sel[w];
    const K lo = st.lo, span = st.span;
    const int lo32 = (int)e.z, hi32 = (int)e.w;
    const bool fcmp = sizeof(T) == 4 && lo >= 1;  // (lo = 0: NaN keys are in range -- key path)
    const float f_lo = __uint_as_float((unsigned)(lo - 1)), f_hi = __uint_as_float((unsigned)(lo + span - 1));
    const uint32_t* ci = a.cidx + ((long long)w * a.nseg + seg) * a.segcap;
    const T* cv = a.cval + ((long long)w * a.nseg + seg) * a.segcap;
    K* bk = a.bkey + (long long)w * a.cap;
    uint32_t* bi = a.bidx + (long long)w * a.cap;
    uint32_t* bp = a.bpos + (long long)w * a.cap;
    unsigned gt = 0;
    T v[CL_EPT];
    if (lo32 < hi32) load16<T, CL_EPT>(cv, lo32 + tid * CL_EPT, hi32, v);
    for (int base = lo32; base < hi32; base += CL_SPAN) {
        const int e0 = base + tid * CL_EPT;
        T x[CL_EPT];
#pragma unroll
        for (int u = 0; u < CL_EPT; ++u) x[u] = v[u];
        if (base + CL_SPAN < hi32) load16<T, CL_EPT>(cv, e0 + CL_SPAN, hi32, v);  // next chunk in flight
        unsigned bm = 0;  // entries inside the rank-m bin (the boundary)
        if (fcmp) {
            // float32: the key tests as |x| compares (key = bits(|x|) + 1 orders like |x|; NaN
            // compares false, as its key 0 < lo): ~3 instructions per entry instead of ~10
            const int lim = hi32 - e0;
#pragma unroll
            for (int u = 0; u < CL_EPT; ++u) {
                const float ax = fabsf((float)x[u]);
                const bool in = u < lim;
                gt += in && ax > f_hi;
                bm |= (in && ax >= f_lo && ax <= f_hi ? 1u : 0u) << u;
            }
        } else {
#pragma unroll
            for (int u = 0; u < CL_EPT; ++u) {
                const K key = KO::key(x[u]);
                const K d = key - lo;  // wraps for key < lo: excluded by the key >= lo test
                const bool ok = e0 + u < hi32 && key >= lo;
                gt += ok && d > span;
                bm |= (ok && d <= span ? 1u : 0u) << u;
            }
        }
        // warp-aggregated append: one global atomic per warp that holds boundary entries
        const unsigned nb = __popc(bm);
        if (__any_sync(FULL, nb != 0)) {
            unsigned incl = nb;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += y;
            }
            unsigned long long wbase = 0;
            if (lane == 31) wbase = atomicAdd(a.bndn + w, (unsigned long long)incl);
            wbase = __shfl_sync(FULL, wbase, 31);
            unsigned long long q = wbase + incl - nb;
            while (bm) {
                const int u = __ffs(bm) - 1;
                bm &= bm - 1;
                if (q >= (unsigned long long)a.cap) break;  // oversized: counted only (slow mode)
SG_CHECK(e0 + u < hi32 && q < (unsigned long long)a.cap);
                bk[q] = KO::key(x[u]);
                bi[q] = ci[e0 + u];
                bp[q] = (uint32_t)(e0 + u);
                ++q;
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) gt += __shfl_xor_sync(FULL, gt, o);
    if (lane == 0) s_gt[warp] = gt;
    __syncthreads();
    if (tid == 0) {
        unsigned t = 0;
        for (int i = 0; i < TK_NW; ++i) t += s_gt[i];
        a.seggt[(long long)w * a.nsub + sub] = t;
    }
}

// --------------------------------------------------------------------------------------
// resolve_small: one CTA per worker finishes the select in shared memory when the
// boundary is small (the normal case): T, the tie cut by index, per-segment output bases.
// --------------------------------------------------------------------------------------
constexpr int RS_DIRECT = 256;  // boundary sets ranked directly (a warp per entry); larger: radix rounds

template <typename T>
SG_DEV void resolve_small(const CollectArgs<T>& a, int w, unsigned long long h, unsigned* hist) {
    using K = typename KeyOf<T>::K;
    constexpr int TILE = tile_elems<T>();
    constexpr int NT = 1024;
    constexpr int RES = TopkTraits<T>::RES;
    __shared__ SelState<K> sst;
    __shared__ unsigned s_eq, s_res[2];
    __shared__ K s_T;           // direct mode: the threshold key and the tie cut
    __shared__ unsigned s_cut0;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#ifdef SG_PHASES
    long long ph[8];
    int nph = 0;
    ph[nph++] = clock64();
#define SG_PH() do { __syncthreads(); if (nph < 8) ph[nph++] = clock64(); } while (0)
#else
#define SG_PH() do {} while (0)
#endif
    K* sk = reinterpret_cast<K*>(smem_raw);
    uint32_t* si = reinterpret_cast<uint32_t*>(sk + RES);
    uint32_t* sp = si + RES;                               // position in the segment list
    unsigned* kb = sp + RES;                               // [nsub]
    unsigned* sc = kb + NSUB_MAX;                          // [nseg] segment candidate counts
    unsigned* pp = sc + BMAX;                              // [nseg + 1] sub-range prefix (adaptive split)
    uint8_t* sf = reinterpret_cast<uint8_t*>(pp + BMAX + 1);
    const K* bk = a.bkey + (long long)w * a.cap;
    const uint32_t* bi = a.bidx + (long long)w * a.cap;
    const uint32_t* bpp = a.bpos + (long long)w * a.cap;
    const bool direct = h <= (unsigned long long)RS_DIRECT;  // the normal case (tens to hundreds of entries)
    if (direct) {
        // every load of the phase in flight before the first shared-memory store
        static_assert(NSUB_MAX <= 2 * NT && BMAX <= NT, "two sub-range words, one segment word per thread");
        const bool has = tid < (int)h;
        const long long sb = (long long)w * a.nsub, cb = (long long)w * a.nseg, pb = (long long)w * (BMAX + 1);
        K k0 = 0;
        uint32_t i0 = 0, p0 = 0;
        if (has) {
            k0 = bk[tid];
            i0 = bi[tid];
            p0 = bpp[tid];
        }
        const unsigned g0 = tid < a.nsub ? a.seggt[sb + tid] : 0u;
        const unsigned g1 = tid + NT < a.nsub ? a.seggt[sb + tid + NT] : 0u;
        const unsigned c0 = tid < a.nseg ? a.segcnt[cb + tid] : 0u;
        const unsigned q0 = tid <= a.nseg ? __ldcg(a.pp + pb + tid) : 0u;
        const unsigned q1 = tid == 0 && a.nseg >= NT ? __ldcg(a.pp + pb + NT) : 0u;
        if (has) {
            sk[tid] = k0;
            si[tid] = i0;
            sp[tid] = p0;
        }
        if (tid < a.nsub) kb[tid] = g0;
        if (tid + NT < a.nsub) kb[tid + NT] = g1;
        if (tid < a.nseg) sc[tid] = c0;
        if (tid <= a.nseg) pp[tid] = q0;
        if (tid == 0 && a.nseg >= NT) pp[NT] = q1;
    } else {
        for (long long i = tid; i < (long long)h; i += NT) {
            sk[i] = bk[i];
            si[i] = bi[i];
            sp[i] = bpp[i];
        }
        for (int i = tid; i < a.nsub; i += NT) kb[i] = a.seggt[(long long)w * a.nsub + i];
        for (int i = tid; i < a.nseg; i += NT) sc[i] = a.segcnt[(long long)w * a.nseg + i];
        for (int i = tid; i <= a.nseg; i += NT) pp[i] = __ldcg(a.pp + (long long)w * (BMAX + 1) + i);
    }
    if (tid == 0) {
        sst = a.sel[w];
        s_eq = 0;
    }
    SG_PH();
    if (direct) {
        // rank every boundary entry in the reference's order (descending key, ascending index):
        // the entry ranked need - 1 is the threshold T and the tie cut (np.lexsort keeps the keys
        // above T and the lowest indices at T) -- one pass instead of radix rounds + a tie pass
        __syncthreads();  // sst, sk, si
        const unsigned long long need0 = sst.rank;
        const int hn = (int)h;
        for (int i = warp; i < hn; i += NT / 32) {  // warp per entry, 32 comparisons per ballot
            const K kk = sk[i];
            const uint32_t ii = si[i];
            unsigned rank = 0;
            for (int j0 = 0; j0 < hn; j0 += 32) {
                const int j = j0 + lane;
                bool before = false;
                if (j < hn) {
                    const K kj = sk[j];
                    before = kj > kk || (kj == kk && si[j] < ii);
                }
                rank += __popc(__ballot_sync(FULL, before));
            }
            if (lane == 0 && (unsigned long long)rank + 1 == need0) {
                s_T = kk;
                s_cut0 = ii;
            }
        }
        __syncthreads();
        if (tid == 0) {
            sst.T = s_T;
            sst.done = 1;
        }
    } else {
        block_select<K, NT>(sk, (long long)h, sst, hist);
    }
    SG_PH();
    // (direct: s_T was written before the barrier above; sst.T is tid 0's copy for the write-back)
    const K T_ = direct ? s_T : sst.T;
    const unsigned long long need = sst.rank;
    // ties at T: keep the `need` lowest indices among keys == T (direct: the cut is known)
    unsigned eqc = 0;
    for (long long i = direct ? (long long)h : tid; i < (long long)h; i += NT) {
        const bool e = sk[i] == T_;
        sf[i] = e;
        eqc += e;
    }
    atomicAdd(&s_eq, eqc);
    __syncthreads();
    unsigned cut = direct ? s_cut0 : 0xffffffffu;
    if (!direct && (unsigned long long)s_eq > need) {
        if (s_eq <= (unsigned)SEL_BINS) {
            // a small tie group: list its indices, and the cut is the one with need-1 smaller
            // (indices are distinct positions)
            __shared__ unsigned s_tn, s_cut;
            if (tid == 0) s_tn = 0;
            __syncthreads();
            for (long long i = tid; i < (long long)h; i += NT)
                if (sf[i]) hist[atomicAdd(&s_tn, 1u)] = si[i];
            __syncthreads();
            const unsigned n = s_tn;
            for (unsigned j = tid; j < n; j += NT) {
                const unsigned x = hist[j];
                unsigned c = 0;
                for (unsigned q = 0; q < n; ++q) c += hist[q] < x;
                if (c == (unsigned)need - 1u) s_cut = x;
            }
            __syncthreads();
            cut = s_cut;
        } else {
            cut = block_select_small_u32<NT>(si, sf, (long long)h, need, hist, s_res);
        }
    }
    __syncthreads();
    SG_PH();
    // kept boundary entries per segment
    for (long long i = tid; i < (long long)h; i += NT) {
        const K key = sk[i];
        if (key > T_ || (key == T_ && si[i] <= cut)) {
            const int seg = (int)((si[i] / TILE) / a.tps);
            atomicAdd(&kb[pp[seg] + sub_of((long long)sc[seg], sp[i], (int)(pp[seg + 1] - pp[seg]))], 1u);
        }
    }
    __syncthreads();
    SG_PH();
    // exclusive scan over sub-ranges of (count above the bin + kept boundary): thread t owns
    // sub-ranges 2t, 2t+1 (nsub <= NSUB_MAX = 2 * NT)
    {
        __shared__ unsigned s_ws[NT / 32];
        const int s0 = 2 * tid;
        const unsigned v0 = s0 < a.nsub ? kb[s0] : 0u, v1 = s0 + 1 < a.nsub ? kb[s0 + 1] : 0u;
        const unsigned v = v0 + v1;
        unsigned incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) s_ws[warp] = incl;
        __syncthreads();
        unsigned wb = 0;
        for (int i = 0; i < warp; ++i) wb += s_ws[i];
        const unsigned ex = wb + incl - v;
        if (s0 < a.nsub) a.segbase[(long long)w * a.nsub + s0] = ex;
        if (s0 + 1 < a.nsub) a.segbase[(long long)w * a.nsub + s0 + 1] = ex + v0;
    }
    if (tid == 0) {
        SelState<K> s = sst;
        s.idx_cut = cut;
        s.wmode = WR_FAST;
        s.done = 1;
        a.sel[w] = s;
    }
#ifdef SG_PHASES
    SG_PH();
    if (tid == 0 && w == 0)
        printf("[resolve w0 h=%llu eq=%u nsub=%d] load %lld select %lld ties %lld kept %lld scan %lld cycles\n", h, s_eq,
               a.nsub, ph[1] - ph[0], ph[2] - ph[1], ph[3] - ph[2], ph[4] - ph[3], ph[5] - ph[4]);
#endif
#undef SG_PH
}

// --------------------------------------------------------------------------------------
// k_resolve: grid (G, k), one launch.  Every CTA reads all k boundary counts, so the common
// case (every boundary fits one CTA's shared memory) needs no grid-wide step: CTA 0 of each
// worker resolves it in shared memory (resolve_small) and the other CTAs exit.  If some
// worker's boundary is oversized (heavy ties), all G*k CTAs -- co-resident by cooperative
// launch -- run the radix rounds over that worker's candidate lists in global memory (the
// boundary itself was only counted) with a grid barrier between the histogram and the bin
// pick; its write then takes the slow mode.
// --------------------------------------------------------------------------------------
template <typename T> struct ResolveArgs {
    SelState<typename KeyOf<T>::K>* sel;
    unsigned* hist;   // [k][ROUNDS_MAX][SEL_BINS] (zeroed per call)
    unsigned* bar;    // grid-barrier counter (zeroed per call)
};

template <typename K>
SG_DEV SelState<K> ld_cg_state(const SelState<K>* p) {
    static_assert(sizeof(SelState<K>) % 8 == 0, "SelState is read as 64-bit words");
    SelState<K> s;
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(p);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(&s);
#pragma unroll
    for (int i = 0; i < (int)(sizeof(SelState<K>) / 8); ++i) dst[i] = __ldcg(src + i);
    return s;
}

SG_DEV void grid_barrier(unsigned* ctr, unsigned nblocks, unsigned& gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned target = (gen + 1) * nblocks;
        atomicAdd(ctr, 1u);
        while (ld_acquire_gpu(ctr) < target) __nanosleep(64);
        __threadfence();
    }
    ++gen;
    __syncthreads();
}

template <typename T>
__global__ void __launch_bounds__(1024)
k_resolve(CollectArgs<T> a, ResolveArgs<T> r) {
    pdl_enter();
    SG_STAMP(4);
    using K = typename KeyOf<T>::K;
    constexpr int RES = TopkTraits<T>::RES;
    constexpr int NT = 1024;
    __shared__ unsigned hist[SEL_BINS];
    __shared__ SelState<K> st;
    const int x = blockIdx.x, w = blockIdx.y, tid = threadIdx.x;
    // any oversized boundary? (every CTA reaches the same answer)
    const bool any = __syncthreads_or(tid < (int)gridDim.y && a.bndn[tid] > (unsigned long long)RES);
    const unsigned long long h = a.bndn[w];
    const bool slow = h > (unsigned long long)RES;
    if (x == 0 && !slow) resolve_small<T>(a, w, h, hist);
    if (!any) return;  // uniform over the grid
    // slow mode: radix rounds over the oversized boundary sets
    const unsigned nblocks = gridDim.x * gridDim.y;
    unsigned gen = 0;
    using KO = KeyOf<T>;
    for (int round = 0; round < TopkTraits<T>::ROUNDS_MAX; ++round) {
        if (tid == 0) st = ld_cg_state(r.sel + w);
        for (int i = tid; i < SEL_BINS; i += NT) hist[i] = 0;
        __syncthreads();
        unsigned* gh = r.hist + ((long long)w * TopkTraits<T>::ROUNDS_MAX + round) * SEL_BINS;
        if (slow && !st.done) {
            const K lo = st.lo, span = st.span;
            const int shift = st.shift;
            // CTA x takes segments x, x + G, ...; its 1024 threads stream each with RS_U
            // independent loads in flight
            constexpr int RS_U = 4;
            for (int seg = x; seg < a.nseg; seg += gridDim.x) {
                const int n = (int)a.segcnt[(long long)w * a.nseg + seg];
                const T* cv = a.cval + ((long long)w * a.nseg + seg) * a.segcap;
                for (int i0 = 0; i0 < n; i0 += RS_U * NT) {
                    T v[RS_U];
#pragma unroll
                    for (int u = 0; u < RS_U; ++u) {
                        const int i = i0 + u * NT + tid;
                        v[u] = i < n ? __ldcg(cv + i) : T(0);
                    }
#pragma unroll
                    for (int u = 0; u < RS_U; ++u) {
                        const K key = KO::key(v[u]);
                        if (i0 + u * NT + tid < n && key >= lo && key - lo <= span)
                            atomicAdd(&hist[digit<K>(key, lo, shift, SEL_BINS)], 1u);
                    }
                }
            }
            __syncthreads();
            for (int i = tid; i < SEL_BINS; i += NT)
                if (hist[i]) atomicAdd(gh + i, hist[i]);
        }
        grid_barrier(r.bar, nblocks, gen);
        if (slow && !st.done && x == 0) {
            for (int i = tid; i < SEL_BINS; i += NT) hist[i] = __ldcg(gh + i);
            __syncthreads();
            if (tid < 32) {
                int bin;
                unsigned long long above;
                find_bin_from_top<SEL_BINS>(hist, st.rank, bin, above);
                if (tid == 0) {
                    SelState<K> s = st;
                    if (bin < 0) {
                        s.done = 1;
                        s.T = s.lo;
                    } else {
                        narrow<K>(s, bin, above, hist[bin], SEL_BINS, SEL_BITS);
                    }
                    r.sel[w] = s;
                }
            }
        }
        grid_barrier(r.bar, nblocks, gen);
    }
    if (slow && x == 0 && tid == 0) {
        SelState<K> s = ld_cg_state(r.sel + w);
        s.wmode = WR_SLOW;
        r.sel[w] = s;
    }
}

// --------------------------------------------------------------------------------------
// k_write: ordered compaction of the kept set + merge offsets + (last CTA) norms and gate.
// --------------------------------------------------------------------------------------
template <typename T> struct WriteArgs {
    long long ntiles, segcap, m;
    int k, nseg, tps, split, nsub, nsubt;
    const uint4* submap;
    const SelState<typename KeyOf<T>::K>* sel;
    const unsigned* tstart;
    const unsigned* segcnt;
    const unsigned* segbase;
    const uint32_t* cidx;
    const T* cval;
    unsigned long long* status;   // [k][nseg] (slow mode look-back)
    unsigned* done;
    uint32_t* idx;
    T* val;
    int* tile_off;                // [k][ntiles+1] or null (f32 merge offsets)
    double* pwrite;               // [k][nseg]
    const double* pmain;          // [k][nseg]
    double* norms2;
    sg_gate_state* states;
    uint8_t* decision;
    double* rho;
    unsigned ring_off;            // float32: byte offset of the candidate ring in the dynamic shared memory
};

constexpr unsigned long long CNT_BITS = 31;
constexpr unsigned long long CNT_MASK = (1ull << CNT_BITS) - 1;

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

constexpr int WR_EPT = 4;                      // consecutive entries per thread per chunk
constexpr int WR_CHUNK = TK_THREADS * WR_EPT;  // 1024

// Sub-range epilogue of k_write: fixed-order partial norm of the kept values.
template <typename T>
SG_DEV void write_tail(const WriteArgs<T>& a, double ss) {
    __shared__ double s_red[TK_NW];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int w = blockIdx.y, sub = blockIdx.x;
    ss = warp_sum(ss);
    if (lane == 0) s_red[warp] = ss;
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;
        for (int i = 0; i < TK_NW; ++i) s = dadd(s, s_red[i]);
        a.pwrite[(long long)w * a.nsub + sub] = s;
    }
}

// Fast-mode write (T and the tie cut are final).  The CTA streams its sub-range in chunks of
// WF_SPAN entries: round r of a chunk is entries [base + 256 r, base + 256 (r + 1)), one per
// thread, so every warp access of a round covers consecutive entries (float32: the chunks come
// through a TMA ring).  The kept entries' output slots come from one barrier per chunk: each
// (round, warp) publishes its kept count (a ballot), and after the barrier a 32-lane scan over
// the (round, warp) slots gives every entry its kept-before count.  Merge offsets,
// toff[t] = kept entries with index < 4096 t, come from the main pass's per-tile candidate starts
// (s_ts: tile t's first candidate's offset in the segment list): the kept-before count at that
// offset, read from the chunk's kept-before array -- no per-entry tile logic.  A tile start lies
// in exactly one sub-range [lo, hi); starts at the segment's end (empty trailing tiles) go to its
// last part.
constexpr int WF_R = 4;                      // rounds (entries per thread) per chunk
constexpr int WF_SPAN = TK_THREADS * WF_R;   // 1024 entries per chunk
static_assert(WF_R * TK_NW == 32, "one lane per (round, warp) slot");
constexpr int WT_STAGES = 3;                                 // float32 ring depth (chunks in flight)
constexpr size_t WT_RING = (size_t)WT_STAGES * 2 * WF_SPAN * 4;

template <typename T>
SG_DEV double write_fast(const WriteArgs<T>& a, int nt, long long t0, int* toff, const unsigned* s_ts,
                         typename KeyOf<T>::K T_, unsigned cut, int seg, int lo32, int n32, bool last_part) {
    using KO = KeyOf<T>;
    using K = typename KO::K;
    __shared__ unsigned s_wt[2][32];  // (round, warp) kept counts, by chunk parity
    __shared__ unsigned s_kb[WF_SPAN];  // kept-before count of every entry of the chunk
    __shared__ int s_jc;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int w = blockIdx.y, sub = blockIdx.x;
    const uint32_t* ci = a.cidx + ((long long)w * a.nseg + seg) * a.segcap;
    const T* cv = a.cval + ((long long)w * a.nseg + seg) * a.segcap;
    uint32_t* oi = a.idx + (long long)w * a.m;
    T* ov = a.val + (long long)w * a.m;
    const unsigned lt_mask = lanemask_lt();
    const bool fcmp = sizeof(T) == 4 && T_ >= 1;  // (T = 0 keeps NaN keys -- key path)
    const float f_T = __uint_as_float((unsigned)(T_ - 1));
    T v[WF_R];
    uint32_t ii[WF_R];
    // float32: the chunks stream through a WT_STAGES-deep shared-memory ring filled by
    // TMA bulk copies (values then indices per stage; sub-range starts are 4-aligned and a
    // segment's list capacity is a multiple of 4096, so a chunk rounded up to 16 bytes stays in
    // the list); otherwise the next chunk's loads are in flight in registers
    constexpr bool ring_on = sizeof(T) == 4;
    extern __shared__ __align__(128) unsigned char wr_smem_raw[];
    uint32_t* ring = reinterpret_cast<uint32_t*>(wr_smem_raw + a.ring_off);  // [WT_STAGES][2][WF_SPAN]
    __shared__ __align__(8) unsigned long long wbar[WT_STAGES];
    const int nch = n32 > lo32 ? (n32 - lo32 + WF_SPAN - 1) / WF_SPAN : 0;
    unsigned long long policy = 0;
    auto issue = [&](int c) {
        const int st = c % WT_STAGES;
        const int b0 = lo32 + c * WF_SPAN;
        const int n = n32 - b0 < WF_SPAN ? n32 - b0 : WF_SPAN;
        const unsigned bytes = (unsigned)((n + 3) & ~3) * 4u;
        uint32_t* d = ring + (size_t)st * 2 * WF_SPAN;
        mbar_expect_tx(&wbar[st], 2 * bytes);
        bulk_g2s(d, cv + b0, bytes, &wbar[st], policy);
        bulk_g2s(d + WF_SPAN, ci + b0, bytes, &wbar[st], policy);
    };
    if constexpr (ring_on) {
        if (tid == 0) {
            policy = policy_evict_first();
            for (int st = 0; st < WT_STAGES; ++st) mbar_init(&wbar[st], 1);
            fence_mbar_init();
            for (int c = 0; c < WT_STAGES && c < nch; ++c) issue(c);
        }
    } else {
#pragma unroll
        for (int r = 0; r < WF_R; ++r) {
            const int e = lo32 + r * TK_THREADS + tid;
            v[r] = e < n32 ? cv[e] : (T)0;
            ii[r] = e < n32 ? ci[e] : 0u;
        }
    }
    if (toff && tid == 0) {  // first tile of the segment whose first candidate is >= lo32
        int l = 0, h = nt;
        while (l < h) {
            const int mid = (l + h) >> 1;
            if ((int)s_ts[mid] < lo32) l = mid + 1;
            else h = mid;
        }
        s_jc = l;
    }
    __syncthreads();
    int jc = toff ? s_jc : 0;
    unsigned g32 = a.segbase[(long long)w * a.nsub + sub];
    double ss = 0.0;
    int par = 0, ch = 0;
    unsigned phase = 0;
    for (int base = lo32; base < n32; base += WF_SPAN, par ^= 1, ++ch) {
        T x[WF_R];
        uint32_t xi[WF_R];
        if constexpr (ring_on) {
            const int st = ch % WT_STAGES;
            mbar_wait(&wbar[st], phase);
            if (st == WT_STAGES - 1) phase ^= 1u;
            const uint32_t* d = ring + (size_t)st * 2 * WF_SPAN;
#pragma unroll
            for (int r = 0; r < WF_R; ++r) {
                if constexpr (sizeof(T) == 4) x[r] = __uint_as_float(d[r * TK_THREADS + tid]);
                xi[r] = d[WF_SPAN + r * TK_THREADS + tid];
            }
        } else {
#pragma unroll
            for (int r = 0; r < WF_R; ++r) {
                x[r] = v[r];
                xi[r] = ii[r];
            }
            if (base + WF_SPAN < n32) {  // next chunk in flight
#pragma unroll
                for (int r = 0; r < WF_R; ++r) {
                    const int e = base + WF_SPAN + r * TK_THREADS + tid;
                    v[r] = e < n32 ? cv[e] : (T)0;
                    ii[r] = e < n32 ? ci[e] : 0u;
                }
            }
        }
        unsigned ball[WF_R];
#pragma unroll
        for (int r = 0; r < WF_R; ++r) {
            const int e = base + r * TK_THREADS + tid;
            bool keep;
            if (fcmp) {  // float32: the key tests as |x| compares (see k_collect)
                const float ax = fabsf((float)x[r]);
                keep = ax > f_T || (ax == f_T && xi[r] <= cut);
            } else {
                const K key = KO::key(x[r]);
                keep = key > T_ || (key == T_ && xi[r] <= cut);
            }
            ball[r] = __ballot_sync(FULL, e < n32 && keep);
            if (lane == 0) s_wt[par][r * TK_NW + warp] = __popc(ball[r]);
        }
        __syncthreads();
        if (ring_on && tid == 0 && ch + WT_STAGES < nch) {  // every thread has read this stage (float32)
            fence_proxy_async();
            issue(ch + WT_STAGES);
        }
        // lane i <-> slot i = (round i / TK_NW, warp i % TK_NW), in index order
        const unsigned c = s_wt[par][lane];
        unsigned incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        const unsigned excl = incl - c, tot = __shfl_sync(FULL, incl, 31);
#pragma unroll
        for (int r = 0; r < WF_R; ++r) {
            const unsigned pos = g32 + __shfl_sync(FULL, excl, r * TK_NW + warp) + __popc(ball[r] & lt_mask);
            if (toff) s_kb[r * TK_THREADS + tid] = pos;
            if ((ball[r] >> lane) & 1u) {
                SG_CHECK(base + r * TK_THREADS + tid < n32);
                if (pos < (unsigned)a.m) {
                    oi[pos] = xi[r];
                    ov[pos] = x[r];
                    ss = fma((double)x[r], (double)x[r], ss);
                }
            }
        }
        if (toff) {
            // tiles whose first candidate lies in this chunk: merge offset = kept before it
            __syncthreads();  // s_kb complete
            const int c1 = base + WF_SPAN < n32 ? base + WF_SPAN : n32;
            for (;;) {
                const int j = jc + tid;
                const bool in = j < nt && (int)s_ts[j] < c1;
                if (in) {
                    SG_CHECK((int)s_ts[j] >= base && (int)s_ts[j] - base < WF_SPAN && t0 + j < a.ntiles);
                    toff[t0 + j] = (int)s_kb[s_ts[j] - base];
                }
                const int cnt = __syncthreads_count(in);
                jc += cnt;
                if (cnt < TK_THREADS) break;
            }
        }
        g32 += tot;
    }
    if (toff && last_part) {
        // tiles with no candidate at or after the segment's last entry: offset = kept total
        SG_CHECK(t0 + nt <= a.ntiles && g32 <= (unsigned)a.m + (unsigned)WF_SPAN);
        for (int j = jc + tid; j < nt; j += TK_THREADS) toff[t0 + j] = (int)g32;
        if (tid == 0 && t0 + nt == a.ntiles) toff[a.ntiles] = (int)a.m;
    }
    return ss;
}

template <typename T>
SG_DEV void write_body(const WriteArgs<T>& a) {
    using KO = KeyOf<T>;
    using K = typename KO::K;
    constexpr int TILE = tile_elems<T>();
    constexpr bool OFFS = TILE == MERGE_TILE;
    __shared__ unsigned s_gw[TK_NW], s_ew[TK_NW];
    __shared__ unsigned long long s_gb, s_eb;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned* s_ts = reinterpret_cast<unsigned*>(smem_raw);  // [tps] tile starts of this segment
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int w = blockIdx.y, sub = blockIdx.x;
    const uint4 e = a.submap[(long long)w * NSUB_MAX + sub];  // (uniform: every thread loads it)
    const int seg = e.x == 0xffffffffu ? -1 : (int)e.x;
    const int part = (int)(e.y & 0xffffu), split = (int)(e.y >> 16);
    if (seg < 0) {  // beyond the worker's sub-ranges: no kept entries, no norm
        if (tid == 0) a.pwrite[(long long)w * a.nsub + sub] = 0.0;
        return;
    }
    const SelState<K> st = a.sel[w];
    const K T_ = st.T;
    const unsigned cut = st.idx_cut;
    const unsigned long long need = st.rank;
    const bool slow = st.wmode == WR_SLOW;
    const long long i_lo = e.z;
    const long long n = e.w;  // end of the sub-range
    const bool last_part = part + 1 == split;
    const uint32_t* ci = a.cidx + ((long long)w * a.nseg + seg) * a.segcap;
    const T* cv = a.cval + ((long long)w * a.nseg + seg) * a.segcap;
    const long long t0 = (long long)seg * a.tps;
    const int nt = (int)(t0 + a.tps < a.ntiles ? a.tps : a.ntiles - t0);
    int* toff = (OFFS && a.tile_off) ? a.tile_off + (long long)w * (a.ntiles + 1) : nullptr;

    if (toff) {
        for (int j = tid; j < nt; j += TK_THREADS) s_ts[j] = a.tstart[(long long)w * a.ntiles + t0 + j];
        __syncthreads();
    }
    if (!slow) {
        write_tail<T>(a, write_fast<T>(a, nt, t0, toff, s_ts, T_, cut, seg, (int)i_lo, (int)n, last_part));
        return;
    }
    unsigned long long gb, eb;  // kept-before counters (fast mode: gb only)
    if (!slow) {
        gb = a.segbase[(long long)w * a.nsub + sub];
        eb = 0;
    } else {
        // pass 1: counts, then a decoupled look-back over this worker's segments
        unsigned gc = 0, ec = 0;
        for (long long i = i_lo + tid; i < n; i += TK_THREADS) {
            const K key = KO::key(cv[i]);
            gc += key > T_;
            ec += key == T_;
        }
        for (int o = 16; o > 0; o >>= 1) {
            gc += __shfl_xor_sync(FULL, gc, o);
            ec += __shfl_xor_sync(FULL, ec, o);
        }
        if (lane == 0) {
            s_gw[warp] = gc;
            s_ew[warp] = ec;
        }
        __syncthreads();
        if (warp == 0) {
            unsigned long long gtot = 0, etot = 0;
            for (int i = 0; i < TK_NW; ++i) {
                gtot += s_gw[i];
                etot += s_ew[i];
            }
            const unsigned long long pre =
                lookback(a.status + (long long)w * a.nsub, sub, (gtot << CNT_BITS) | etot);
            if (lane == 0) {
                s_gb = pre >> CNT_BITS;
                s_eb = pre & CNT_MASK;
            }
        }
        __syncthreads();
        gb = s_gb;
        eb = s_eb;
    }
    uint32_t* oi = a.idx + (long long)w * a.m;
    T* ov = a.val + (long long)w * a.m;
    double ss = 0.0;
    __shared__ unsigned s_kb[WR_CHUNK];  // kept-before count per entry of the chunk (merge offsets)
    __shared__ int s_jc;
    // 32-bit bookkeeping: segment positions < 2^31, output positions < m < 2^31
    const int lo32 = (int)i_lo, n32 = (int)n;
    unsigned g32 = (unsigned)gb, e32 = (unsigned)eb;
    const unsigned need32 = (unsigned)(need < 0xffffffffull ? need : 0xffffffffull);
    __syncthreads();  // s_ts complete (fast mode has no barrier above)
    if (toff && tid == 0) {  // first tile of this segment whose first candidate is >= i_lo
        int l = 0, h = nt;
        while (l < h) {
            const int mid = (l + h) >> 1;
            if ((int)s_ts[mid] < lo32) l = mid + 1;
            else h = mid;
        }
        s_jc = l;
    }
    __syncthreads();
    int jc = toff ? s_jc : 0;
    for (int c0 = lo32; c0 < n32; c0 += WR_CHUNK) {
        const int c1 = c0 + WR_CHUNK < n32 ? c0 + WR_CHUNK : n32;
        const int e0i = c0 + tid * WR_EPT;
        T vv[WR_EPT];
        uint32_t ii[WR_EPT];
        if (sizeof(T) == 4 && e0i + WR_EPT <= n32) {  // segment base and chunk start are 16-byte aligned
            if constexpr (sizeof(T) == 4) {
                const float4 v4 = *reinterpret_cast<const float4*>(cv + e0i);
                const uint4 i4 = *reinterpret_cast<const uint4*>(ci + e0i);
                vv[0] = v4.x; vv[1] = v4.y; vv[2] = v4.z; vv[3] = v4.w;
                ii[0] = i4.x; ii[1] = i4.y; ii[2] = i4.z; ii[3] = i4.w;
            }
        } else {
#pragma unroll
            for (int u = 0; u < WR_EPT; ++u) {
                const bool ok = e0i + u < n32;
                vv[u] = ok ? cv[e0i + u] : (T)0;
                ii[u] = ok ? ci[e0i + u] : 0u;
            }
        }
        unsigned kflag = 0, eflag = 0;
#pragma unroll
        for (int u = 0; u < WR_EPT; ++u) {
            const K key = KO::key(vv[u]);
            const bool ok = e0i + u < n32;
            if (!slow) {
                kflag |= (ok && (key > T_ || (key == T_ && ii[u] <= cut)) ? 1u : 0u) << u;
            } else {
                kflag |= (ok && key > T_ ? 1u : 0u) << u;
                eflag |= (ok && key == T_ ? 1u : 0u) << u;
            }
        }
        // warp-inclusive scans of the per-thread counts (packed: kept in the low half,
        // ties at T in the high half; both <= 4 * 32)
        const unsigned cnt = __popc(kflag) | ((unsigned)__popc(eflag) << 16);
        unsigned incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) s_gw[warp] = incl;
        __syncthreads();
        unsigned wb = 0, tot = 0;
#pragma unroll
        for (int i = 0; i < TK_NW; ++i) {
            const unsigned t = s_gw[i];
            wb += i < warp ? t : 0u;
            tot += t;
        }
        const unsigned ex = wb + incl - cnt;
        unsigned gpos = g32 + (ex & 0xffffu), epos = e32 + (ex >> 16);
#pragma unroll
        for (int u = 0; u < WR_EPT; ++u) {
            const bool isk = (kflag >> u) & 1u, ise = (eflag >> u) & 1u;
            const unsigned kb4 = slow ? gpos + (epos < need32 ? epos : need32) : gpos;
            if (toff) s_kb[tid * WR_EPT + u] = kb4;
            bool keep = isk;
            unsigned pos = kb4;
            if (slow && ise && epos < need32) {
                keep = true;
                pos = gpos + epos;
            }
            if (keep && pos < (unsigned)a.m) {
                oi[pos] = ii[u];
                ov[pos] = vv[u];
                ss = fma((double)vv[u], (double)vv[u], ss);
            }
            gpos += isk;
            epos += ise;
        }
        g32 += tot & 0xffffu;
        e32 += tot >> 16;
        __syncthreads();  // s_gw reuse; s_kb complete
        if (toff) {
            // tiles whose first candidate lies in this chunk: merge offset = kept before it
            for (;;) {
                const int j = jc + tid;
                const bool in = j < nt && (int)s_ts[j] < c1;
                if (in) toff[t0 + j] = (int)s_kb[s_ts[j] - c0];
                const int c = __syncthreads_count(in);
                jc += c;
                if (c < TK_THREADS) break;
            }
        }
    }
    if (toff && last_part) {
        // tiles with no candidate at or after the segment's last entry: offset = kept total
        const unsigned kept = slow ? g32 + (e32 < need32 ? e32 : need32) : g32;
        for (int j = jc + tid; j < nt; j += TK_THREADS) toff[t0 + j] = (int)kept;
        if (tid == 0 && t0 + nt == a.ntiles) toff[a.ntiles] = (int)a.m;
    }
    write_tail<T>(a, ss);
}

// Lane `lane`'s partial of a fixed-order norm reduction: p[lane] + p[lane + 32] + ... in
// ascending order (the order the gate's bits depend on), with the loads of OS_U consecutive
// terms in flight at once -- the last CTA's serial tail was one L2 round trip per term.
constexpr int OS_U = 16;
SG_DEV double lane_ordered_sum(const double* p, int n, int lane) {
    double s = 0.0;
    for (int i0 = lane; i0 < n; i0 += 32 * OS_U) {
        double v[OS_U];
#pragma unroll
        for (int u = 0; u < OS_U; ++u) v[u] = i0 + 32 * u < n ? __ldcg(p + i0 + 32 * u) : 0.0;
#pragma unroll
        for (int u = 0; u < OS_U; ++u)
            if (i0 + 32 * u < n) s = dadd(s, v[u]);
    }
    return s;
}

// k_write: the ordered compaction of every sub-range, then -- in the last CTA to finish --
// the fixed-order norm reductions and the gate (comm.py:129-160), formerly a separate
// one-CTA launch.
template <typename T>
__global__ void __launch_bounds__(TK_THREADS, CW_PER_SM)
k_write(WriteArgs<T> a) {
    pdl_enter();
    SG_STAMP(5);
    write_body<T>(a);
    __shared__ int s_lastw;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __syncthreads();
    SG_MARK(14);
    if (tid == 0) {
        __threadfence();
        s_lastw = atomicAdd(a.done, 1u) == gridDim.x * gridDim.y - 1;
    }
    __syncthreads();
    if (!s_lastw) return;
    __threadfence();
    SG_MARK(15);
    for (int ww = warp; ww < a.k; ww += TK_NW) {
        double sf = lane_ordered_sum(a.pmain + (long long)ww * a.nseg, a.nseg, lane);
        double sk = lane_ordered_sum(a.pwrite + (long long)ww * a.nsub, a.nsub, lane);
        sf = warp_sum(sf);
        sk = warp_sum(sk);
        if (lane == 0) {
            a.norms2[2 * ww] = sf;
            a.norms2[2 * ww + 1] = sk;
            if (a.states) {
                sg_gate_state st = a.states[ww];
                uint8_t d;
                double r;
                gate_math(st, sf, sk, d, r);
                a.states[ww] = st;
                if (a.decision) a.decision[ww] = d;
                if (a.rho) a.rho[ww] = r;
            }
        }
    }
}

// Diagnostics of the last sg_topk_gate call on this workspace, per worker:
// {candidates, boundary entries, fallback pass taken, oversized-tie (slow) write mode}.
template <typename T>
__global__ void k_topk_stats(const SelState<typename KeyOf<T>::K>* sel, const unsigned long long* count,
                             const unsigned long long* bndn, int k, long long* out) {
    pdl_enter();
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= k) return;
    const bool fb = sel[w].mode == MODE_FALLBACK;
    out[4 * w] = (long long)(fb ? count[k + w] : count[w]);
    out[4 * w + 1] = (long long)bndn[w];
    out[4 * w + 2] = fb;
    out[4 * w + 3] = sel[w].wmode == WR_SLOW;
}

__global__ void k_gate_update(const double* norms2, int k, sg_gate_state* states, uint8_t* decision,
                              double* rho) {
    pdl_enter();
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
constexpr size_t MN_SMEM = (size_t)MN_STAGES * MN_TILE * sizeof(float);

// Resident main-pass CTAs per SM, queried once per device (the plan is rebuilt on every call).
inline bool resolve_coop() {  // SG_RESOLVE_COOP=0: k_resolve without the cooperative attribute (A/B runs)
    static const bool on = [] {
        const char* e = getenv("SG_RESOLVE_COOP");
        return !(e && *e == '0');
    }();
    return on;
}

template <typename T> int main_ctas_per_sm() {
    static int cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && cache[dev] > 0) return cache[dev];
    int per_sm = 0;
    cudaError_t e;
    if constexpr (sizeof(T) == 4) {
        smem_attr((const void*)k_main_tma, (int)MN_SMEM);
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_main_tma, TK_THREADS, MN_SMEM);
    } else {
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_main<T>, TK_THREADS, 0);
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        per_sm = sizeof(T) == 4 ? 3 : 4;
    }
    if (per_sm < 1) per_sm = 1;
    if (dev >= 0 && dev < 64) cache[dev] = per_sm;
    return per_sm;
}

// Main-pass segments per worker: a whole number of waves of CTAs over all workers (a partial
// last wave leaves HBM idle in the tail), as many as give segments of ~MAIN_SEG_TILES tiles.
// Real gradients crowd their candidates into a few layers and a candidate-dense segment runs
// ~2x slower than a sparse one; with short segments (4 waves at k = 8) the hardware's CTA
// scheduler evens that out (ResNet-152, k = 8: main pass 0.89 -> 0.38 ms).  At k = 1 one wave
// already gives short segments.
constexpr long long MAIN_SEG_TILES = 64;

template <typename T> int segments_per_worker(int k, long long dim) {
    long long wave = (long long)num_sms() * main_ctas_per_sm<T>() / k;
    if (wave < 1) wave = 1;
    const long long ntiles = (dim + tile_elems<T>() - 1) / tile_elems<T>();
    long long waves = (ntiles + MAIN_SEG_TILES * wave / 2) / (MAIN_SEG_TILES * wave);  // rounded
    if (waves < 1) waves = 1;
    long long s = waves * wave;
    if (s > BMAX) s = BMAX;
    return (int)s;
}

template <typename T>
int topk_gate(const T* g, int k, long long ld, long long dim, long long m, uint32_t* idx, T* val,
              double* norms2, sg_gate_state* states, uint8_t* decision, double* rho, int* tile_off,
              void* ws, size_t ws_bytes, cudaStream_t stream) {
    using K = typename KeyOf<T>::K;
    constexpr int TILE = tile_elems<T>();
    if (!g || !idx || !val || !norms2 || k < 1 || dim < 1 || m < 1 || m > dim || ld < dim)
        return SG_ERR_INVALID;
    if (k > MAX_WORKERS || dim >= (1ll << 31)) return SG_ERR_UNSUPPORTED;
    if (tile_off && TILE != MERGE_TILE) return SG_ERR_INVALID;
    const TopkPlan p = make_plan<T>(k, dim, m, segments_per_worker<T>(k, dim), (long long)num_sms() * CW_PER_SM);
    if (!ws || ws_bytes < p.total) return SG_ERR_WORKSPACE;
    unsigned char* base = reinterpret_cast<unsigned char*>(align_up(reinterpret_cast<size_t>(ws), 256));
    auto at = [&](size_t off) { return base + off; };
    unsigned long long* count = reinterpret_cast<unsigned long long*>(at(p.off_count));
    K* maxkey = reinterpret_cast<K*>(at(p.off_maxkey));
    unsigned* ctr = reinterpret_cast<unsigned*>(at(p.off_ctr));
    unsigned long long* bndn = reinterpret_cast<unsigned long long*>(at(p.off_bndn));
    unsigned* hist0 = reinterpret_cast<unsigned*>(at(p.off_hist0));
    unsigned* hist0fb = reinterpret_cast<unsigned*>(at(p.off_hist0fb));
    unsigned* histr = reinterpret_cast<unsigned*>(at(p.off_histr));
    unsigned long long* status = reinterpret_cast<unsigned long long*>(at(p.off_status));
    SelState<K>* sel = reinterpret_cast<SelState<K>*>(at(p.off_sel));
    unsigned* cnt = reinterpret_cast<unsigned*>(at(p.off_cnt));
    unsigned* tstart = reinterpret_cast<unsigned*>(at(p.off_tstart));
    unsigned* segcnt = reinterpret_cast<unsigned*>(at(p.off_segcnt));
    unsigned* seggt = reinterpret_cast<unsigned*>(at(p.off_seggt));
    unsigned* segbase = reinterpret_cast<unsigned*>(at(p.off_segbase));
    double* pmain = reinterpret_cast<double*>(at(p.off_pmain));
    double* pwrite = reinterpret_cast<double*>(at(p.off_pwrite));
    uint32_t* cidx = reinterpret_cast<uint32_t*>(at(p.off_cidx));
    T* cval = reinterpret_cast<T*>(at(p.off_cval));
    K* bkey = reinterpret_cast<K*>(at(p.off_bkey));
    uint32_t* bidx = reinterpret_cast<uint32_t*>(at(p.off_bidx));
    // counters: [1] write (slow-mode look-back), [8 + w] main done, [8 + k + w] fb done,
    // [8 + 2k + w] collect, [8 + 3k + w * ROUNDS_MAX + r] resolve rounds
    unsigned* c_main = ctr + 8;
    unsigned* c_fb = ctr + 8 + k;
    unsigned* c_col = ctr + 8 + 2 * k;
    unsigned* c_res = ctr + 8 + 3 * k;

    const bool vec_ok = (reinterpret_cast<size_t>(g) % 16 == 0) && ((ld * (long long)sizeof(T)) % 16 == 0);
    const int sms = num_sms();

    // 1. sample (+ zero the small scratch, incl. the slow-mode look-back status words), estimate
    K* samp = reinterpret_cast<K*>(at(p.off_samp));
    K* mm = reinterpret_cast<K*>(at(p.off_mm));
    unsigned* hs1 = reinterpret_cast<unsigned*>(at(p.off_hs1));
    uint4* zero = reinterpret_cast<uint4*>(base + p.zero_begin);
    const long long zero_vec = (long long)((p.zero_end - p.zero_begin) / 16);
    if constexpr (sizeof(K) == 4) {
        if (sample_est_fused()) {
            const int G = se_ctas(k);
            cudaError_t e = smem_attr((const void*)k_sample_est_f32, (int)se_smem(G));
            if (e != cudaSuccess) return e;
            SampleEstArgs sa;
            sa.g = (const float*)g;
            sa.ld = ld;
            sa.dim = dim;
            sa.s_eff = p.s_eff;
            sa.r_est = p.r_est;
            sa.r_hi = p.r_hi;
            sa.vec = (reinterpret_cast<size_t>(g) % 16 == 0) && (ld % 4 == 0) && p.s_eff < dim &&
                     dim / (p.s_eff / SE_CHUNK) >= SE_CHUNK + 4;
            sa.sel = reinterpret_cast<SelState<uint32_t>*>(sel);
            sa.zero = zero;
            sa.zero_vec = zero_vec;
            sa.bkeys = reinterpret_cast<uint32_t*>(samp);
            sa.boff = reinterpret_cast<uint16_t*>(at(p.off_boff));
            sa.h1g = reinterpret_cast<unsigned*>(at(p.off_se_h1));
            sa.mmg = reinterpret_cast<unsigned*>(at(p.off_se_mm));
            sa.doneg = reinterpret_cast<unsigned*>(at(p.off_se_done));
            launch_pdl(k_sample_est_f32, dim3(G, k), dim3(SE_THREADS), se_smem(G), stream, sa);
            debug_sync("k_sample_est", stream);
        } else {
            launch_pdl(k_sample<T>, dim3(EST_G, k), dim3(256), 0, stream, g, ld, dim, p.s_eff, samp, mm, zero, zero_vec,
                       hs1);
            debug_sync("k_sample", stream);
            launch_pdl(k_estimate<T>, dim3(k), dim3(EST_THREADS), 0, stream, dim, p.s_eff, p.r_est,
                       (const K*)samp, (const K*)mm, EST_G, sel, hs1);
            debug_sync("k_estimate", stream);
        }
    } else {
        launch_pdl(k_sample<T>, dim3(EST_G, k), dim3(256), 0, stream, g, ld, dim, p.s_eff, samp, mm, zero, zero_vec, hs1);
        debug_sync("k_sample", stream);
        launch_pdl(k_estimate<T>, dim3(k), dim3(EST_THREADS), 0, stream, dim, p.s_eff, p.r_est,
                   (const K*)samp, (const K*)mm, EST_G, sel, hs1);
        debug_sync("k_estimate", stream);
    }
    // 2. main streaming pass, then the (normally empty) fallback pass
    MainArgs<T> ma;
    ma.g = g;
    ma.ld = ld;
    ma.dim = dim;
    ma.ntiles = p.ntiles;
    ma.m = m;
    ma.segcap = p.segcap;
    ma.k = k;
    ma.vec_ok = vec_ok;
    ma.pass = 0;
    ma.nseg = p.nseg;
    ma.tps = p.tps;
    ma.sel = sel;
    ma.cnt = cnt;
    ma.tstart = tstart;
    ma.segcnt = segcnt;
    ma.cidx = cidx;
    ma.cval = cval;
    ma.pmain = pmain;
    ma.count = count;
    ma.maxkey = maxkey;
    ma.hist0 = hist0;
    ma.done = c_main;
    ma.nsubt = p.nsubt;
    ma.nsub = p.nsub;
    ma.pp = reinterpret_cast<unsigned*>(at(p.off_pp));
    ma.submap = reinterpret_cast<uint4*>(at(p.off_submap));
    ma.dense_thr = mn_dense();
    ma.split_late = 0;
    const dim3 sgrid((unsigned)p.nseg, (unsigned)k);
    bool tma = false;
    if constexpr (sizeof(T) == 4) tma = vec_ok;
    auto launch_main = [&]() {
        if constexpr (sizeof(T) == 4) {
            if (tma) {
                launch_pdl(k_main_tma, dim3(sgrid), dim3(TK_THREADS), MN_SMEM, stream, ma);
                return;
            }
        }
        launch_pdl(k_main<T>, dim3(sgrid), dim3(TK_THREADS), 0, stream, ma);
    };
    launch_main();
    debug_sync("k_main", stream);
    ma.pass = 1;
    ma.hist0 = hist0fb;
    ma.done = c_fb;
    ma.split_late = tma ? 1 : 0;
    // the fallback pass (normally an early exit) is the generic kernel: it also builds the split
    // after the TMA pass.  A small grid striding over the segments: launching a CTA per segment
    // only for them to exit cost ~2 us per step at k = 1
    const unsigned fb_x = (unsigned)(p.nseg < FB_CTAS ? p.nseg : FB_CTAS);
    launch_pdl(k_main<T>, dim3(fb_x, (unsigned)k), dim3(TK_THREADS), 0, stream, ma);
    debug_sync("k_main(fb)", stream);
    // 3. per-segment counts + boundary, in-CTA resolve
    CollectArgs<T> ca;
    ca.segcap = p.segcap;
    ca.cap = TopkTraits<T>::RES;
    ca.nseg = p.nseg;
    ca.tps = p.tps;
    ca.split = p.split;
    ca.nsub = p.nsub;
    ca.nsubt = p.nsubt;
    ca.pp = ma.pp;
    ca.submap = ma.submap;
    ca.bpos = reinterpret_cast<uint32_t*>(at(p.off_bpos));
    ca.sel = sel;
    ca.segcnt = segcnt;
    ca.cidx = cidx;
    ca.cval = cval;
    ca.seggt = seggt;
    ca.segbase = segbase;
    ca.bkey = bkey;
    ca.bidx = bidx;
    ca.bndn = bndn;
    ca.done = c_col;
    const dim3 subgrid((unsigned)p.nsub, (unsigned)k);
    launch_pdl(k_collect<T>, dim3(subgrid), dim3(TK_THREADS), 0, stream, ca);
    debug_sync("k_collect", stream);
    // 4. resolve: in-CTA for the normal boundary, cooperative radix rounds for oversized ones
    const size_t res_smem = (sizeof(K) + 2 * sizeof(uint32_t) + 1) * TopkTraits<T>::RES +
                            sizeof(unsigned) * (NSUB_MAX + 2 * BMAX + 1);
    smem_attr((const void*)k_resolve<T>, (int)res_smem);
    ResolveArgs<T> ra;
    ra.sel = sel;
    ra.hist = histr;
    ra.bar = c_res;
    int gres = sms / k;  // one 1024-thread CTA per SM: the whole grid is co-resident
    if (gres > 16) gres = 16;
    if (gres < 1) gres = 1;
    if (resolve_coop())
        launch_coop(k_resolve<T>, dim3((unsigned)gres, (unsigned)k), dim3(1024), res_smem, stream, ca, ra);
    else  // A/B: a plain PDL launch (the grid still fits the SMs; its barrier needs co-residency)
        launch_pdl(k_resolve<T>, dim3((unsigned)gres, (unsigned)k), dim3(1024), res_smem, stream, ca, ra);
    debug_sync("k_resolve", stream);
    // 5. ordered write + norms + gate
    WriteArgs<T> wa;
    wa.ntiles = p.ntiles;
    wa.segcap = p.segcap;
    wa.m = m;
    wa.k = k;
    wa.nseg = p.nseg;
    wa.tps = p.tps;
    wa.split = p.split;
    wa.nsub = p.nsub;
    wa.nsubt = p.nsubt;
    wa.submap = ma.submap;
    wa.sel = sel;
    wa.tstart = tstart;
    wa.segcnt = segcnt;
    wa.segbase = segbase;
    wa.cidx = cidx;
    wa.cval = cval;
    wa.status = status;
    wa.done = ctr + 1;  // k_write's last-CTA counter (zeroed per call by k_sample)
    wa.idx = idx;
    wa.val = val;
    wa.tile_off = tile_off;
    wa.pwrite = pwrite;
    wa.pmain = pmain;
    wa.norms2 = norms2;
    wa.states = states;
    wa.decision = decision;
    wa.rho = rho;
    // slow mode: the segment's tile starts; float32: then the candidate ring
    wa.ring_off = (unsigned)align_up(sizeof(unsigned) * (size_t)p.tps, 128);
    const size_t wr_smem = sizeof(T) == 4 ? wa.ring_off + WT_RING : align_up(sizeof(unsigned) * (size_t)p.tps, 16);
    smem_attr((const void*)k_write<T>, (int)wr_smem);
    launch_pdl(k_write<T>, dim3(subgrid), dim3(TK_THREADS), wr_smem, stream, wa);
    debug_sync("k_write", stream);
    return cudaGetLastError() == cudaSuccess ? SG_OK : SG_ERR_CUDA;
}

template <typename T>
int topk_stats(int k, long long dim, long long m, const void* ws, size_t ws_bytes, int64_t* out, cudaStream_t stream) {
    using K = typename KeyOf<T>::K;
    if (!ws || !out || k < 1 || dim < 1 || m < 1 || m > dim) return SG_ERR_INVALID;
    const TopkPlan p = make_plan<T>(k, dim, m, segments_per_worker<T>(k, dim), (long long)num_sms() * CW_PER_SM);
    if (ws_bytes < p.total) return SG_ERR_WORKSPACE;
    const unsigned char* base = reinterpret_cast<const unsigned char*>(align_up(reinterpret_cast<size_t>(ws), 256));
    launch_pdl(k_topk_stats<T>, dim3(1), dim3(64), 0, stream, reinterpret_cast<const SelState<K>*>(base + p.off_sel),
                                          reinterpret_cast<const unsigned long long*>(base + p.off_count),
                                          reinterpret_cast<const unsigned long long*>(base + p.off_bndn), k,
                                          reinterpret_cast<long long*>(out));
    return cudaGetLastError() == cudaSuccess ? SG_OK : SG_ERR_CUDA;
}

// The float32 path is the persistent fused kernel (topk_fused.cu).
int topk_fused_f32(const float* g, int k, long long ld, long long dim, long long m, uint32_t* idx, float* val,
                   double* norms2, sg_gate_state* states, uint8_t* decision, double* rho, int* tile_off, void* ws,
                   size_t ws_bytes, int nseg_target, cudaStream_t stream);
size_t topk_fused_workspace_bytes(int k, long long dim, long long m, int nseg_target);
size_t topk_fused_zero_bytes(int k, long long dim, long long m, int nseg_target);
int topk_fused_ctas_per_sm();
int topk_fused_stats(int k, long long dim, long long m, int nseg_target, const void* ws, size_t ws_bytes,
                     int64_t* out, cudaStream_t stream);
int topk_fused_segments(int k, long long dim, long long m, int nseg_target);
int topk_fused_phases(int k, long long dim, long long m, int nseg_target, const void* ws, size_t ws_bytes,
                      unsigned long long* out, long long out_len, cudaStream_t stream);

inline int fused_segments(int k) {
    const int s = num_sms() * topk_fused_ctas_per_sm() / k;
    return s < 1 ? 1 : s;
}

}  // namespace sg

using namespace sg;

SG_STAMPS_EXPORT(sg_diag_stamps_topk)

extern "C" {

size_t sg_topk_workspace_bytes_f32(int k, int64_t dim, int64_t m) {
    if (k < 1 || dim < 1 || m < 1 || m > dim || k > MAX_WORKERS) return 0;
    return make_plan<float>(k, dim, m, segments_per_worker<float>(k, dim), (long long)num_sms() * CW_PER_SM).total;
}

size_t sg_topk_workspace_bytes_fused_f32(int k, int64_t dim, int64_t m) {
    if (k < 1 || dim < 1 || m < 1 || m > dim || k > MAX_WORKERS) return 0;
    return topk_fused_workspace_bytes(k, dim, m, fused_segments(k));
}

size_t sg_topk_workspace_zero_bytes_f32(int k, int64_t dim, int64_t m) {
    // k_sample_est's histogram / key range / arrival counters (restored by every call), plus the
    // slack of the 256-byte base alignment
    if (k < 1 || dim < 1 || m < 1 || m > dim || k > MAX_WORKERS) return 0;
    return make_plan<float>(k, dim, m, segments_per_worker<float>(k, dim), (long long)num_sms() * CW_PER_SM).state_end +
           256;
}

size_t sg_topk_workspace_zero_bytes_fused_f32(int k, int64_t dim, int64_t m) {
    if (k < 1 || dim < 1 || m < 1 || m > dim || k > MAX_WORKERS) return 0;
    return topk_fused_zero_bytes(k, dim, m, fused_segments(k));
}
size_t sg_topk_workspace_bytes_f64(int k, int64_t dim, int64_t m) {
    if (k < 1 || dim < 1 || m < 1 || m > dim || k > MAX_WORKERS) return 0;
    return make_plan<double>(k, dim, m, segments_per_worker<double>(k, dim), (long long)num_sms() * CW_PER_SM).total;
}

int sg_topk_gate_f32(const float* g, int k, int64_t ld, int64_t dim, int64_t m, uint32_t* idx,
                     float* val, double* norms2, sg_gate_state* states, uint8_t* decision,
                     double* rho, int32_t* tile_off, void* workspace, size_t workspace_bytes,
                     void* stream) {
    return topk_gate<float>(g, k, ld, dim, m, idx, val, norms2, states, decision, rho, tile_off,
                            workspace, workspace_bytes, (cudaStream_t)stream);
}

int sg_topk_gate_fused_f32(const float* g, int k, int64_t ld, int64_t dim, int64_t m, uint32_t* idx,
                           float* val, double* norms2, sg_gate_state* states, uint8_t* decision,
                           double* rho, int32_t* tile_off, void* workspace, size_t workspace_bytes,
                           void* stream) {
    if (!g || !idx || !val || !norms2 || k < 1 || dim < 1 || m < 1 || m > dim || ld < dim) return SG_ERR_INVALID;
    if (k > MAX_WORKERS || dim >= (1ll << 31)) return SG_ERR_UNSUPPORTED;
    return topk_fused_f32(g, k, ld, dim, m, idx, val, norms2, states, decision, rho, tile_off, workspace,
                          workspace_bytes, fused_segments(k), (cudaStream_t)stream);
}
int sg_topk_gate_f64(const double* g, int k, int64_t ld, int64_t dim, int64_t m, uint32_t* idx,
                     double* val, double* norms2, sg_gate_state* states, uint8_t* decision,
                     double* rho, void* workspace, size_t workspace_bytes, void* stream) {
    return topk_gate<double>(g, k, ld, dim, m, idx, val, norms2, states, decision, rho, nullptr,
                             workspace, workspace_bytes, (cudaStream_t)stream);
}

int sg_topk_stats_f32(int k, int64_t dim, int64_t m, const void* workspace, size_t workspace_bytes, int64_t* out,
                      void* stream) {
    return topk_stats<float>(k, dim, m, workspace, workspace_bytes, out, (cudaStream_t)stream);
}

int sg_topk_stats_fused_f32(int k, int64_t dim, int64_t m, const void* workspace, size_t workspace_bytes,
                            int64_t* out, void* stream) {
    if (!workspace || !out || k < 1 || dim < 1 || m < 1 || m > dim) return SG_ERR_INVALID;
    return topk_fused_stats(k, dim, m, fused_segments(k), workspace, workspace_bytes, out, (cudaStream_t)stream);
}
int sg_topk_segments_f32(int k, int64_t dim, int64_t m) {
    if (k < 1 || dim < 1 || m < 1 || m > dim || k > MAX_WORKERS) return -1;
    return topk_fused_segments(k, dim, m, fused_segments(k));
}

int sg_topk_phases_f32(int k, int64_t dim, int64_t m, const void* workspace, size_t workspace_bytes, uint64_t* out,
                       int64_t out_len, void* stream) {
    if (!workspace || !out || k < 1 || dim < 1 || m < 1 || m > dim || out_len < 0) return SG_ERR_INVALID;
    return topk_fused_phases(k, dim, m, fused_segments(k), workspace, workspace_bytes,
                             reinterpret_cast<unsigned long long*>(out), out_len, (cudaStream_t)stream);
}

int sg_topk_stats_f64(int k, int64_t dim, int64_t m, const void* workspace, size_t workspace_bytes, int64_t* out,
                      void* stream) {
    return topk_stats<double>(k, dim, m, workspace, workspace_bytes, out, (cudaStream_t)stream);
}

int sg_gate_update(const double* norms2, int k, sg_gate_state* states, uint8_t* decision,
                   double* rho, void* stream) {
    if (!norms2 || !states || k < 1) return SG_ERR_INVALID;
    launch_pdl(k_gate_update, dim3((k + 63) / 64), dim3(64), 0, (cudaStream_t)stream, norms2, k, states, decision, rho);
    return cudaGetLastError() == cudaSuccess ? SG_OK : SG_ERR_CUDA;
}

}  // extern "C"
