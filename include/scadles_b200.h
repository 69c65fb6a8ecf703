/*
 * scadles_b200.h — C-ABI of the B200-native ScaDLES gradient-aggregation hot path.
 *
 * The reference (streamsgd, pure Python/numpy) has no FFI: its drop-in surface is the
 * Python module API of `streamsgd.comm` and `streamsgd.nn.sgd_momentum_step`, resolved by
 * the engine as `comm.<fn>` at call time (reference pkg/src/streamsgd/engine.py:18,253-270,
 * 282-283).  Each entry point below replaces one of those functions (cited per entry) and is
 * what a ctypes / cffi binding of that module binds.
 *
 * Conventions
 *   - Every data pointer is a caller-owned DEVICE pointer unless documented as host.
 *   - Nothing is allocated, synchronised or kept in globals.  Scratch comes from a caller
 *     workspace sized by the matching *_workspace_bytes() query.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Return value: SG_OK (0) or a negative SG_ERR_* status; sg_status_string() names it.
 *   - A "bucket" is the flattened per-worker gradient (reference nn.py:122-124):
 *     k worker rows of `dim` elements, row j at base + j*ld.
 *   - Top-k key: NaN sorts below every number, -0 == +0, ties go to the lower index,
 *     kept indices ascending (reference comm.py:90-96).
 */
#ifndef SCADLES_B200_H
#define SCADLES_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SG_ABI_VERSION 2

#define SG_OK 0
#define SG_ERR_INVALID (-1)     /* bad argument (the reference raises ValueError) */
#define SG_ERR_CUDA (-2)        /* a CUDA launch failed */
#define SG_ERR_WORKSPACE (-3)   /* workspace NULL or smaller than the query */
#define SG_ERR_UNSUPPORTED (-4) /* shape outside this build's limits (dim >= 2^31, k > 64) */

/* Per-worker gate state.  Mirrors CompressionState (reference comm.py:99-119); lives in
 * device memory, one per worker, mutated in place by sg_topk_gate_* / sg_gate_update. */
typedef struct sg_gate_state {
    double cr;            /* compression ratio in (0, 1]                         */
    double delta;         /* threshold delta >= 0                                */
    double ewma_factor;   /* in (0, 1); 0.9 by default                          */
    double ewma_full;     /* EWMA of |g|^2                                        */
    double ewma_topk;     /* EWMA of |topk(g)|^2                                  */
    int64_t n_compressed;
    int64_t n_uncompressed;
    int32_t raw_gate;     /* gate on per-iteration norms instead of the EWMAs     */
    int32_t initialized;  /* first call seeds the EWMAs (comm.py:143-146)         */
} sg_gate_state;

int sg_abi_version(void);
const char* sg_status_string(int status);

/* m = max(1, ceil(cr*dim - 1e-12)), host arithmetic; -1 if cr outside (0, 1].
 * Replaces comm.topk_count (comm.py:81-87). */
int64_t sg_topk_count(int64_t dim, double cr);

/* ---- Top-k + squared norms + adaptive gate (items 3 and 4) -------------------------------
 * Replaces comm.topk_sparsify (comm.py:90-96) and comm.compression_gate (comm.py:129-160),
 * batched over the k workers of one GPU.  For worker j:
 *   idx[j*m .. j*m+m)   kept indices, strictly ascending (uint32)
 *   val[j*m .. j*m+m)   g[idx] (copies, bit-exact)
 *   norms2[2j], [2j+1]  s_full = g.g and s_topk = val.val in float64 (deterministic order)
 * If `states` is non-NULL the gate is applied: states[j] is updated exactly as comm.py:143-159
 * (IEEE round-to-nearest, no contraction), decision[j] = 1 iff compressed, rho[j] = ratio.
 * f32 only: if `tile_off` is non-NULL it receives, per worker, the [ceil(dim/4096)+1] merge
 * offsets (number of kept indices below t*4096) that sg_weighted_aggregate_* accepts.
 * `ld` is the row stride in elements; rows must be 16-byte aligned for the vector path
 * (unaligned rows fall back to scalar loads, still on the GPU). */
size_t sg_topk_workspace_bytes_f32(int k, int64_t dim, int64_t m);
size_t sg_topk_workspace_bytes_f64(int k, int64_t dim, int64_t m);
/* Zero-state of a workspace between calls: the first sg_topk_workspace_zero_bytes_f32 bytes
 * (launch chain: the sampler's histogram, key range and arrival counters) or
 * sg_topk_workspace_zero_bytes_fused_f32 bytes (fused variant) must be zero before the first
 * call and whenever (k, dim, m) change; every call leaves them as it found them. */
size_t sg_topk_workspace_zero_bytes_f32(int k, int64_t dim, int64_t m);
/* Persistent float32 variant: the same contract as sg_topk_gate_f32 in ONE cooperative
 * kernel (sample -> estimate -> single read -> select -> ordered write -> gate, synchronised
 * per worker on the device), with a ~2m-entry candidate pool instead of per-segment slots of D
 * (workspace ~16 m + 2 MB per worker). */
size_t sg_topk_workspace_bytes_fused_f32(int k, int64_t dim, int64_t m);
size_t sg_topk_workspace_zero_bytes_fused_f32(int k, int64_t dim, int64_t m);
int sg_topk_gate_fused_f32(const float* g, int k, int64_t ld, int64_t dim, int64_t m,
                           uint32_t* idx, float* val, double* norms2,
                           sg_gate_state* states, uint8_t* decision, double* rho,
                           int32_t* tile_off,
                           void* workspace, size_t workspace_bytes, void* stream);
int sg_topk_stats_fused_f32(int k, int64_t dim, int64_t m, const void* workspace, size_t workspace_bytes,
                            int64_t* out, void* stream);
int sg_topk_gate_f32(const float* g, int k, int64_t ld, int64_t dim, int64_t m,
                     uint32_t* idx, float* val, double* norms2,
                     sg_gate_state* states, uint8_t* decision, double* rho,
                     int32_t* tile_off,
                     void* workspace, size_t workspace_bytes, void* stream);
int sg_topk_gate_f64(const double* g, int k, int64_t ld, int64_t dim, int64_t m,
                     uint32_t* idx, double* val, double* norms2,
                     sg_gate_state* states, uint8_t* decision, double* rho,
                     void* workspace, size_t workspace_bytes, void* stream);

/* Diagnostics of the most recent sg_topk_gate_* call that used `workspace` (same k, dim, m):
 * out[4j..4j+3] (device int64) = {candidates kept by the main pass, boundary entries, fallback
 * pass taken (0/1), oversized-tie write mode (0/1)} for worker j.  (The fused variant's stats:
 * {candidates, boundary entries, estimate undershot (0/1), exact multi-pass fallback (0/1)}.) */
int sg_topk_stats_f32(int k, int64_t dim, int64_t m, const void* workspace, size_t workspace_bytes,
                      int64_t* out, void* stream);
int sg_topk_stats_f64(int k, int64_t dim, int64_t m, const void* workspace, size_t workspace_bytes,
                      int64_t* out, void* stream);

/* Fused-variant diagnostics: segments (CTAs) per worker of the persistent Top-k kernel, and the
 * %globaltimer stamps (ns) of its phases in the last call: out[(w*nseg + s)*16 + i], the phase
 * list in csrc/topk_fused.cu (start, sample, estimate, main pass, selection, write, done). */
int sg_topk_segments_f32(int k, int64_t dim, int64_t m);
int sg_topk_phases_f32(int k, int64_t dim, int64_t m, const void* workspace, size_t workspace_bytes, uint64_t* out,
                       int64_t out_len, void* stream);

/* Gate update alone from precomputed norms2[2k] (comm.py:143-160). */
int sg_gate_update(const double* norms2, int k, sg_gate_state* states,
                   uint8_t* decision, double* rho, void* stream);

/* ---- Weighted aggregation with decompression (item 2 + sparse merge) ----------------------
 * Replaces comm.weighted_aggregate (comm.py:67-78) with densify (comm.py:45-50) folded in:
 *   out = sum_j weights[j] * densify(payload_j), folded in ascending j, float64 round-to-
 *   nearest arithmetic (acc = acc + w_j*x_j, no FMA), rounded once to the output type.
 * Worker j is sparse iff compressed != NULL && compressed[j] != 0 (device bytes); its payload
 * is idx/val[row_ptr[j] .. row_ptr[j+1]) (device int64 row_ptr, indices ascending < dim);
 * `tile_off` ([nw][ceil(dim/4096)+1] int32, row-relative, from sg_topk_gate_f32) may be NULL,
 * in which case it is computed into the workspace.  When `tile_off` is given, worker j's
 * entry count is tile_off[j][last] and only row_ptr[0 .. nw) (the row starts) are read, so
 * the rows may sit apart (e.g. inside a gathered multi-rank buffer).  `dense` may be NULL
 * only if every worker is compressed.
 * Otherwise it is dense: dense + j*ld_dense.  `weights` is a HOST array of nw doubles (the
 * caller passes r = S/sum(S) from comm.weights_from_rates, or 1/n; never batch sizes).
 * With params/momentum_buf non-NULL the momentum-SGD step (nn.py:161-172) is fused into the
 * epilogue using the float64 aggregate: buf = buf*mu + (agg + wd*p); p = p - lr*buf
 * (first_step: buf treated as zeros).  `out` may be NULL when the step is fused. */
size_t sg_aggregate_workspace_bytes(int nw, int64_t dim);
/* `sparse_merge` picks the kernel for an all-sparse float32 merge with fused SGD (launch
 * policy only, no reference counterpart; every choice gives bit-identical results): -1 launches
 * both and the device picks by payload density (>= 0.2 kept entries per position:
 * k_merge_own, else k_merge_ws), 0 only k_merge_ws, 1 only k_merge_own.  A caller that knows
 * its density (GradientExchange: W*m/dim) saves the launch of the kernel that would exit. */
int sg_weighted_aggregate_f32(int nw, const double* weights, const uint8_t* compressed,
                              const float* dense, int64_t ld_dense,
                              const uint32_t* idx, const float* val, const int64_t* row_ptr,
                              const int32_t* tile_off, int64_t dim, float* out,
                              float* params, float* momentum_buf,
                              double lr, double momentum, double weight_decay, int first_step,
                              int sparse_merge, void* workspace, size_t workspace_bytes, void* stream);
int sg_weighted_aggregate_f64(int nw, const double* weights, const uint8_t* compressed,
                              const double* dense, int64_t ld_dense,
                              const uint32_t* idx, const double* val, const int64_t* row_ptr,
                              const int32_t* tile_off, int64_t dim, double* out,
                              double* params, double* momentum_buf,
                              double lr, double momentum, double weight_decay, int first_step,
                              void* workspace, size_t workspace_bytes, void* stream);

/* ---- Multi-GPU merge over peer memory (one process per GPU, NVLink) -----------------------
 * The all-sparse case of sg_weighted_aggregate_f32 with fused momentum SGD, where worker j's
 * payload is addressed by per-worker device pointers that may point into other GPUs' memory
 * (peer-mapped symmetric buffers): idx_ptrs[j] / val_ptrs[j] hold its m ascending entries and
 * tile_off_ptrs[j] its [ceil(dim/4096)+1] merge offsets (from sg_topk_gate_f32), so the
 * payload exchange is fused into the merge (each rank reads the remote entries over NVLink
 * while it streams its parameters).  The three pointer arrays are HOST arrays of nw <= 16
 * device pointers; `compressed` is the (local) device array of nw decision bytes and must be
 * all ones -- the caller checks the decisions first (workers that did not compress are
 * exchanged densely); with a zero byte the kernel writes nothing.  Workers
 * [local_lo, local_lo + local_n) are this device's own (their offsets are scanned to balance the
 * tile ranges; remote ones are not); `sparse_merge` as for sg_weighted_aggregate_f32.  Replaces the
 * comm.weighted_aggregate (comm.py:67-78) + nn.sgd_momentum_step (nn.py:161-172) pair of
 * engine.py:270-283 for the all-compressed iteration. */
int sg_weighted_aggregate_peers_f32(int nw, const double* weights, const uint8_t* compressed,
                                    const uint32_t* const* idx_ptrs, const float* const* val_ptrs,
                                    const int32_t* const* tile_off_ptrs, int64_t dim, float* out,
                                    float* params, float* momentum_buf, double lr, double momentum,
                                    double weight_decay, int first_step, int local_lo, int local_n,
                                    int sparse_merge, void* stream);

/* The dense side of a mixed (or dense-workload) multi-GPU step over peer memory, O(D) NVLink
 * bytes per rank (a ring all-reduce's 2(P-1)/P * 4D), every launch guarded on the gathered
 * decisions `guard[0..guard_n)` (device bytes; a no-op unless some worker did not compress;
 * guard_n = 0: unconditional).  Together they replace the partial + all-reduce + SGD of
 * engine.py:270-283 when decisions are mixed, without a host read of the decisions:
 *   sg_weighted_partial_f32     this rank's workers (dense rows or payloads, the
 *                               sg_weighted_aggregate_f32 argument meaning) folded into `out`,
 *                               the rank's partial (float32);
 *   sg_peer_reduce_slice_f32    position-sharded reduce: rank `rank` owns slice
 *                               [rank*L, min((rank+1)*L, dim)), L = sg_peer_slice_len(dim, P);
 *                               dst[slice] = sum_q w_q * src_q[slice] in ascending q (float64,
 *                               round-to-nearest, rounded once to float32; weights NULL = 1.0).
 *                               src: HOST array of nranks <= 8 device pointers (peers' memory
 *                               allowed, 16-byte aligned); dst may be src[rank];
 *   sg_peer_allgather_sgd_f32   element i's aggregate read from src[owner(i)] (the reduced
 *                               slices), momentum SGD (nn.py:161-172) on the full replica;
 *                               `out` (optional) receives the aggregate; `rank` staggers the
 *                               slice order so the P ranks pull from P different owners. */
int sg_weighted_partial_f32(int nw, const double* weights, const uint8_t* compressed, const float* dense,
                            int64_t ld_dense, const uint32_t* idx, const float* val, const int64_t* row_ptr,
                            const int32_t* tile_off, int64_t dim, float* out, const uint8_t* guard,
                            int guard_n, void* workspace, size_t workspace_bytes, void* stream);
int64_t sg_peer_slice_len(int64_t dim, int nranks);
int sg_peer_reduce_slice_f32(int nranks, const float* const* src, const double* weights, int rank,
                             const uint8_t* guard, int guard_n, int64_t dim, float* dst, void* stream);
/* Reduce-and-push variant: rank `rank`'s reduced slice is written (posted NVLink stores) into
 * every rank's buffer dsts[q] (HOST array of nranks device pointers, peers' memory allowed), so
 * after a barrier every rank holds the full aggregate locally and updates with
 * sg_peer_allgather_sgd_f32(1, &own_buffer, 0, ...). */
int sg_peer_reduce_push_f32(int nranks, const float* const* src, const double* weights, int rank,
                            const uint8_t* guard, int guard_n, int64_t dim, float* const* dsts, void* stream);
/* The whole dense side in ONE cooperative launch per rank: the partial fold of this rank's
 * dense rows (or, dense == NULL, a partial already in partials[rank]), the position-sharded
 * reduce (chunks of 16384 elements round-robin over the ranks) pushed into every rank's
 * aggregate buffer, and the momentum SGD from the local copy, overlapped chunk by chunk and
 * synchronised across GPUs by per-chunk epoch flags (flags[q]: rank q's peer-mapped array of
 * sg_dense_exchange_flag_words(dim, P) zero-initialised words; epoch >= 1, increasing by one per
 * call, identical on every rank).  partials / aggs / flags: HOST arrays of nranks device
 * pointers (peers' memory).  Replaces the partial + all-reduce + SGD of engine.py:270-283. */
/* NVLink SHARP: rank `rank`'s slice (sg_peer_slice_len) of the dense side reduced IN THE
 * SWITCH over every rank's partial (multimem.ld_reduce on the multicast address mc_src of the
 * peer-mapped partial buffers, float32 adds) and broadcast to every rank's aggregate buffer
 * with one multicast store (mc_dst).  After a barrier each rank updates from its own copy
 * (sg_peer_allgather_sgd_f32 with one source).  4D NVLink bytes per rank and direction. */
int sg_nvls_reduce_bcast_f32(int nranks, int rank, const float* mc_src, float* mc_dst, int64_t dim,
                             const uint8_t* guard, int guard_n, void* stream);
size_t sg_dense_exchange_flag_words(int64_t dim, int nranks);
int sg_dense_exchange_f32(int nranks, int rank, int k, const double* weights, const float* dense, int64_t ld,
                          int64_t dim, const float* const* partials, float* const* aggs, unsigned* const* flags,
                          unsigned epoch, const uint8_t* guard, int guard_n, float* out, float* params,
                          float* momentum_buf, double lr, double momentum, double weight_decay, int first_step,
                          void* stream);
int sg_peer_allgather_sgd_f32(int nranks, const float* const* src, int rank, const uint8_t* guard, int guard_n,
                              int64_t dim, float* out, float* params, float* momentum_buf, double lr, double momentum,
                              double weight_decay, int first_step, void* stream);

/* NVLink SHARP payload broadcast: `words` 32-bit words (a multiple of 4, 16-byte aligned) of
 * this rank's packed Top-k output [decisions | idx | val | merge offsets] copied to the multicast
 * address mc_dst of its slot in every rank's peer-mapped gather buffer (multimem.st: one NVLink
 * write per byte, replicated in the switch), so after a barrier every rank merges all W payloads
 * from its own HBM.  Replaces the sparse allgather of engine.py:255-265 / SURVEY §8(e). */
int sg_multicast_copy_u32(const void* src, void* mc_dst, int64_t words, void* stream);

/* Peer barrier of a multi-GPU step over peer-mapped flag words (flags: HOST array of nranks
 * device pointers, rank q's zero-initialised array of slots x nranks unsigned words): this rank
 * publishes `epoch` in every rank's word [slot * nranks + rank] and waits for every rank's epoch
 * in its own words.  epoch == 0: a device counter (*counter) incremented per executed call.  With
 * a guard (the gathered decisions) the call is skipped when every worker compressed (the dense
 * side's barriers).  With dec_dst the ranks' decision bytes (dec_src[q], dec_each each) are
 * gathered after the barrier.  Replaces the per-iteration synchronisation of engine.py:248-286
 * across processes (one launch instead of a collective library barrier plus a gather). */
int sg_peer_signal_wait(int nranks, int rank, unsigned* const* flags, int slot, unsigned epoch, unsigned* counter,
                        const uint8_t* guard, int guard_n, const uint8_t* const* dec_src, int64_t dec_each,
                        uint8_t* dec_dst, void* stream);

/* dst[i * each + b] = src[i][b] for i < nsrc (<= 64 device pointers in a HOST array; peers'
 * memory allowed): gathers the ranks' decision bytes before the host reads them. */
int sg_gather_bytes(int nsrc, const uint8_t* const* src, int64_t each, uint8_t* dst, void* stream);

/* ---- Momentum SGD (nn.sgd_momentum_step, nn.py:161-172) -----------------------------------
 * buf = buf*mu; buf = buf + (g + wd*p); p = p - lr*buf, float64 round-to-nearest per element,
 * in place.  first_step != 0 means the lazily created zero buffer (nn.py:167-168). */
int sg_sgd_momentum_f32(float* params, float* momentum_buf, const float* grad, int64_t dim,
                        double lr, double momentum, double weight_decay, int first_step,
                        void* stream);
int sg_sgd_momentum_f64(double* params, double* momentum_buf, const double* grad, int64_t dim,
                        double lr, double momentum, double weight_decay, int first_step,
                        void* stream);

/* ---- Streaming sampler batch gather (item 5) ----------------------------------------------
 * Replaces the id -> sample map and _materialize (engine.py:223-227, 201-204) plus the
 * injected rows of datagen.inject (datagen.py:182-210).  Row r of the output batch is the
 * train sample rows[r] (device int64, already resolved pools[d][a % len]); features are
 * x[r,:] = train_x[rows[r],:] + augment[rows[r],:] (float64 add, bit-exact), labels copied.
 * rows for all devices are concatenated (CSR by device on the host side). */
int sg_gather_batch_f64(const double* train_x, const double* augment, const int64_t* train_y,
                        int64_t feature_dim, const int64_t* rows, int64_t n_rows,
                        double* x_out, int64_t* y_out, void* stream);
int sg_gather_batch_f32(const float* train_x, const float* augment, const int64_t* train_y,
                        int64_t feature_dim, const int64_t* rows, int64_t n_rows,
                        float* x_out, int64_t* y_out, void* stream);
/* Resolve stream ids to train rows on device: for device d with contiguous drawn ids
 * [head[d], head[d]+b[d]) the row is pool[d][(head[d]+i) % pool_len[d]] (engine.py:223-227);
 * out is CSR by device (out_ptr[d] .. out_ptr[d]+b[d]); pools are CSR (pool_ptr, pool_rows). */
int sg_resolve_stream_rows(int n_dev, const int64_t* head, const int64_t* b,
                           const int64_t* out_ptr, const int64_t* pool_ptr,
                           const int64_t* pool_rows, int64_t total, int64_t* out,
                           void* stream);
/* Non-IID injection (datagen.py:182-210): recipient d's batch is its own rows
 * base_rows[base_ptr[d] .. base_ptr[d+1]) followed, for every plan entry k whose sender
 * senders[k] != d (plan order = ascending sender), by the sender's rows at the pick
 * positions picks[pick_ptr[k] .. pick_ptr[k+1]) (positions into the sender's pre-injection
 * batch, drawn on the host with the reference's numpy RNG).  out_ptr is the CSR of the
 * augmented batches (host-computed sizes). */
int sg_inject_rows(int n_dev, const int64_t* base_ptr, const int64_t* base_rows, int n_send,
                   const int32_t* senders, const int64_t* pick_ptr, const int64_t* picks,
                   const int64_t* out_ptr, int64_t* out_rows, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SCADLES_B200_H */
