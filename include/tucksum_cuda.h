/*
 * tucksum_cuda.h — C ABI of the B200-native KRP sketched Tucker summation.
 *
 * Drop-in boundary for the reference's `krp_sum` hot path (arXiv 2603.13532,
 * reference /root/reference/proj).  Eigen-free, plain pointers and sizes; the
 * C++/Python adapters that restore the reference signatures live above it
 * (paper_2603_13532_b200/tucksum.py).
 *
 * Reference interfaces replaced (paths relative to /root/reference/proj):
 *   ts_tucker_view        ← tucksum::TuckerTensor / CoreBlock storage
 *                           (include/tucksum/tucker.hpp:13-48, src/tucker.cpp:16-79)
 *   ts_batch_upload       ← SumRequest::summands (include/tucksum/sketch.hpp:43-50); the
 *                           device copy uses the formal-sum layout of formal_sum
 *                           (src/tucker.cpp:183-226): per mode one stacked factor matrix
 *   ts_omega_prepare      ← gaussian_matrix(dims[n], s, seed.substream(n))
 *                           (src/kernels.cpp:88-101, src/sketch.cpp:91-95)
 *   ts_krp_sum            ← krp_sum(req, plan, stats) → sketched_sum(krp=true)
 *                           (include/tucksum/sketch.hpp:85-86, src/sketch.cpp:66-181,360-362)
 *   ts_effective_subrank  ← effective_subrank(..., Strategy::Krp, ...) (src/sketch.cpp:272-349)
 *   ts_kron_sum           ← kron_sum(req, plan, stats) → sketched_sum(krp=false)
 *                           (include/tucksum/sketch.hpp:89-90, src/sketch.cpp:66-181,364-366)
 *   ts_effective_subrank_kron ← effective_subrank(..., Strategy::Kron, ...) (src/sketch.cpp:272-349)
 *   ts_kron_sketch_dims   ← kron_sketch_dims (src/sketch.cpp:222-270)
 *   ts_lazy_sum           ← round_sum with Strategy::Lazy = tucker_rounding(formal_sum(...), eps)
 *                           (src/sketch.cpp:48-50, src/tucker.cpp:132-159,285-296)
 *   ts_tucker_norm        ← tucker_norm(formal_sum(...)) (src/tucker.cpp:132-159)
 *   ts_tucker_inner       ← tucker_inner (src/tucker.cpp:161-181), weighted over two batches
 *   ts_rel_error_to_sum   ← tucker_rel_error(x, formal_sum(summands, weights)) (src/tucker.cpp:298-303)
 *   ts_substream          ← RngSeed::substream (include/tucksum/types.hpp:17-24, src/kernels.cpp:23-25)
 *   ts_gaussian_matrix    ← gaussian_matrix (src/kernels.cpp:88-101)
 *   status codes          ← std::invalid_argument / std::runtime_error thrown by
 *                           src/sketch.cpp:16-30,69-71,80-85 (adapters rethrow the same types)
 */
#ifndef TUCKSUM_CUDA_H
#define TUCKSUM_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes. */
#define TS_OK 0
#define TS_INVALID_ARGUMENT 1 /* reference: std::invalid_argument */
#define TS_RUNTIME 2          /* reference: std::runtime_error */
#define TS_CUDA 3
#define TS_NCCL 4
#define TS_OOM 5
#define TS_UNSUPPORTED 6

#define TS_MAX_ORDER 8

typedef struct ts_ctx ts_ctx;
typedef struct ts_batch ts_batch;
typedef struct ts_result ts_result;

/* Borrowed host view of one Tucker tensor (reference TuckerTensor).
 * factors[k]: column-major dims[k] × ranks[k] (ld = dims[k]).
 * Core: num_blocks super-diagonal blocks; block b has offsets
 * block_offsets[b*order + k], extents block_shapes[b*order + k] and
 * column-major data block_data[b] (first index fastest).  A dense core is one
 * block at zero offsets spanning the rank box. */
typedef struct ts_tucker_view {
    int64_t order;
    const int64_t* dims;
    const int64_t* ranks;
    const double* const* factors;
    int64_t num_blocks;
    const int64_t* block_offsets;
    const int64_t* block_shapes;
    const double* const* block_data;
} ts_tucker_view;

/* Last error message of the calling thread (valid until the next call). */
const char* ts_last_error(void);

/* Library version string. */
const char* ts_version(void);

/* ---- context: one per GPU (one CUDA stream, workspace arena, Ω cache) ---- */
int ts_ctx_create(int device, ts_ctx** out);
int ts_ctx_destroy(ts_ctx* ctx);
/* Multi-GPU: join an NCCL communicator of `nranks` ranks (one ctx per GPU).
 * `unique_id` is the 128-byte ncclUniqueId produced by ts_nccl_unique_id on
 * rank 0 and shared by the host (e.g. torch.distributed broadcast).  With a
 * communicator, ts_krp_sum all-reduces the partial sketches Y and the partial
 * projected core h over the ranks; each rank passes its own shard of summands. */
int ts_nccl_unique_id(void* unique_id_128);
int ts_ctx_init_nccl(ts_ctx* ctx, const void* unique_id_128, int nranks, int rank);
/* Alternative to NCCL: the two exchange points of a sharded sum (partial Y after
 * stage C, partial h after stage F) call `fn(user, host_buf, count)`, which must
 * replace host_buf[0..count) by its sum over the `nranks` ranks (e.g. a gloo
 * all-reduce) and return 0.  The library copies the device buffer to the host,
 * calls fn, and copies the sum back.  fn = NULL removes the hook. */
typedef int (*ts_host_allreduce_fn)(void* user, double* host_buf, int64_t count);
int ts_ctx_set_host_allreduce(ts_ctx* ctx, ts_host_allreduce_fn fn, void* user, int nranks, int rank);
/* The communicator's size and this context's rank (ncclCommCount /
 * ncclCommUserRank); 1 / 0 without a communicator. */
int ts_ctx_comm_info(ts_ctx* ctx, int* nranks, int* rank);
/* The CUDA stream (cudaStream_t) the context launches on. */
void* ts_ctx_stream(ts_ctx* ctx);
/* Number of kernels the context launched so far (for the bench's gpu_launches). */
int64_t ts_ctx_launch_count(ts_ctx* ctx);

/* ---- device-resident summand storage ---- */
/* Copies K summands (host memory) to the device in the stacked formal-sum layout. */
int ts_batch_upload(ts_ctx* ctx, const ts_tucker_view* summands, int64_t count, ts_batch** out);
/* The same from data already in the stacked formal-sum layout (reference
 * formal_sum, src/tucker.cpp:183-226, with dense cores): factors[j] is one
 * column-major dims[j] × (Σ_k ranks[k*order + j]) host array per mode (the
 * summands' factors side by side), cores the K dense cores concatenated, each
 * column-major.  One H2D copy per mode + one for the cores. */
int ts_batch_upload_stacked(ts_ctx* ctx, int64_t order, const int64_t* dims, int64_t count, const int64_t* ranks,
                            const double* const* factors, const double* cores, ts_batch** out);
int ts_batch_free(ts_batch* batch);
int64_t ts_batch_count(const ts_batch* batch);
/* Device bytes held by the batch (factors + cores + atom table). */
int64_t ts_batch_bytes(const ts_batch* batch);

/* ---- RNG (bit-identical to the reference's libstdc++ stream) ---- */
void ts_substream(uint64_t seed, uint64_t stream, uint64_t salt, uint64_t* out_seed, uint64_t* out_stream);
int ts_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, uint64_t stream, double* out_colmajor);
/* Generates Ω_n = gaussian_matrix(dims[n], width, {seed, stream}.substream(n)) for
 * n < order on the host and caches them on the device (keyed by seed, stream, dims,
 * width).  ts_krp_sum calls this implicitly; calling it first keeps host Ω
 * generation out of a timed region. */
int ts_omega_prepare(ts_ctx* ctx, int64_t order, const int64_t* dims, int64_t width, uint64_t seed,
                     uint64_t stream);

/* ---- the hot path ---- */
/* krp_sum with the plan given: widths[n] = plan.mode_sketch_dims (uniform width
 * s = max(widths) is used, src/sketch.cpp:86-87).  weights[count] belong to the
 * batch's summands.  eps >= 0 is the st_hosvd tolerance (src/tucker.cpp:239-283).
 * max_rank (nullable, [order], entries <= 0 mean "no cap") is the optional
 * per-mode rank cap of SURVEY.md §8(d); NULL reproduces the reference exactly. */
int ts_krp_sum(ts_ctx* ctx, const ts_batch* batch, const double* weights, const int64_t* widths, uint64_t seed,
               uint64_t stream, double eps, const int64_t* max_rank, ts_result** out);
/* kron_sum with the plan given: Ω_n is
 * dims[n] × widths[n] and the mode-n sketch has C_n = prod_{j != n} widths[j]
 * columns (src/sketch.cpp:91-101,132-140), any size (C_n > 96 takes the
 * generic-width stages of wide.cu).  Other arguments as ts_krp_sum. */
int ts_kron_sum(ts_ctx* ctx, const ts_batch* batch, const double* weights, const int64_t* widths, uint64_t seed,
                uint64_t stream, double eps, const int64_t* max_rank, ts_result** out);
/* Lazy rounding of the formal sum (the paper's deterministic baseline):
 * orthogonalize the stacked factors (thin QR of F_n), absorb R_n into the block
 * cores, st_hosvd(eps [, max_rank]) and Q·P — on the device, through the same
 * stage D-H kernels as ts_krp_sum; stacked ranks sum_k ranks_n^(k) > 96 take
 * the generic-width stages (wide.cu).  Needs order >= 2; not available with a
 * NCCL communicator. */
int ts_lazy_sum(ts_ctx* ctx, const ts_batch* batch, const double* weights, double eps, const int64_t* max_rank,
                ts_result** out);
/* ‖Σ_k w_k X_k‖_F by the reference's orthogonalized-core norm (thin QR of every
 * stacked factor, R absorbed into the block cores): accurate for cancelling
 * sums; any size (as ts_lazy_sum). */
int ts_tucker_norm(ts_ctx* ctx, const ts_batch* batch, const double* weights, double* out);
/* Σ_{a,b} wx_a wy_b <X_a, Y_b> by per-block Gram contractions (the reference's
 * tucker_inner, no densification, any size): one cross-Gram DMMA GEMM per mode
 * plus one stage-F projection per block of x. */
int ts_tucker_inner(ts_ctx* ctx, const ts_batch* x, const double* wx, const ts_batch* y, const double* wy,
                    double* out);
/* ‖r − Σ_k w_k X_k‖ / ‖Σ_k w_k X_k‖ through ts_tucker_inner expansions
 * (‖r‖² − 2<r, S> + ‖S‖²): meant for large sums (config 5); resolves relative
 * errors down to ~1e-6 (fp64 cancellation below that). */
int ts_rel_error_to_sum(ts_ctx* ctx, const ts_result* r, const ts_batch* batch, const double* weights, double* out);
/* Kron widths for per-mode targets (host arithmetic, bit-identical rule). */
int ts_kron_sketch_dims(int64_t order, const int64_t* targets, const int64_t* dims, int64_t* out_widths);
/* Segmented independent sums (one round_sum per NDG
 * node with a shared plan, reference src/ndg.cpp:401-462; the GMRES sums of
 * src/cookie.cpp:389-421): ONE batch holds the summands of `nsums` sums, sum s
 * owning summands [segments[s], segments[s+1]) (segments[0] = 0,
 * segments[nsums] = count, every segment nonempty); weights are per summand;
 * all sums share `widths` (the plan) and `max_rank`; sum s uses the seed
 * {seeds[s], streams[s]}.  out[s] = exactly ts_krp_sum of that segment.  Every
 * stage runs as one launch over all sums (grouped GEMMs over (sum, mode),
 * stage-B / F1 kernels over all atoms, one Cholesky / eigensolver CTA per
 * (sum, mode)), so many small sums cost about what one does. */
int ts_krp_sum_segmented(ts_ctx* ctx, const ts_batch* batch, int64_t nsums, const int64_t* segments,
                         const double* weights, const int64_t* widths, const uint64_t* seeds, const uint64_t* streams,
                         double eps, const int64_t* max_rank, ts_result** out);
/* Independent sums in one call (SURVEY.md §8(f) row 2 — one round_sum per NDG
 * node, many GMRES steps): sum i = krp_sum of batches[i] with weights[i] and the
 * Ω stream (seeds[i], streams[i]); widths / eps / max_rank are shared.  Sums run
 * concurrently on up to `lanes` internal streams (<= 16); each result equals
 * the corresponding ts_krp_sum call bitwise.  out[count] receives owned results
 * (all NULL on error).  Replaces a caller-side loop over tucksum::krp_sum
 * (proj/src/ndg.cpp:401-462, proj/src/cookie.cpp:389-421). */
int ts_krp_sum_many(ts_ctx* ctx, int64_t count, const ts_batch* const* batches, const double* const* weights,
                    const int64_t* widths, const uint64_t* seeds, const uint64_t* streams, double eps,
                    const int64_t* max_rank, int lanes, ts_result** out);
/* Plan stage for Strategy::Krp (src/sketch.cpp:272-349): effective ranks,
 * targets and the uniform widths.  oversampling[order] >= 0. */
int ts_effective_subrank(ts_ctx* ctx, const ts_batch* batch, const double* weights, double eps,
                         const int64_t* oversampling, int64_t* effective_ranks, int64_t* targets, int64_t* widths);
/* Plan stage for Strategy::Kron: same ranks/targets, widths = kron_sketch_dims(targets, dims). */
int ts_effective_subrank_kron(ts_ctx* ctx, const ts_batch* batch, const double* weights, double eps,
                              const int64_t* oversampling, int64_t* effective_ranks, int64_t* targets,
                              int64_t* widths);

/* Small symmetric eigensolver used by ST-HOSVD's fast path (reference sym_eig,
 * src/kernels.cpp:70-86): a (n × n, column-major, host; positive semidefinite
 * for n > 96) → values (descending) and column eigenvectors (host).  n <= 96:
 * one-CTA two-sided Jacobi; n > 96: block one-sided Jacobi (wide.cu).  sweeps /
 * ms (nullable) report the Jacobi sweeps and the time. */
int ts_sym_eig(ts_ctx* ctx, int64_t n, const double* a, double* values, double* vectors, int* sweeps, double* ms);
/* The stage-G default for n <= 64: register-resident Householder
 * tridiagonalisation + multisection + inverse iteration + Löwdin
 * re-orthonormalisation in one CTA (same reference semantics); *flag = 1 when
 * its residual / orthogonality acceptance check failed (the pipeline then falls
 * back to the Jacobi solver of ts_sym_eig). */
int ts_sym_eig_tri(ts_ctx* ctx, int64_t n, const double* a, double* values, double* vectors, int* flag, double* ms);
/* Test hook of the FP64 GEMM on the int8 tensor cores (Ozaki splitting, the
 * stage-A / stage-E engine): out (n_cols × m, column-major, ld n_cols) = Fᵀ·B
 * for host F (k × m) and B (k × n_cols), n_cols <= 64; *ms = kernel time. */
/* Which of the last call's big contractions ran on the int8 tensor-core engine
 * (ozaki.cu; large sums only): bit 0 stage A, bit 1 stage C, bit 2 stage E,
 * bit 3 stage F2. */
int ts_ctx_last_int8_stages(ts_ctx* ctx);
int ts_debug_ozaki_gemm(ts_ctx* ctx, int64_t k, int64_t m, int64_t n_cols, const double* f, const double* b, double* out,
                        double* ms);
/* The same engine in stage C's orientation: out (m × n_cols, column-major) =
 * A·Btᵀ for host A (m × k, column-major) and Bt (n_cols × k), n_cols <= 64. */
int ts_debug_ozaki_gemm_nt(ts_ctx* ctx, int64_t m, int64_t k, int64_t n_cols, const double* a, const double* bt,
                           double* out, double* ms);

/* ---- result: a dense-core Tucker tensor owned by the library ---- */
int64_t ts_result_order(const ts_result* r);
void ts_result_dims(const ts_result* r, int64_t* dims);
void ts_result_ranks(const ts_result* r, int64_t* ranks);
/* Copies (device → host) factor `mode` (dims × ranks, column-major) / the core. */
int ts_result_factor(const ts_result* r, int64_t mode, double* out_host);
int ts_result_core(const ts_result* r, double* out_host);
/* Device pointers (valid until ts_result_free). */
const double* ts_result_factor_device(const ts_result* r, int64_t mode);
const double* ts_result_core_device(const ts_result* r);
/* Stage intermediates kept by the last call when the context has debug capture
 * on (ts_ctx_set_debug): which = 0 Ω_n, 1 Y_n, 2 Û_n, 3 h. Returns element count;
 * rows/cols receive the shape (h: rows = prod(q), cols = 1). */
int64_t ts_result_intermediate(const ts_result* r, int which, int64_t mode, double* out_host, int64_t* rows,
                               int64_t* cols);
int ts_result_free(ts_result* r);

/* Which numerical path the last ts_krp_sum took: number of modes whose thin QR
 * fell back from CholeskyQR2 to Householder TSQR, and number of ST-HOSVD modes
 * whose Gram-eigenvalue decision was not provably exact and used the accurate
 * TSQR + one-sided Jacobi SVD. */
int ts_ctx_last_paths(ts_ctx* ctx, int* qr_fallback_modes, int* svd_fallback_modes);

/* Debug capture of stage intermediates (0/1). */
int ts_ctx_set_debug(ts_ctx* ctx, int enabled);
/* Per-stage CUDA-event times (ms) of the last ts_krp_sum: A, B, C, allreduce Y,
 * D, E, F1, F2, allreduce h, G, H; returns the number written (<= cap). */
int ts_ctx_stage_times(ts_ctx* ctx, double* ms, int cap);
/* CUDA-graph replay of repeated calls (default on): the second identical call
 * (same batch upload, weights, widths, cap, seed; eps == 0) is captured into a
 * graph and later identical calls replay it with one launch.  0 disables it and
 * drops the cache.  ts_ctx_graph_replays counts replays. */
int ts_ctx_set_graphs(ts_ctx* ctx, int enabled);
int64_t ts_ctx_graph_replays(ts_ctx* ctx);
/* Enables per-stage event timing (adds event records; off by default). */
int ts_ctx_set_timing(ts_ctx* ctx, int enabled);

#ifdef __cplusplus
}
#endif

#endif /* TUCKSUM_CUDA_H */
