// kernels.cuh — non-GEMM kernels of the KRP sketched sum (sm_100a).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "common.cuh"
#include "runtime.hpp"

namespace ts {

// One core block ("atom") of the device-resident formal-sum layout
// (reference src/tucker.cpp:183-226): summand index (for its weight), the block's
// core data offset, its column offset into every stacked factor, and its extents.
struct Atom {
    int summand;
    int pad;
    int64_t core_off;
    int col[kMaxOrder];
    int shape[kMaxOrder];
};

// Stage B (reference src/sketch.cpp:117-131): for every atom b and mode n,
//   W_n[col_b[n] + a, c] = w_b · Σ_J G_b,(n)(a, J) · Π_{j≠n} M_j(col_b[j] + a_j(J), c)
// i.e. the core times the implicit Khatri-Rao product of the M_j slices, with
// M_j stored transposed as Z_j (s × R_j).  The KRP is generated in shared memory
// chunk by chunk and never reaches HBM.
struct KrpArgs {
    const double* Z[kMaxOrder];
    double* W[kMaxOrder];  // Wt_n: s × R_n column-major (transposed W_n)
    int64_t R[kMaxOrder];
    int order;
    int s;
    int natoms;
    const Atom* atoms;
    const double* cores;
    const double* weights;  // per summand
    double* Wpart[kMaxOrder];  // split-J partials (set by launch_krp_contract)
    int splits;
};
void launch_krp_contract(const KrpArgs& args, int max_shape, CallScratch& sc);

// Stage F1 fused for order 3 (ttm3.cu): T_stack[:, col_b[2] + a2] =
// w_b · vec(P_0,b · G_b[:, :, a2] · P_1,bᵀ).  Returns false when the shapes exceed
// the kernel's tile (ranks > 32 or q > 64); the caller then uses the GEMM chain.
struct Ttm3Args {
    const double* P[kMaxOrder];  // P_n (q_n × R_n)
    int64_t q[kMaxOrder];
    const Atom* atoms;
    const double* cores;
    const double* weights;
    double* Tstack;  // Qp × R_2
    int64_t Qp;
    int natoms;
    // Optional: per-row exponent bounds of T_stack (max over all its columns of
    // |T| < 2^e) for stage F2 on the int8 engine: kTtmExpBuckets × Qp ints
    // pre-filled with the floor by launch_fill_exponents (bucket = atom mod 16),
    // folded into the first Qp by launch_reduce_exponents; nullptr = not tracked.
    int* rowexp = nullptr;
};
bool launch_ttm3(const Ttm3Args& args, int max_shape, int max_r2, CallScratch& sc);

// Stage D building blocks: Householder TSQR with the R_ii >= 0 sign convention
// of qr_econ (reference src/kernels.cpp:50-63).
struct QrTask {
    double* A;  // rows × cols block (in/out: Householder vectors below the diagonal)
    int64_t lda;
    int rows, cols;
    double* tau;  // [cols]
    double* R;    // out: min(rows,cols) × cols upper-triangular (ld ldr)
    int64_t ldr;
};
struct QrApplyTask {
    const double* V;  // Householder vectors of the block (rows × kk)
    int64_t ldv;
    const double* tau;
    int rows, kk, q;
    const double* Qin;  // parent piece kk × q (ld ldqin); nullptr → [I; 0]
    int64_t ldqin;
    double* Q;  // out rows × q
    int64_t ldq;
    const double* Rsign;  // top level: flip column c when Rsign[c + c*ldrs] < 0
    int64_t ldrs;
};

// A full TSQR of one tall matrix (rows × cols), planned on the host.
struct TsqrPlan {
    std::vector<std::vector<QrTask>> levels;       // bottom-up factor tasks
    std::vector<std::vector<QrApplyTask>> applies;  // top-down Q-formation tasks
    double* Rtop = nullptr;                        // kk × cols (ld kk)
    int64_t kk = 0;
};
// Builds the plan for `A` (rows × cols, ld lda).  If Q != nullptr the thin Q
// (rows × min(rows,cols), ld ldq) is formed by the apply tasks.
TsqrPlan plan_tsqr(double* A, int64_t lda, int64_t rows, int64_t cols, double* Q, int64_t ldq, CallScratch& sc);
// Runs several plans level-synchronously (factor levels bottom-up, then the
// Q-formation levels top-down), batching the plans' tasks per level.
void run_tsqr(const std::vector<TsqrPlan*>& plans, CallScratch& sc, bool form_q);

// One-sided Jacobi SVD of a small m × nc matrix R in one CTA (stage G).
// Writes sigma[nc] (descending) and U (nc × nc, ld nc): the right singular
// vectors of R, i.e. the left singular vectors of Rᵀ.
void launch_jacobi_svd(const double* R, int64_t ldr, int m, int nc, double* sigma, double* U, CallScratch& sc);

// Two-sided Jacobi eigensolver of a small symmetric n × n matrix (one CTA):
// lambda[n] descending, V (n × n, ld n) matching eigenvectors.
void launch_sym_jacobi(const double* C, int64_t ldc, int n, double* lambda, double* V, CallScratch& sc,
                       int* sweeps = nullptr);
// Fixed-address (permuted-layout) variant for n ≤ 64 (eig.cu); false if n > 64.
bool launch_sym_jacobi_pp(const double* C, int64_t ldc, int n, double* lambda, double* V, CallScratch& sc,
                          int* sweeps);
// `count` independent problems of the same n ≤ 64 (problem b at C + b·strideC,
// lambda + b·strideL, V + b·strideV), one CTA each.  rel_only: rotate on the
// relative criterion only (no absolute floor) — the block one-sided Jacobi of
// wide.cu needs tiny columns orthogonalised too.
bool launch_sym_jacobi_batched(const double* C, int64_t ldc, int n, double* lambda, double* V, CallScratch& sc,
                               int count, int64_t strideC, int64_t strideL, int64_t strideV, bool rel_only,
                               int* sweeps = nullptr);
// TS_EIG=jacobi: stage G uses the Jacobi solver even for n ≤ 64 (A/B timing).
bool jacobi_eig_forced();
// R⁻¹ of the Cholesky factor of small SPD matrices G[b] (n ≤ 96, one CTA each);
// *flag[b] |= 1 on a non-positive pivot, |= 2 when check_identity and
// max|G - I| > 1e-2.
struct CholBatch {
    const double* G[kMaxOrder];
    double* Rinv[kMaxOrder];
    int* flag[kMaxOrder];
    // Device arrays of the same pointers for batches larger than kMaxOrder
    // (segmented sums); when set they replace G / Rinv / flag.
    const double* const* Gd = nullptr;
    double* const* Rd = nullptr;
    int* const* Fd = nullptr;
    int64_t ldg, ldri;
    int n;
    int check_identity;
};
void launch_chol_inv(const CholBatch& cb, int count, CallScratch& sc);
// R-form accuracy check: G = YᵀY, Rinv = R⁻¹; *flag[b] |= 4 when
// trace(G)·‖R⁻¹‖_F² > 1e8 (κ_F(Y) > 1e4).
void launch_rform_check(const CholBatch& cb, int count, CallScratch& sc);
// Device check of the ε = 0 Gram fast path (twin of capi.cu gram_rank): *flag |= 1 on rejection.
void launch_gram_check(const double* lam, int q, int cap, const double* resid, int* flag, CallScratch& sc,
                       int count = 1, int64_t strideL = 0);
// Device check of the ε > 0 Gram fast path with a known output rank `expect`
// (twin of capi.cu gram_rank, θ from the device ‖h‖² *hss): *flag |= 1 on rejection.
void launch_gram_rank_check(const double* lam, int q, int cap, double eps, int order, const double* hss,
                            const double* resid, int expect, int* flag, CallScratch& sc);
// Stage-G eigensolver for n ≤ 64 (eig_trd.cu): Householder tridiagonalisation,
// multisection, inverse iteration, back-transformation, Löwdin
// re-orthonormalisation, all in one CTA.  lambda descending, V (n × n) the
// matching columns; *resid = ‖C V − V Λ‖_F (measured); *flag |= 1 when the
// result is not acceptable (then use launch_sym_jacobi).  False if n > 64.
// count > 1: `count` independent problems, problem b at C + b·strideC,
// lambda + b·strideL, V + b·strideV, flag + b, resid + b (one CTA each).
bool launch_sym_trd(const double* C, int64_t ldc, int n, double* lambda, double* V, int* flag, double* resid,
                    CallScratch& sc, int count = 1, int64_t strideC = 0, int64_t strideL = 0, int64_t strideV = 0);

// Eigenvalues only (descending) of a symmetric n × n matrix, n ≤ 128, one CTA
// (eig_trd.cu): register-resident tridiagonalisation + full-precision
// multisection.  The plan stage's Gram eigenvalues.  False if n > 128.
bool launch_sym_eigvals(const double* C, int64_t ldc, int n, double* lambda, CallScratch& sc);

// X (rest × shape[mode]) = unfold(g, mode)ᵀ for a column-major tensor g.
void launch_unfold_t(const double* g, int order, const int64_t* shape, int mode, double* X, CallScratch& sc);
// Same for `count` tensors of one shape: device pointer arrays gs[count] → Xs[count].
void launch_unfold_t_batched(const double* const* gs, double* const* Xs, int count, int order, const int64_t* shape,
                             int mode, CallScratch& sc);
// out[0] = Σ x_i² (single-CTA, deterministic).
void launch_sumsq(const double* x, int64_t n, double* out, CallScratch& sc);

// out = F·diag(scale) (n × R, ld n) or its transpose (R × n, ld R) when transpose.
void launch_scale_columns(const double* F, int64_t n, int64_t R, const double* scale, double* out, bool transpose,
                          CallScratch& sc);

// out[a] = Σ core(atom a)² (one CTA per atom, deterministic).
void launch_atom_sumsq(const double* cores, const Atom* atoms, int natoms, int order, double* out, CallScratch& sc);

// Kron stage B epilogue (reference src/sketch.cpp:132-140): per atom, the
// sketched block V (column-major; L = Π_{j<n} extents, r = its mode-n extent)
// is unfolded along n, transposed, scaled by its summand's weight and written to
// columns [col, col + r) of Wt_n (C × R_n, C = Π_{j≠n} s_j).
struct KronGather {
    const double* V;
    int64_t L;
    int r;
    int col;
    int summand;
    int pad;
};
void launch_kron_gather(const std::vector<KronGather>& g, int64_t C, double* Wt, const double* weights,
                        CallScratch& sc);

// acc[0] += alpha · <x, y> (single CTA, deterministic; n ≲ 10^6).
void launch_dot_accumulate(const double* x, const double* y, int64_t n, double alpha, double* acc, CallScratch& sc);

// Kron stage B fused for order 3 (kron3.cu): Wt_n for all three modes in one
// launch, one CTA per atom.  Returns false (nothing launched) when a block rank
// exceeds 32 or a mode's sketch width Π_{j≠n} s_j exceeds 96.
struct Kron3Args {
    const double* Z[3];  // Z_j = Ω_jᵀF_j (s_j × R_j)
    double* W[3];        // Wt_n (C_n × R_n)
    int s[3];
    int natoms;
    const Atom* atoms;
    const double* cores;
    const double* weights;
};
bool launch_kron3(const Kron3Args& args, int max_shape, CallScratch& sc);

int max_tsqr_cols();

// ---- ozaki.cu: FP64 C = α·FᵀB + βC on the int8 tcgen05 tensor cores (Ozaki
// splitting into 7 byte digits, int32 TMEM accumulators), out(m, n) at
// C[n + m·ldc].  F: K × M column-major (the stacked factors), its per-column
// exponent bounds aexp[M] (launch_col_exponents, once per upload); B: K × N
// (N ≤ 64) pre-sliced by prepare_ozaki_b.
struct OzOperand {
    uint8_t* slices = nullptr;
    int* exp = nullptr;
    int K = 0, N = 0;
};
struct OzProblem {
    const double* F;
    int64_t ldf;
    const int* aexp;  // per m (a column of F; a row when a_mn)
    int M, K;
    OzOperand B;
    double* C;
    int64_t ldc;
    double alpha = 1.0, beta = 0.0;
    bool a_mn = false;       // F(k, m) stored at F[m + k·ldf] (M contiguous) instead of F[k + m·ldf]
    bool c_colmajor = false;  // out(m, n) at C[m + n·ldc]
};
bool ozaki_enabled();  // TS_OZAKI=0 turns it off (A/B against the DMMA GEMM)
void launch_col_exponents(const double* X, int64_t ld, int64_t rows, int64_t cols, int* out, CallScratch& sc);
// trans: B(k, n) is stored at B[n + k·ldb].
OzOperand prepare_ozaki_b(const double* B, int64_t ldb, int K, int N, CallScratch& sc, bool trans = false);
void launch_row_exponents(const double* X, int64_t ld, int64_t rows, int64_t cols, int* out, CallScratch& sc);
// out[0..n) = the exponent floor (−900) that kernels raise with atomicMax (ttm3.cu).
void launch_fill_exponents(int* out, int64_t n, CallScratch& sc);
constexpr int kOzExpFloor = -900;
constexpr int kTtmExpBuckets = 16;
// e[i] = max_b e[b·n + i] over `buckets` copies.
void launch_reduce_exponents(int* e, int64_t n, int buckets, CallScratch& sc);
// Several small operands in one launch (exponents + slices fused; scratch-owned).
struct OzSmall {
    const double* B;
    int64_t ldb;
    int K, N;
    bool trans;
};
std::vector<OzOperand> prepare_ozaki_b_batch(const std::vector<OzSmall>& reqs, CallScratch& sc);
// Same into caller-owned buffers (slices: ozaki_b_bytes(K) bytes, exp: 64 ints).
size_t ozaki_b_bytes(int K);
void prepare_ozaki_b_into(const double* B, int64_t ldb, int K, int N, const OzOperand& o, CallScratch& sc,
                          bool trans = false);
// False (nothing launched) when a problem does not qualify.
bool launch_ozaki_gemm(const std::vector<OzProblem>& probs, CallScratch& sc, int num_sms, int* launched);

// ---- wide.cu: generic widths (any column count)
// Thin Q (rows × min(rows, cols), ld ldq) of Y (rows × cols, ld ldy; not
// modified): BCGS2 over 64-column TSQR panels for tall Y, the identity for wide Y.
void wide_qr(const double* Y, int64_t ldy, int64_t rows, int64_t cols, double* Q, int64_t ldq, CallScratch& sc,
             int num_sms);
// Block one-sided Jacobi SVD of A (rows × cols, rows ≥ cols, ld lda; not
// modified), cols ≥ 4: sigma[cols] descending and (if V) the right singular
// vectors V (cols × cols, ld ldv).  Host-synchronising (one read per sweep).
// Returns the number of sweeps.
int bosj_svd(const double* A, int64_t lda, int64_t rows, int64_t cols, double* sigma, double* V, int64_t ldv,
             CallScratch& sc, int num_sms);
// Device buffer of the values-kernel phase probe (non-null iff TS_EIG_PROFILE is set).
unsigned long long* eig_probe_buffer();

}  // namespace ts
