// wide.cu — generic-width dense linear algebra: the stage-D thin QR and the
// stage-G / plan singular-value problems for any number of columns, beyond the
// one-CTA kernels (TSQR, Cholesky, Jacobi: ≤ 96 columns held in one SM's
// shared memory).  The reference has no width limit (Eigen HouseholderQR,
// BDCSVD and SelfAdjointEigenSolver at any size: src/kernels.cpp:50-86), so
// KRP widths s > 96, Kron widths Π_{j≠n} s_j > 96, Lazy / Eager stacked ranks
// Σ_k r_n^(k) > 96 and the plan stage's energy-weighted stacks
// (src/sketch.cpp:301-338) land here.  Everything is expressed through the
// grouped DMMA GEMM (gemm.cuh) plus the one-CTA kernels on ≤ 64-column blocks:
//
//  * wide_qr — block classical Gram-Schmidt with reorthogonalisation (BCGS2)
//    over 64-column panels, each panel orthonormalised by the Householder TSQR
//    (kernels.cu) twice: X₁ = (I − QQᵀ)X, Q₁ = tsqr(X₁); X₂ = (I − QQᵀ)Q₁,
//    Q₂ = tsqr(X₂).  The second pass acts on unit columns, so a panel that lies
//    (numerically) in span(Q) — rank-deficient Y — still yields columns
//    orthogonal to Q to working precision: the Householder completion of the
//    reference.  For full-rank Y the result is the unique thin Q with R_ii > 0,
//    i.e. qr_econ's (src/kernels.cpp:50-63) up to roundoff.  Wide Y (rows ≤
//    cols): every orthonormal basis of R^rows spans range(Y); the identity is
//    exact (the sum's factors × core does not depend on the basis).
//
//  * bosj_svd — block one-sided Jacobi (Hestenes) SVD of a tall A: columns in
//    blocks of ≤ 32, a round-robin tournament of block pairs; per round ONE
//    grouped GEMM forms every pair's Gram [A_I A_J]ᵀ[A_I A_J], one batched
//    launch of the two-sided Jacobi eigensolver (eig.cu, relative rotation
//    criterion only) diagonalises them, and ONE grouped GEMM applies the
//    rotations to [A; V], writing the rotated blocks straight into the next
//    round's pair layout (pairs contiguous, so every Gram is one GEMM problem).
//    A sweep ends with the largest normalised pair cosine |a_iᵀa_j|/(‖a_i‖‖a_j‖)
//    (read by the host); σ = the final column norms, V the rotated identity.
//    Rotations are products of Givens rotations, so V is orthogonal to working
//    precision whatever the convergence state.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <vector>

#include "gemm.cuh"
#include "kernels.cuh"
#include "tucksum_cuda.h"

namespace ts {
namespace {

constexpr int kBlk = 32;        // BOSJ block width (pairs ≤ 64 = the eig.cu limit)
constexpr int kPanel = 64;      // wide_qr panel width (TSQR)
constexpr int kMaxBosjSweeps = 40;

// S (ld L, rows + cols rows) ← [A; I] with A's column j placed at column pos[j].
__global__ void bosj_init_kernel(const double* __restrict__ A, int64_t lda, int64_t rows, int cols,
                                 const int* __restrict__ pos, double* __restrict__ S, int64_t L) {
    const int j = blockIdx.y;
    double* dst = S + static_cast<int64_t>(pos[j]) * L;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < L;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double v = 0.0;
        if (i < rows) v = A[i + j * lda];
        else if (i - rows == j) v = 1.0;
        dst[i] = v;
    }
}

// Largest normalised off-diagonal |G_ij| / sqrt(G_ii G_jj) of every pair Gram
// (problem p: G + p·strideG, w_p × w_p, ld ldg) into *out (atomic max on the
// bit pattern: non-negative doubles order like their bits).
__global__ void pair_cosine_kernel(const double* __restrict__ G, int64_t strideG, const int* __restrict__ w,
                                   int ldg, double* __restrict__ out) {
    const int p = blockIdx.x;
    const int n = w[p];
    const double* g = G + p * strideG;
    double mx = 0.0;
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
        const int i = idx % n, j = idx / n;
        if (j <= i) continue;
        const double a = g[i + i * ldg], b = g[j + j * ldg];
        if (a > 0.0 && b > 0.0) mx = fmax(mx, fabs(g[i + j * ldg]) / sqrt(a * b));
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0 && mx > 0.0)
        atomicMax(reinterpret_cast<unsigned long long*>(out), static_cast<unsigned long long>(__double_as_longlong(mx)));
}

// norms[j] = ‖S[0:rows, j]‖₂ (one warp per column, fixed summation order).
__global__ void column_norms_kernel(const double* __restrict__ S, int64_t L, int64_t rows, int cols,
                                    double* __restrict__ norms) {
    const int j = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (j >= cols) return;
    const int lane = threadIdx.x & 31;
    const double* c = S + static_cast<int64_t>(j) * L;
    double s = 0.0;
    for (int64_t i = lane; i < rows; i += 32) s = fma(c[i], c[i], s);
    s = warp_sum(s);
    if (lane == 0) norms[j] = sqrt(s);
}

// sigma[k] = norms[perm[k]], V[:, k] = S[rows : rows + cols, perm[k]].
__global__ void bosj_gather_kernel(const double* __restrict__ S, int64_t L, int64_t rows, int cols,
                                   const int* __restrict__ perm, const double* __restrict__ norms,
                                   double* __restrict__ sigma, double* __restrict__ V, int64_t ldv) {
    const int k = blockIdx.x;
    const int src = perm[k];
    if (threadIdx.x == 0 && sigma) sigma[k] = norms[src];
    if (!V) return;
    const double* c = S + static_cast<int64_t>(src) * L + rows;
    for (int i = threadIdx.x; i < cols; i += blockDim.x) V[i + k * ldv] = c[i];
}

// Q (rows × rows) = I.
__global__ void identity_kernel(double* __restrict__ Q, int64_t ldq, int64_t rows) {
    const int64_t j = blockIdx.y;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < rows;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        Q[i + j * ldq] = i == j ? 1.0 : 0.0;
}

// Round-robin tournament over P players (P even; player P-1 may be a bye):
// round r pairs (r, P-1) and ((r+i) mod (P-1), (r-i) mod (P-1)), i = 1..P/2-1.
std::vector<std::pair<int, int>> round_pairs(int P, int r) {
    std::vector<std::pair<int, int>> out;
    const int m = P - 1;
    out.emplace_back(r % m, P - 1);
    for (int i = 1; i < P / 2; ++i) out.emplace_back((r + i) % m, ((r - i) % m + m) % m);
    return out;
}

}  // namespace

void wide_qr(const double* Y, int64_t ldy, int64_t rows, int64_t cols, double* Q, int64_t ldq, CallScratch& sc,
             int num_sms) {
    cudaStream_t st = sc.stream();
    if (rows <= cols) {  // every orthonormal basis of R^rows spans range(Y)
        identity_kernel<<<dim3(static_cast<unsigned>((rows + 255) / 256), static_cast<unsigned>(rows)), 256, 0, st>>>(
            Q, ldq, rows);
        TS_LAUNCH_CHECK();
        sc.launches += 1;
        return;
    }
    double* X = sc.alloc_n<double>(static_cast<size_t>(rows * kPanel));
    double* Z = sc.alloc_n<double>(static_cast<size_t>(rows * kPanel));
    double* T = sc.alloc_n<double>(static_cast<size_t>(cols * kPanel));
    // (I − Q₀Q₀ᵀ) B in place, Q₀ = Q[:, :done]
    auto project_out = [&](double* B, int64_t done, int64_t pb) {
        GemmProblem p{};
        p.A = Q;
        p.lda = ldq;
        p.B = B;
        p.ldb = rows;
        p.C = T;
        p.ldc = done;
        p.M = static_cast<int>(done);
        p.N = static_cast<int>(pb);
        p.K = static_cast<int>(rows);
        launch_grouped_gemm(Layout::TN, {p}, sc, num_sms);
        GemmProblem u{};
        u.A = Q;
        u.lda = ldq;
        u.B = T;
        u.ldb = done;
        u.C = B;
        u.ldc = rows;
        u.M = static_cast<int>(rows);
        u.N = static_cast<int>(pb);
        u.K = static_cast<int>(done);
        u.alpha = -1.0;
        u.beta = 1.0;
        launch_grouped_gemm(Layout::NN, {u}, sc, num_sms);
    };
    for (int64_t done = 0; done < cols; done += kPanel) {
        const int64_t pb = std::min<int64_t>(kPanel, cols - done);
        TS_CUDA_CHECK(cudaMemcpy2DAsync(X, sizeof(double) * static_cast<size_t>(rows), Y + done * ldy,
                                        sizeof(double) * static_cast<size_t>(ldy), sizeof(double) * static_cast<size_t>(rows),
                                        static_cast<size_t>(pb), cudaMemcpyDeviceToDevice, st));
        double* dst = Q + done * ldq;
        if (done == 0) {
            TsqrPlan plan = plan_tsqr(X, rows, rows, pb, dst, ldq, sc);
            run_tsqr({&plan}, sc, true);
            continue;
        }
        project_out(X, done, pb);
        TsqrPlan p1 = plan_tsqr(X, rows, rows, pb, Z, rows, sc);
        run_tsqr({&p1}, sc, true);
        project_out(Z, done, pb);
        TsqrPlan p2 = plan_tsqr(Z, rows, rows, pb, dst, ldq, sc);
        run_tsqr({&p2}, sc, true);
    }
}

int bosj_svd(const double* A, int64_t lda, int64_t rows, int64_t cols, double* sigma, double* V, int64_t ldv,
             CallScratch& sc, int num_sms) {
    if (cols < 4 || rows < cols) throw Error(TS_INVALID_ARGUMENT, "bosj_svd: need rows >= cols >= 4");
    cudaStream_t st = sc.stream();
    // Blocks of ≤ kBlk columns (at least two), widths differing by at most one.
    const int nb = std::max(2, static_cast<int>((cols + kBlk - 1) / kBlk));
    std::vector<int> bw(static_cast<size_t>(nb));
    for (int i = 0; i < nb; ++i) bw[static_cast<size_t>(i)] = static_cast<int>(cols / nb + (i < cols % nb ? 1 : 0));
    std::vector<int> bstart(static_cast<size_t>(nb) + 1, 0);
    for (int i = 0; i < nb; ++i) bstart[static_cast<size_t>(i) + 1] = bstart[static_cast<size_t>(i)] + bw[static_cast<size_t>(i)];
    const int P = nb + (nb & 1);  // players (a bye when nb is odd)
    const int rounds = std::max(1, P - 1);
    int64_t L = rows + cols;
    L += L & 1;
    // Layout of round r: the pairs' blocks back to back, then the bye.
    auto layout = [&](int r, std::vector<std::pair<int, int>>& pairs, int& bye, std::vector<int64_t>& off) {
        pairs.clear();
        bye = -1;
        off.assign(static_cast<size_t>(nb), 0);
        int64_t o = 0;
        for (auto pr : round_pairs(P, r)) {
            if (pr.first >= nb || pr.second >= nb) {
                bye = pr.first >= nb ? pr.second : pr.first;
                continue;
            }
            pairs.push_back(pr);
            off[static_cast<size_t>(pr.first)] = o;
            o += bw[static_cast<size_t>(pr.first)];
            off[static_cast<size_t>(pr.second)] = o;
            o += bw[static_cast<size_t>(pr.second)];
        }
        if (bye >= 0) off[static_cast<size_t>(bye)] = o;
    };
    double* S0 = sc.alloc_n<double>(static_cast<size_t>(L * cols));
    double* S1 = sc.alloc_n<double>(static_cast<size_t>(L * cols));
    std::vector<std::pair<int, int>> pairs, npairs;
    int bye = -1, nbye = -1;
    std::vector<int64_t> off, noff;
    layout(0, pairs, bye, off);
    {
        std::vector<int> pos(static_cast<size_t>(cols));
        for (int b = 0; b < nb; ++b)
            for (int c = 0; c < bw[static_cast<size_t>(b)]; ++c)
                pos[static_cast<size_t>(bstart[static_cast<size_t>(b)] + c)] = static_cast<int>(off[static_cast<size_t>(b)] + c);
        auto* dpos = static_cast<int*>(sc.upload(pos.data(), sizeof(int) * pos.size()));
        bosj_init_kernel<<<dim3(static_cast<unsigned>(std::min<int64_t>(64, (L + 255) / 256)), static_cast<unsigned>(cols)), 256,
                           0, st>>>(A, lda, rows, static_cast<int>(cols), dpos, S0, L);
        TS_LAUNCH_CHECK();
        sc.launches += 1;
    }
    const int npairs_max = std::max(1, nb / 2);
    double* G = sc.alloc_n<double>(static_cast<size_t>(npairs_max) * 64 * 64);
    double* Vp = sc.alloc_n<double>(static_cast<size_t>(npairs_max) * 64 * 64);
    double* lam = sc.alloc_n<double>(static_cast<size_t>(npairs_max) * 64);
    double* d_cos = sc.alloc_n<double>(kMaxBosjSweeps);
    TS_CUDA_CHECK(cudaMemsetAsync(d_cos, 0, sizeof(double) * kMaxBosjSweeps, st));
    const double tol = std::max(1e-14, 8.0 * 2.220446049250313e-16 * std::sqrt(static_cast<double>(rows)));
    double* cur = S0;
    double* nxt = S1;
    int sweeps = 0;
    {
        for (int sweep = 0; sweep < kMaxBosjSweeps; ++sweep) {
            for (int r = 0; r < rounds; ++r) {
                layout((r + 1) % rounds, npairs, nbye, noff);
                const int np_ = static_cast<int>(pairs.size());
                // Pair Grams (one grouped GEMM), widths w_p = bw_I + bw_J.
                std::vector<GemmProblem> gp;
                std::vector<int> w(static_cast<size_t>(np_));
                for (int p = 0; p < np_; ++p) {
                    const int I = pairs[static_cast<size_t>(p)].first, J = pairs[static_cast<size_t>(p)].second;
                    w[static_cast<size_t>(p)] = bw[static_cast<size_t>(I)] + bw[static_cast<size_t>(J)];
                    GemmProblem g{};
                    g.A = g.B = cur + off[static_cast<size_t>(I)] * L;
                    g.lda = g.ldb = L;
                    g.C = G + static_cast<int64_t>(p) * 64 * 64;
                    g.ldc = 64;
                    g.M = g.N = w[static_cast<size_t>(p)];
                    g.K = static_cast<int>(rows);
                    gp.push_back(g);
                }
                launch_grouped_gemm(Layout::TN, gp, sc, num_sms);
                auto* dw = static_cast<int*>(sc.upload(w.data(), sizeof(int) * w.size()));
                pair_cosine_kernel<<<static_cast<unsigned>(np_), 128, 0, st>>>(G, 64 * 64, dw, 64, d_cos + sweep);
                TS_LAUNCH_CHECK();
                sc.launches += 1;
                // Batched eigensolves, one launch per distinct pair width.
                std::vector<int> widths(w);
                std::sort(widths.begin(), widths.end());
                widths.erase(std::unique(widths.begin(), widths.end()), widths.end());
                for (int wd : widths) {
                    // Pairs of this width are consecutive problems only if sorted;
                    // launch one problem range per run of equal widths.
                    int p = 0;
                    while (p < np_) {
                        if (w[static_cast<size_t>(p)] != wd) {
                            ++p;
                            continue;
                        }
                        int e = p;
                        while (e < np_ && w[static_cast<size_t>(e)] == wd) ++e;
                        launch_sym_jacobi_batched(G + static_cast<int64_t>(p) * 64 * 64, 64, wd,
                                                  lam + static_cast<int64_t>(p) * 64, Vp + static_cast<int64_t>(p) * 64 * 64, sc,
                                                  e - p, 64 * 64, 64, 64 * 64, true);
                        p = e;
                    }
                }
                // Rotations: [A_I A_J; V_I V_J] · Vp → the next round's slots of I and J.
                // (eig.cu writes V with ld = w; the problem stride is 64·64.)
                std::vector<GemmProblem> rp;
                for (int p = 0; p < np_; ++p) {
                    const int I = pairs[static_cast<size_t>(p)].first, J = pairs[static_cast<size_t>(p)].second;
                    const int wp = bw[static_cast<size_t>(I)] + bw[static_cast<size_t>(J)];
                    // The block with the lower id receives the dominant directions
                    // (eigenvalues are descending).  A consistent order matters:
                    // sorting towards whichever block is listed first stalls the
                    // round-robin ordering (measured: no convergence in 40 sweeps).
                    const int lo = std::min(I, J), hi = std::max(I, J);
                    const int wlo = bw[static_cast<size_t>(lo)], whi = bw[static_cast<size_t>(hi)];
                    const double* Vb = Vp + static_cast<int64_t>(p) * 64 * 64;
                    for (int h = 0; h < 2; ++h) {
                        GemmProblem g{};
                        g.A = cur + off[static_cast<size_t>(I)] * L;
                        g.lda = L;
                        g.B = Vb + (h == 0 ? 0 : static_cast<int64_t>(wlo) * wp);
                        g.ldb = wp;
                        g.C = nxt + noff[static_cast<size_t>(h == 0 ? lo : hi)] * L;
                        g.ldc = L;
                        g.M = static_cast<int>(L);
                        g.N = h == 0 ? wlo : whi;
                        g.K = wp;
                        rp.push_back(g);
                    }
                }
                launch_grouped_gemm(Layout::NN, rp, sc, num_sms);
                if (bye >= 0)
                    TS_CUDA_CHECK(cudaMemcpyAsync(nxt + noff[static_cast<size_t>(bye)] * L, cur + off[static_cast<size_t>(bye)] * L,
                                                  sizeof(double) * static_cast<size_t>(L * bw[static_cast<size_t>(bye)]),
                                                  cudaMemcpyDeviceToDevice, st));
                std::swap(cur, nxt);
                pairs.swap(npairs);
                off.swap(noff);
                bye = nbye;
            }
            ++sweeps;
            double c = 0.0;
            TS_CUDA_CHECK(cudaMemcpyAsync(&c, d_cos + sweep, sizeof(double), cudaMemcpyDeviceToHost, st));
            TS_CUDA_CHECK(cudaStreamSynchronize(st));
            static const bool dbg = std::getenv("TS_DEBUG_BOSJ") != nullptr;
            if (dbg) std::fprintf(stderr, "[bosj] rows=%lld cols=%lld sweep %d max cosine %.3e (tol %.1e)\n",
                                  static_cast<long long>(rows), static_cast<long long>(cols), sweep, c, tol);
            if (!(c > tol)) break;  // this sweep found every pair orthogonal (NaN also stops)
        }
    }
    // σ = column norms, descending (ties: current column order), V = rotated identity.
    double* norms = sc.alloc_n<double>(static_cast<size_t>(cols));
    column_norms_kernel<<<static_cast<unsigned>((cols + 7) / 8), 256, 0, st>>>(cur, L, rows, static_cast<int>(cols), norms);
    TS_LAUNCH_CHECK();
    std::vector<double> hn(static_cast<size_t>(cols));
    TS_CUDA_CHECK(cudaMemcpyAsync(hn.data(), norms, sizeof(double) * hn.size(), cudaMemcpyDeviceToHost, st));
    TS_CUDA_CHECK(cudaStreamSynchronize(st));
    std::vector<int> perm(static_cast<size_t>(cols));
    std::iota(perm.begin(), perm.end(), 0);
    std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return hn[static_cast<size_t>(a)] > hn[static_cast<size_t>(b)]; });
    auto* dperm = static_cast<int*>(sc.upload(perm.data(), sizeof(int) * perm.size()));
    bosj_gather_kernel<<<static_cast<unsigned>(cols), 128, 0, st>>>(cur, L, rows, static_cast<int>(cols), dperm, norms,
                                                                   sigma, V, ldv);
    TS_LAUNCH_CHECK();
    sc.launches += 2;
    return sweeps;
}

}  // namespace ts
