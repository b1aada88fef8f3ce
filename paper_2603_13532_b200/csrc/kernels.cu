// kernels.cu — stage D (TSQR, CholeskyQR), stage G (Jacobi SVD / eigensolver,
// unfolding) kernels for sm_100a.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <stdexcept>

#include "../../include/tucksum_cuda.h"
#include "kernels.cuh"

namespace ts {
namespace {

// ------------------------------------------------------------------ TSQR
constexpr int kQrThreads = 512;
constexpr int kQrWarps = kQrThreads / 32;
constexpr int kQrMaxCPW = 6;  // columns per warp: 96 / 16

// Householder parameters with Eigen's makeHouseholder convention: beta =
// -sign(c0)·‖x‖, tau = (beta - c0)/beta, v = [1; x_tail/(c0 - beta)]; tau = 0
// when the tail is below the smallest normal (see oracle/tucksum_oracle.cpp).
// sqrt / reciprocal from the MUFU approximations plus Newton steps (≤ 1 ulp):
// no IEEE div/sqrt slow-path call sites, which would force the register-resident
// TSQR block out to local memory around every call.
__device__ __forceinline__ double nr_rcp(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    y = y * fma(-x, y, 2.0);
    y = y * fma(-x, y, 2.0);
    return fma(y, fma(-x, y, 1.0), y);
}
__device__ __forceinline__ double nr_sqrt(double x) {
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    r = r * fma(-0.5 * x, r * r, 1.5);
    r = r * fma(-0.5 * x, r * r, 1.5);
    const double s = x * r;
    return fma(0.5 * r, fma(-s, s, x), s);  // one Newton step on s = √x
}

__device__ __forceinline__ void householder_params(double c0, double tail, double* beta, double* tau, double* inv) {
    if (tail <= DBL_MIN) {
        *tau = 0.0;
        *beta = c0;
        *inv = 0.0;
    } else {
        double b = nr_sqrt(fma(c0, c0, tail));
        if (c0 >= 0.0) b = -b;
        *beta = b;
        *inv = nr_rcp(c0 - b);
        *tau = (b - c0) * nr_rcp(b);
    }
}

// Householder QR of one rows × cols block (rows ≤ 256, cols ≤ 96), register
// resident: warp w owns columns w, w+16, …, w+80; lane l owns rows l, l+32, …, so
// the trailing update needs no shared-memory traffic except the reflector
// itself.  Step k: the owner warp of column k forms the reflector (Eigen's
// makeHouseholder convention, see householder_params) and publishes the scaled
// vector v = [1; x·inv] through a double-buffered shared array; after ONE
// barrier every warp applies H_k = I − τ·v·vᵀ to its own columns j > k.
constexpr int kQrFThreads = 512;  // factor kernel: 16 warps; ≤ 8 rows per lane (256-row blocks), ≤ 6 column slots (96 cols)
constexpr int kQrFWarps = kQrFThreads / 32;

// RPL rows per lane (32·RPL rows per block), CPW column slots per warp (16·CPW
// columns): instantiated for the launch's largest block so small blocks (the
// 64-row sketches of short modes, the last TSQR levels) carry no dead rows.
template <int RPL, int CPW>
__global__ void __launch_bounds__(kQrFThreads) tsqr_factor_kernel(const QrTask* __restrict__ tasks) {
    const QrTask tk = tasks[blockIdx.x];
    const int rows = tk.rows, cols = tk.cols, kk = min(rows, cols);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __shared__ __align__(16) double vbuf[2][RPL * 32];
    __shared__ double s_tau[2];
    double a[CPW][RPL];
#pragma unroll
    for (int i = 0; i < CPW; ++i) {
        const int c = warp + kQrFWarps * i;
        const double* __restrict__ col = tk.A + static_cast<int64_t>(c < cols ? c : 0) * tk.lda + lane;
#pragma unroll
        for (int t = 0; t < RPL; ++t)
            a[i][t] = (c < cols && lane + 32 * t < rows) ? __ldg(col + 32 * t) : 0.0;
    }
    for (int k = 0; k < kk; ++k) {
        const int buf = k & 1;
        const int ow = k % kQrFWarps, oi = k / kQrFWarps;  // owner warp / slot of column k
        if (warp == ow) {
            // Column k = slot oi (run-time) of this warp, read and written through
            // selects so every register index stays static (no local memory).
            auto col = [&](int t) {
                double v = a[0][t];
#pragma unroll
                for (int i = 1; i < CPW; ++i) v = i == oi ? a[i][t] : v;
                return v;
            };
            double tail = 0.0, c0 = 0.0;
#pragma unroll
            for (int t = 0; t < RPL; ++t) {
                const int r = lane + 32 * t;
                const double v = col(t);
                if (r > k && r < rows) tail = fma(v, v, tail);
                if (r == k) c0 = v;
            }
            tail = warp_sum(tail);
            c0 = __shfl_sync(0xffffffffu, c0, k & 31);
            double beta, tau, inv;
            householder_params(c0, tail, &beta, &tau, &inv);
#pragma unroll
            for (int t = 0; t < RPL; ++t) {
                const int r = lane + 32 * t;
                const double xv = col(t);
                double v = 0.0, nv = xv;
                if (r == k) {
                    v = 1.0;
                    nv = beta;  // R_kk
                } else if (r > k && r < rows) {
                    v = tau == 0.0 ? 0.0 : xv * inv;
                    nv = v;  // Householder vector below the diagonal
                }
                vbuf[buf][r] = v;
#pragma unroll
                for (int i = 0; i < CPW; ++i) a[i][t] = i == oi ? nv : a[i][t];
            }
            if (lane == 0) {
                s_tau[buf] = tau;
                tk.tau[k] = tau;
            }
        }
        __syncthreads();
        const double tau = s_tau[buf];
        if (tau != 0.0) {
            const double* vb = vbuf[buf] + lane;  // v is 0 above row k
            // All owned columns' dot products first, then one interleaved
            // reduction (their shuffle latencies overlap), then the updates.
            double dot[CPW];
#pragma unroll
            for (int i = 0; i < CPW; ++i) {
                dot[i] = 0.0;
#pragma unroll
                for (int t = 0; t < RPL; ++t) dot[i] = fma(vb[32 * t], a[i][t], dot[i]);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int i = 0; i < CPW; ++i) dot[i] += __shfl_xor_sync(0xffffffffu, dot[i], o);
#pragma unroll
            for (int i = 0; i < CPW; ++i) {
                const int c = warp + kQrFWarps * i;
                const double w = (c > k && c < cols) ? tau * dot[i] : 0.0;  // columns ≤ k are final
#pragma unroll
                for (int t = 0; t < RPL; ++t) a[i][t] = fma(-w, vb[32 * t], a[i][t]);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < CPW; ++i) {
        const int c = warp + kQrFWarps * i;
        if (c >= cols) continue;
        double* __restrict__ colA = tk.A + static_cast<int64_t>(c) * tk.lda + lane;
        double* __restrict__ colR = tk.R + static_cast<int64_t>(c) * tk.ldr + lane;
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
            const int r = lane + 32 * t;
            if (r < rows) colA[32 * t] = a[i][t];
            if (r < kk) colR[32 * t] = r <= c ? a[i][t] : 0.0;
        }
    }
}

// Q formation for one block: Q = H_0 ⋯ H_{kk-1} · [Qin; 0], optional column
// signs.  Reflector k-1 is prefetched (cp.async) while reflector k is applied.
template <int CPW>  // column slots per warp (16·CPW columns of Q)
__global__ void __launch_bounds__(kQrThreads) tsqr_apply_kernel(const QrApplyTask* __restrict__ tasks) {
    const QrApplyTask tk = tasks[blockIdx.x];
    const int rows = tk.rows, kk = tk.kk, q = tk.q;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    extern __shared__ __align__(16) double Qs[];
    double* vbuf = Qs + rows * q;      // 2 × rows
    double* taus = vbuf + 2 * rows;    // kk
    const unsigned Qb = smem_u32(Qs);
    for (int idx = tid; idx < rows * q; idx += kQrThreads) {
        const int i = idx % rows, c = idx / rows;
        double val = 0.0;
        if (i < kk) val = tk.Qin ? tk.Qin[i + static_cast<int64_t>(c) * tk.ldqin] : (i == c ? 1.0 : 0.0);
        Qs[idx] = val;
    }
    for (int i = tid; i < kk; i += kQrThreads) taus[i] = tk.tau[i];
    if (kk > 0)
        for (int i = kk + tid; i < rows; i += kQrThreads)
            cp_async8(vbuf + ((kk - 1) & 1) * rows + i, tk.V + i + static_cast<int64_t>(kk - 1) * tk.ldv, 8);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    for (int k = kk - 1; k >= 0; --k) {
        if (k > 0)
            for (int i = k + tid; i < rows; i += kQrThreads)
                cp_async8(vbuf + ((k - 1) & 1) * rows + i, tk.V + i + static_cast<int64_t>(k - 1) * tk.ldv, 8);
        cp_async_commit();
        const double tau = taus[k];
        if (tau != 0.0) {
            // Explicit shared addresses (see tsqr_factor_kernel).
            const unsigned vb = Qb + 8u * static_cast<unsigned>(rows * q + (k & 1) * rows);
            int nc = 0;
            unsigned cb[CPW];
#pragma unroll
            for (int i = 0; i < CPW; ++i) {
                const int c = warp + kQrWarps * i;
                if (c < q) nc = i + 1;
                cb[i] = Qb + 8u * static_cast<unsigned>((c < q ? c : 0) * rows);
            }
            double dot[CPW];
#pragma unroll
            for (int i = 0; i < CPW; ++i) dot[i] = 0.0;
            for (int r = k + 1 + lane; r < rows; r += 32) {
                const double vr = lds64(vb + 8u * r);
#pragma unroll
                for (int i = 0; i < CPW; ++i)
                    if (i < nc) dot[i] = fma(vr, lds64(cb[i] + 8u * r), dot[i]);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int i = 0; i < CPW; ++i) dot[i] += __shfl_xor_sync(0xffffffffu, dot[i], o);
            double w[CPW];
#pragma unroll
            for (int i = 0; i < CPW; ++i) w[i] = i < nc ? tau * (lds64(cb[i] + 8u * k) + dot[i]) : 0.0;
            for (int r = k + 1 + lane; r < rows; r += 32) {
                const double vr = lds64(vb + 8u * r);
#pragma unroll
                for (int i = 0; i < CPW; ++i)
                    if (i < nc) sts64(cb[i] + 8u * r, lds64(cb[i] + 8u * r) - w[i] * vr);
            }
            __syncwarp();
            if (lane == 0)
#pragma unroll
                for (int i = 0; i < CPW; ++i)
                    if (i < nc) sts64(cb[i] + 8u * k, lds64(cb[i] + 8u * k) - w[i]);
        }
        cp_async_wait<0>();
        __syncthreads();
    }
    for (int idx = tid; idx < rows * q; idx += kQrThreads) {
        const int i = idx % rows, c = idx / rows;
        double val = Qs[idx];
        if (tk.Rsign && tk.Rsign[c + static_cast<int64_t>(c) * tk.ldrs] < 0.0) val = -val;
        tk.Q[i + static_cast<int64_t>(c) * tk.ldq] = val;
    }
}

// ------------------------------------------------------------------ Jacobi
constexpr int kJacThreads = 1024;
constexpr int kJacWarps = kJacThreads / 32;

__device__ __forceinline__ double rcp_approx(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return y;
}
__device__ __forceinline__ double rsqrt_approx(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return y;
}

// Jacobi rotation (c, s) for [[a, g], [g, b]] (the reference formula of the
// oracle's sym_eig / one-sided Jacobi): θ = (b - a)/(2g), t = sign(θ)/(|θ| +
// sqrt(1 + θ²)), c = 1/sqrt(1 + t²), s = t·c.  The rounds of a Jacobi sweep are
// sequential, so this chain is the solver's critical path: t is formed with the
// ~20-bit MUFU approximations (an angle that annihilates g to ~1e-6 relative is
// all the iteration needs), while c is Newton-refined to full precision so every
// applied rotation is orthogonal to working accuracy (c² + s² = 1 ± 1 ulp).
__device__ __forceinline__ void jacobi_rotation(double a, double b, double g, double& c, double& s, double& t) {
    const double theta = (b - a) * rcp_approx(2.0 * g);
    const double at = fabs(theta);
    if (at > 1e150) {
        t = 0.5 * rcp_approx(theta);
    } else {
        const double u = fma(theta, theta, 1.0);
        const double sq = u * rsqrt_approx(u);
        t = copysign(rcp_approx(at + sq), theta);
    }
    const double w = fma(t, t, 1.0);
    double r = rsqrt_approx(w);
    r = r * fma(-0.5 * w, r * r, 1.5);
    r = r * fma(-0.5 * w, r * r, 1.5);
    c = r;
    s = t * c;
}

__device__ __forceinline__ void pair_of(int r, int pi, int np, int* p, int* q) {
    // r < np - 1 and pi < np / 2, so one conditional wrap replaces the modulo
    // (an integer division on the round's critical path).
    int a, b;
    if (pi == 0) {
        a = np - 1;
        b = r;
    } else {
        a = r + pi;
        if (a >= np - 1) a -= np - 1;
        b = r - pi;
        if (b < 0) b += np - 1;
    }
    *p = min(a, b);
    *q = max(a, b);
}

// Writes sigma/U sorted by descending key (stable): U[:, rank(c)] = J[:, c].
__device__ void sort_desc_store(const double* key, const double* J, int nc, double* sigma, double* U) {
    for (int c = threadIdx.x; c < nc; c += blockDim.x) {
        const double v = key[c];
        int rank = 0;
        for (int i = 0; i < nc; ++i) rank += (key[i] > v) || (key[i] == v && i < c);
        sigma[rank] = v;
        for (int i = 0; i < nc; ++i) U[i + static_cast<int64_t>(rank) * nc] = J[i + c * nc];
    }
}

// One-sided (Hestenes) Jacobi SVD of a small m × nc matrix R (accurate path).
// One column pair per warp per round (round-robin ordering); squared column
// norms are carried through the rotations so each pair needs one reduction.
__global__ void __launch_bounds__(kJacThreads) jacobi_svd_kernel(const double* __restrict__ R, int64_t ldr, int m,
                                                                 int nc, double* __restrict__ sigma,
                                                                 double* __restrict__ U,
                                                                 unsigned long long* __restrict__ prof) {
    extern __shared__ __align__(16) double sm[];
    double* W = sm;             // m × nc (ld m)
    double* J = W + m * nc;     // nc × nc (ld nc)
    double* nrm = J + nc * nc;  // nc (squared norms, then norms)
    __shared__ int rotated;
    __shared__ double maxn;
    const unsigned Wb = smem_u32(W), Jb = smem_u32(J);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int idx = tid; idx < m * nc; idx += kJacThreads) {
        const int i = idx % m, c = idx / m;
        W[idx] = R[i + static_cast<int64_t>(c) * ldr];
    }
    for (int idx = tid; idx < nc * nc; idx += kJacThreads) J[idx] = (idx % nc == idx / nc) ? 1.0 : 0.0;
    const int np = nc + (nc & 1);
    const double tol = 1e-15;
    for (int sweep = 0; sweep < 30; ++sweep) {  // LAPACK dgesvj caps at 30 sweeps
        __syncthreads();
        for (int c = warp; c < nc; c += kJacWarps) {  // exact norms once per sweep
            double a = 0.0;
            for (int i = lane; i < m; i += 32) a = fma(W[i + c * m], W[i + c * m], a);
            a = warp_sum(a);
            if (lane == 0) nrm[c] = a;
        }
        if (tid == 0) {
            rotated = 0;
            double mx = 0.0;
            for (int c = 0; c < nc; ++c) mx = fmax(mx, nrm[c]);
            maxn = mx;
        }
        __syncthreads();
        // Pairs whose coupling is below (1e-15·max‖w_c‖)² are left alone: they
        // move singular values by less than 1e-15·σ₁ (under the reference's own
        // accuracy and the 1e-14·σ₁ rank floor), and rotating them only churns
        // the rounding-noise subspace of rank-deficient inputs sweep after sweep.
        const double abs_floor = 1e-30 * maxn;
        for (int r = 0; r < np - 1; ++r) {
            for (int pi = warp; pi < np / 2; pi += kJacWarps) {
                int p, q;
                pair_of(r, pi, np, &p, &q);
                if (q >= nc) continue;
                // Explicit shared addresses (run-time column offsets into the
                // extern array otherwise re-derive its window base per access).
                const unsigned wp = Wb + 8u * static_cast<unsigned>(p * m), wq = Wb + 8u * static_cast<unsigned>(q * m);
                double ga = 0.0;
                for (int i = lane; i < m; i += 32) ga = fma(lds64(wp + 8u * i), lds64(wq + 8u * i), ga);
                ga = warp_sum(ga);
                const double al = nrm[p], be = nrm[q];
                // Also skip when either column is itself below 1e-15·σ₁: such a
                // column is rounding noise of a rank-deficient input (its σ falls
                // under the 1e-14·σ₁ rank floor whatever its direction), and
                // rotating it against a signal column only re-randomises it —
                // every sweep would find O(1) relative coupling again.
                if (ga == 0.0 || ga * ga <= (tol * tol) * (al * be) || fabs(ga) <= abs_floor ||
                    fmin(al, be) <= abs_floor)
                    continue;
                double c, s, t;
                jacobi_rotation(al, be, ga, c, s, t);
                for (int i = lane; i < m; i += 32) {
                    const double x = lds64(wp + 8u * i), y = lds64(wq + 8u * i);
                    sts64(wp + 8u * i, c * x - s * y);
                    sts64(wq + 8u * i, s * x + c * y);
                }
                const unsigned jp = Jb + 8u * static_cast<unsigned>(p * nc), jq = Jb + 8u * static_cast<unsigned>(q * nc);
                for (int i = lane; i < nc; i += 32) {
                    const double x = lds64(jp + 8u * i), y = lds64(jq + 8u * i);
                    sts64(jp + 8u * i, c * x - s * y);
                    sts64(jq + 8u * i, s * x + c * y);
                }
                __syncwarp();
                if (lane == 0) {
                    nrm[p] = al - t * ga;
                    nrm[q] = be + t * ga;
                    rotated = 1;
                }
            }
            __syncthreads();
        }
        if (!rotated) {
            if (prof != nullptr && tid == 0) prof[16] = static_cast<unsigned long long>(sweep + 1);
            break;
        }
    }
    __syncthreads();
    for (int c = warp; c < nc; c += kJacWarps) {
        double a = 0.0;
        for (int i = lane; i < m; i += 32) a = fma(W[i + c * m], W[i + c * m], a);
        a = warp_sum(a);
        if (lane == 0) nrm[c] = sqrt(a);
    }
    __syncthreads();
    sort_desc_store(nrm, J, nc, sigma, U);
}

// Two-sided cyclic Jacobi eigensolver for a small symmetric n × n matrix C
// (fast path of ST-HOSVD on the Gram of an unfolding), one CTA.
//
// The matrix is padded to an even order np and each round rotates the np/2
// disjoint pairs of a round-robin tournament (players a, b meet in round R iff
// a + b ≡ 2R mod (np-1); the last player meets R).  A round is ONE pass and ONE
// barrier: every thread owns upper-triangular 2×2 blocks A[P_i, P_j] of the pair
// grid and applies R_iᵀ·A[P_i,P_j]·R_j (plus the mirror block), updates its
// eigenvector items, and — when its block holds the next round's pair (x, y) —
// immediately derives that pair's rotation from the rotated entries (the new
// diagonal entries follow in closed form from the pairs' saved 2×2 blocks).
// The rotation-parameter latency thus overlaps the block updates instead of
// costing a separate phase and barrier.
__global__ void __launch_bounds__(kJacThreads) sym_jacobi_kernel(const double* __restrict__ Cin, int64_t ldc, int n,
                                                                 double* __restrict__ lambda, double* __restrict__ V,
                                                                 int* __restrict__ sweeps_out) {
    extern __shared__ __align__(16) double sm[];
    const int np = n + (n & 1);
    const int npair = np / 2;
    const int m = np - 1;
    const int ld = np + 1;                        // padded row stride
    double* A = sm;                               // np × ld
    double* Vs = A + np * ld;                     // np × ld, Vs[k*ld + j] = V(k, j)
    double2* cs = reinterpret_cast<double2*>(Vs + np * ld);  // [2][npair] (c, s)
    double* dg = reinterpret_cast<double*>(cs + 2 * npair);   // [2][npair][3] (a_pp, a_qq, a_pq)
    double* diag = dg + 6 * npair;                            // np
    __shared__ int stop;
    __shared__ double red[2 * kJacWarps];
    __shared__ double prev_off, amax_s;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int idx = tid; idx < np * np; idx += kJacThreads) {
        const int i = idx % np, j = idx / np;
        double v = 0.0;
        if (i < n && j < n) v = 0.5 * (Cin[i + static_cast<int64_t>(j) * ldc] + Cin[j + static_cast<int64_t>(i) * ldc]);
        A[i * ld + j] = v;
        Vs[i * ld + j] = (i == j) ? 1.0 : 0.0;
    }
    if (tid == 0) {
        amax_s = 0.0;
        prev_off = 0.0;
        stop = 0;
    }
    __syncthreads();
    {
        double mx = 0.0;
        for (int i = tid; i < n; i += kJacThreads) mx = fmax(mx, fabs(A[i * ld + i]));
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0 && mx > 0.0) atomicMax(reinterpret_cast<unsigned long long*>(&amax_s), __double_as_longlong(mx));
    }
    __syncthreads();
    // Entries below 1e-15·max|a_ii| sit under the Gram's own rounding noise (the
    // fast path needs absolute accuracy only); rotating them only burns sweeps.
    const double abs_floor = 1e-15 * amax_s;
    const double tol2 = 1e-30;
    auto pair_at = [m](int R, int i, int& p, int& q) {  // pair i of round R (p < q)
        int a, b;
        if (i == 0) {
            a = m;
            b = R;
        } else {
            a = R + i;
            a -= (a >= m) ? m : 0;
            b = R - i;
            b += (b < 0) ? m : 0;
        }
        p = min(a, b);
        q = max(a, b);
    };
    auto partner = [m](int x, int R) {  // x's opponent in round R
        if (x == m) return R;
        if (x == R) return m;
        int y = 2 * R - x;
        y -= (y >= m) ? m : 0;
        y += (y < 0) ? m : 0;
        return y;
    };
    auto pair_index = [m](int x, int R) {  // index of the pair holding x in round R
        if (x == m || x == R) return 0;
        int i = x - R;
        i += (i < 0) ? m : 0;
        return min(i, m - i);
    };
    auto rotation = [&](double app, double aqq, double apq, int slot, int i) {
        double c = 1.0, s = 0.0;
        if (fabs(apq) > abs_floor && apq * apq > tol2 * fabs(app * aqq)) {
            double t;
            jacobi_rotation(app, aqq, apq, c, s, t);
        }
        cs[slot * npair + i] = make_double2(c, s);
        double* d = dg + (slot * npair + i) * 3;
        d[0] = app;
        d[1] = aqq;
        d[2] = apq;
    };
    // Per-thread work list fixed for the whole solve: upper-triangular blocks
    // (bi ≤ bj) of the pair grid and (row, pair) items of V.
    constexpr int kMaxBlk = 2, kMaxV = 5;  // np ≤ 96: 1176 blocks, 4608 V items
    int blk_i[kMaxBlk], blk_j[kMaxBlk], vk[kMaxV], vp[kMaxV];
    int nb = 0, nv = 0;
    {
        const int nub = npair * (npair + 1) / 2;
        for (int b = tid; b < nub && nb < kMaxBlk; b += kJacThreads) {
            int bi = 0, rem = b;
            while (rem >= npair - bi) {
                rem -= npair - bi;
                ++bi;
            }
            blk_i[nb] = bi;
            blk_j[nb] = bi + rem;
            ++nb;
        }
        for (int e = tid; e < np * npair && nv < kMaxV; e += kJacThreads) {
            vk[nv] = e % np;
            vp[nv] = e / np;
            ++nv;
        }
    }
    // Rotations of round 0.
    if (tid < npair) {
        int p, q;
        pair_at(0, tid, p, q);
        rotation(A[p * ld + p], A[q * ld + q], A[p * ld + q], 0, tid);
    }
    __syncthreads();
    int sweeps_done = 0, gr = 0;  // gr: global round counter (slot = gr & 1)
    for (int sweep = 0; sweep < 40; ++sweep) {
        sweeps_done = sweep + 1;
        for (int r = 0; r < m; ++r, ++gr) {
            const int slot = gr & 1;
            const double2* csr = cs + slot * npair;
            const double* dgr = dg + slot * npair * 3;
            const int Rn = (r + 1 == m) ? 0 : r + 1;  // next round (the schedule repeats every sweep)
            for (int u = 0; u < nb; ++u) {
                const int bi = blk_i[u], bj = blk_j[u];
                int p1, q1, p2, q2;
                pair_at(r, bi, p1, q1);
                pair_at(r, bj, p2, q2);
                const double2 r1 = csr[bi], r2 = csr[bj];
                const double c1 = r1.x, s1 = r1.y, c2 = r2.x, s2 = r2.y;
                const double a11 = A[p1 * ld + p2], a12 = A[p1 * ld + q2];
                const double a21 = A[q1 * ld + p2], a22 = A[q1 * ld + q2];
                // rows: Rᵀ·B with R = [[c, s], [-s, c]], then columns: ·R
                const double b11 = c1 * a11 - s1 * a21, b12 = c1 * a12 - s1 * a22;
                const double b21 = s1 * a11 + c1 * a21, b22 = s1 * a12 + c1 * a22;
                double d11 = c2 * b11 - s2 * b12, d12 = s2 * b11 + c2 * b12;
                double d21 = c2 * b21 - s2 * b22, d22 = s2 * b21 + c2 * b22;
                if (bi == bj) {
                    const double off = 0.5 * (d12 + d21);
                    d12 = d21 = off;
                    A[p1 * ld + p1] = d11;
                    A[q1 * ld + q1] = d22;
                    A[p1 * ld + q1] = off;
                    A[q1 * ld + p1] = off;
                } else {
                    A[p1 * ld + p2] = d11;
                    A[p1 * ld + q2] = d12;
                    A[q1 * ld + p2] = d21;
                    A[q1 * ld + q2] = d22;
                    A[p2 * ld + p1] = d11;
                    A[q2 * ld + p1] = d12;
                    A[p2 * ld + q1] = d21;
                    A[q2 * ld + q1] = d22;
                }
                // Does this block hold a pair (x, y) of the next round?
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int x = e == 0 ? p1 : q1;
                    const int y = partner(x, Rn);
                    int f = -1;
                    if (y == p2) f = 0;
                    else if (y == q2) f = 1;
                    if (f < 0 || (bi == bj && y <= x)) continue;
                    const double gxy = e == 0 ? (f == 0 ? d11 : d12) : (f == 0 ? d21 : d22);
                    // New diagonal entries of x (in pair bi) and y (in pair bj):
                    // (Rᵀ·[[app, apq], [apq, aqq]]·R)_kk, k = position in the pair.
                    auto newdiag = [&](int pi, int k) {
                        const double2 rr = csr[pi];
                        const double* d = dgr + pi * 3;
                        const double c = rr.x, s = rr.y, cc = c * c, ss = s * s, c2s = 2.0 * c * s;
                        return k == 0 ? cc * d[0] - c2s * d[2] + ss * d[1] : ss * d[0] + c2s * d[2] + cc * d[1];
                    };
                    const double ax = newdiag(bi, e), ay = newdiag(bj, f);
                    const int j = pair_index(x, Rn);
                    if (x < y) rotation(ax, ay, gxy, slot ^ 1, j);
                    else rotation(ay, ax, gxy, slot ^ 1, j);
                }
            }
            for (int u = 0; u < nv; ++u) {  // eigenvector columns: V·R
                const double2 rr = csr[vp[u]];
                if (rr.y == 0.0) continue;
                int p, q;
                pair_at(r, vp[u], p, q);
                const int k = vk[u];
                const double x = Vs[k * ld + p], y = Vs[k * ld + q];
                Vs[k * ld + p] = rr.x * x - rr.y * y;
                Vs[k * ld + q] = rr.y * x + rr.x * y;
            }
            __syncthreads();
        }
        // Stop at off(A) ≤ 1e-14·‖A‖_F, or once stalled on rounding noise ≤ 1e-12·‖A‖_F.
        double off = 0.0, tot = 0.0;
        for (int idx = tid; idx < np * np; idx += kJacThreads) {
            const int i = idx % np, j = idx / np;
            const double a = A[i * ld + j];
            tot = fma(a, a, tot);
            if (i != j) off = fma(a, a, off);
        }
        off = warp_sum(off);
        tot = warp_sum(tot);
        if (lane == 0) {
            red[2 * warp] = off;
            red[2 * warp + 1] = tot;
        }
        __syncthreads();
        if (tid == 0) {
            double o = 0.0, t = 0.0;
            for (int w = 0; w < kJacWarps; ++w) {
                o += red[2 * w];
                t += red[2 * w + 1];
            }
            stop = (o <= 1e-28 * t) || (o <= 1e-24 * t && o > 0.25 * prev_off);
            prev_off = o;
        }
        __syncthreads();
        if (stop) break;
    }
    for (int i = tid; i < np; i += kJacThreads) diag[i] = i < n ? A[i * ld + i] : -INFINITY;
    if (tid == 0 && sweeps_out) *sweeps_out = sweeps_done;
    __syncthreads();
    // Stable descending order of the n real eigenvalues (the padding sorts last).
    for (int c = tid; c < n; c += kJacThreads) {
        const double v = diag[c];
        int rank = 0;
        for (int i = 0; i < n; ++i) rank += (diag[i] > v) || (diag[i] == v && i < c);
        lambda[rank] = v;
        for (int i = 0; i < n; ++i) V[i + static_cast<int64_t>(rank) * n] = Vs[i * ld + c];
    }
}

// Cholesky R (upper, RᵀR = G) of small SPD matrices and their inverses R⁻¹, one
// CTA per matrix (blockIdx.x indexes the batch).  flag[b] |= 1 when a pivot is
// not safely positive, |= 2 when check_identity and max|G - I| > 1e-2 (second
// CholQR pass on a badly conditioned input).
//
// Thread (g, j) of the 4 × NC grid keeps column j, rows g, g+4, g+8, … in
// registers; each elimination step is one broadcast of a pivot row through
// shared memory plus one FMA per owned row — one barrier per step.  Both
// loops are fully unrolled over the row blocks so every register index is
// static (a run-time index would send the array to local memory) and rows
// already finished drop out at compile time.
//  1. outer-product Cholesky on unscaled rows: G = Uᵀ·D⁻¹·U, R = D^{-1/2}·U,
//     D = diag(U).  Published rows carry zeros left of the diagonal, so the
//     update needs no row predicate.
//  2. R⁻¹ from the last row up: X[q][c] = d_q·(δ_qc − d_q·Σ_{m>q} U[q][m]·X[m][c]),
//     d_q = U[q][q]^{-1/2} = 1 / R[q][q].
#ifdef TS_CHOL_PROBE
__device__ long long g_chol_probe[8];
#define CHOL_T(i) if (threadIdx.x == 0 && blockIdx.x == 0) g_chol_probe[i] = clock64();
#else
#define CHOL_T(i)
#endif
template <int NC>
__global__ void __launch_bounds__(4 * NC) chol_inv_kernel(CholBatch cb) {
    constexpr int RPT = NC / 4;  // rows per thread
    constexpr int LD = NC + 1;   // odd stride: the column-major store below is conflict-free
    const int b = blockIdx.x;
    const int n = cb.n;
    const double* __restrict__ G = cb.Gd ? cb.Gd[b] : cb.G[b];
    extern __shared__ __align__(16) double sm[];
    double* U = sm;           // n × LD: published rows of U
    double* X = U + n * LD;   // n × LD: rows of R⁻¹
    double* rd = X + n * LD;  // n: U[q][q]^{-1/2}
    __shared__ int bad;
    __shared__ double dmax;
    const int tid = threadIdx.x;
    const int j = tid % NC, g = tid / NC;
    if (tid == 0) {
        bad = 0;
        dmax = 0.0;
    }
    __syncthreads();
    double a[RPT];
    double dev = 0.0, dm = 0.0;
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
        const int i = g + 4 * r;
        double v = 0.0;
        if (i < n && j < n) {
            v = G[i + static_cast<int64_t>(j) * cb.ldg];
            dev = fmax(dev, fabs(v - (i == j ? 1.0 : 0.0)));
            if (i == j) dm = fmax(dm, v);
        }
        a[r] = v;
    }
    if (cb.check_identity && dev > 1e-2) atomicOr(&bad, 2);
    for (int o = 16; o > 0; o >>= 1) dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
    if ((tid & 31) == 0 && dm > 0)
        atomicMax(reinterpret_cast<unsigned long long*>(&dmax), __double_as_longlong(dm));
    __syncthreads();
    const double floor_piv = 1e-28 * dmax;
    const double repl = fmax(dmax, 1.0);
    const unsigned Ub = smem_u32(U), Xb = smem_u32(X), rdb = smem_u32(rd);
    constexpr unsigned ld8 = 8u * LD;
    const unsigned urow = Ub + g * ld8;  // this thread's first row of U (rows g + 4r)
    CHOL_T(0)

    // 1. Cholesky.  Step k = 4·kk + g4: the owners of row k publish it, everyone eliminates.
#pragma unroll
    for (int kk = 0; kk < RPT; ++kk) {
#pragma unroll
        for (int g4 = 0; g4 < 4; ++g4) {
            const int k = 4 * kk + g4;
            if (k < n) {
                const unsigned rowk = Ub + k * ld8;
                if (g == g4) {
                    double v = (j >= k && j < n) ? a[kk] : 0.0;
                    if (j == k && !(v > floor_piv)) {
                        bad |= 1;  // benign race: every writer stores the same bit
                        v = repl;
                    }
                    sts64(rowk + 8u * j, v);
                }
                __syncthreads();
                const double p = lds64(rowk + 8u * k);
                const double f = (j > k && j < n) ? lds64(rowk + 8u * j) / p : 0.0;
#pragma unroll
                for (int r = kk; r < RPT; ++r) a[r] = fma(-lds64(rowk + 8u * (g + 4 * r)), f, a[r]);
            }
        }
    }
    __syncthreads();
    for (int q = tid; q < n; q += 4 * NC) rd[q] = 1.0 / sqrt(U[q * LD + q]);
    __syncthreads();
    CHOL_T(1)

    // 2. R⁻¹, last row first; a[r] accumulates Σ_m U[i][m]·X[m][j] for own rows i.
#pragma unroll
    for (int r = 0; r < RPT; ++r) a[r] = 0.0;
#pragma unroll
    for (int qq = RPT - 1; qq >= 0; --qq) {
#pragma unroll
        for (int g4 = 3; g4 >= 0; --g4) {
            const int q = 4 * qq + g4;
            if (q < n) {
                const unsigned rowq = Xb + q * ld8;
                if (g == g4) {
                    const double dq = lds64(rdb + 8u * q);
                    const double v = (j >= q && j < n) ? dq * ((j == q ? 1.0 : 0.0) - dq * a[qq]) : 0.0;
                    sts64(rowq + 8u * j, v);
                }
                __syncthreads();
                const double xq = lds64(rowq + 8u * j);
#pragma unroll
                for (int r = 0; r <= qq; ++r) a[r] = fma(lds64(urow + r * 4u * ld8 + 8u * q), xq, a[r]);
            }
        }
    }
    __syncthreads();
    CHOL_T(2)
    double* Rinv = cb.Rd ? cb.Rd[b] : cb.Rinv[b];
    for (int idx = tid; idx < n * n; idx += 4 * NC) {
        const int i = idx % n, c = idx / n;
        Rinv[i + static_cast<int64_t>(c) * cb.ldri] = X[i * LD + c];
    }
    CHOL_T(4)
    if (tid == 0 && bad) atomicOr(cb.Fd ? cb.Fd[b] : cb.flag[b], bad);
}

// ------------------------------------------------------------------ misc
// Device twin of the ε = 0 branch of gram_rank (capi.cu): with the rank fixed to
// the cap (else q), accept the Gram fast path only when λ_rank is resolvable and
// the kept subspace is separated enough for the 1e-10 parity bar; *flag |= 1
// otherwise.
// Absolute eigen-residual the subspace bound uses: the solver's measured
// ‖C V − V Λ‖_F when it reports one, else the Jacobi solver's 1e-14·λ₁.
__device__ __forceinline__ double resid_abs(const double* resid, double l1) {
    return resid ? fmax(resid[0], 1e-16 * l1) : 1e-14 * l1;
}

__global__ void gram_check_kernel(const double* __restrict__ lam, int q, int cap, const double* __restrict__ resid,
                                  int* __restrict__ flag, int64_t strideL) {
    if (threadIdx.x != 0) return;
    {  // batched: CTA b checks problem b
        const int64_t b = blockIdx.x;
        lam += b * strideL;
        if (resid) resid += b;
        flag += b;
    }
    const double l1 = lam[0];
    bool ok = l1 > 0.0;
    if (ok) {
        const double resolvable = 1e-8 * l1;
        const int rank = (cap > 0 && cap < q) ? cap : q;
        const double lr = fmax(lam[rank - 1], 0.0);
        ok = lr >= resolvable;
        if (ok && rank < q) {
            const double lnext = fmax(lam[rank], 0.0);
            const double gap = lr - lnext;
            ok = gap > 0.0;
            if (ok) ok = !(resid_abs(resid, l1) / gap * sqrt(lnext / l1) > 1e-11);
        }
    }
    if (!ok) atomicOr(flag, 1);
}

constexpr int kMaxRankRule = 128;

// Device twin of the ε > 0 branch of gram_rank (capi.cu) for a call whose output
// rank is already known (a CUDA-graph replay or a speculated call): recomputes
// θ = ε²‖h‖²/d from the device ‖h‖², the reference tail rule on the Gram
// eigenvalues (suffix sums in the same order, no FMA contraction, so the decision
// is bitwise the host's), the provability margins and the subspace separation,
// and sets *flag |= 1 unless the fast path is accepted with exactly `expect`.
__global__ void gram_rank_check_kernel(const double* __restrict__ lam, int q, int cap, double eps, int order,
                                       const double* __restrict__ hss, const double* __restrict__ resid, int expect,
                                       int* __restrict__ flag) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const double l1 = fmax(lam[0], 0.0);
    bool ok = lam[0] > 0.0;
    int rank = 1;
    if (ok) {
        const double theta = __ddiv_rn(__dmul_rn(__dmul_rn(eps, eps), hss[0]), static_cast<double>(order));
        const double noise = __dmul_rn(1e-12, l1);
        double suffix[kMaxRankRule + 1];
        suffix[q] = 0.0;
        for (int j = q - 1; j >= 0; --j) suffix[j] = __dadd_rn(suffix[j + 1], fmax(lam[j], 0.0));
        int r = q;
        for (int i = 1; i <= q; ++i)
            if (suffix[i] <= theta) {
                r = i;
                break;
            }
        const double margin = __dmul_rn(static_cast<double>(q), noise);
        if (r < q && suffix[r] > __dsub_rn(theta, margin)) ok = false;
        if (r > 1 && suffix[r - 1] <= __dadd_rn(theta, margin)) ok = false;
        rank = (cap > 0 && cap < r) ? cap : r;
        if (ok && rank < q) {
            const double lr = fmax(lam[rank - 1], 0.0), lnext = fmax(lam[rank], 0.0);
            const double gap = __dsub_rn(lr, lnext);
            ok = gap > 0.0;
            if (ok) ok = !(resid_abs(resid, l1) / gap * sqrt(lnext / l1) > 1e-11);
        }
    }
    if (!ok || rank != expect) atomicOr(flag, 1);
}

struct UnfoldArgs {
    int64_t shape[kMaxOrder];
    int order, mode;
};

__global__ void unfold_t_kernel(const double* __restrict__ g, UnfoldArgs a, double* __restrict__ X, int64_t total) {
    int64_t left = 1, right = 1;
    for (int j = 0; j < a.order; ++j) {
        if (j < a.mode) left *= a.shape[j];
        else if (j > a.mode) right *= a.shape[j];
    }
    const int64_t qk = a.shape[a.mode], rest = left * right;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t l = e % left;
        const int64_t i = (e / left) % qk;
        const int64_t r = e / (left * qk);
        X[(l + left * r) + i * rest] = g[e];
    }
}

// Batched: problem blockIdx.y reads gs[y] and writes Xs[y] (same shape).
__global__ void unfold_t_batched_kernel(const double* const* __restrict__ gs, UnfoldArgs a, double* const* __restrict__ Xs,
                                        int64_t total) {
    int64_t left = 1, right = 1;
    for (int j = 0; j < a.order; ++j) {
        if (j < a.mode) left *= a.shape[j];
        else if (j > a.mode) right *= a.shape[j];
    }
    const int64_t qk = a.shape[a.mode], rest = left * right;
    const double* __restrict__ g = gs[blockIdx.y];
    double* __restrict__ X = Xs[blockIdx.y];
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t l = e % left;
        const int64_t i = (e / left) % qk;
        const int64_t r = e / (left * qk);
        X[(l + left * r) + i * rest] = g[e];
    }
}

// Σ x_i² in two deterministic passes: fixed contiguous chunks per CTA, then the
// per-CTA partials summed in order by one CTA.
constexpr int kSumsqBlocks = 128;

__device__ __forceinline__ double block_sum(double s, double* part) {
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
    __syncthreads();
    double v = 0.0;
    if (threadIdx.x < 32) {
        v = threadIdx.x < blockDim.x / 32 ? part[threadIdx.x] : 0.0;
        v = warp_sum(v);
    }
    return v;
}

__global__ void sumsq_partial_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ partial) {
    __shared__ double part[32];
    const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
    const int64_t b = blockIdx.x * chunk, e = min(n, b + chunk);
    double s = 0.0;
    for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x) s = fma(x[i], x[i], s);
    const double v = block_sum(s, part);
    if (threadIdx.x == 0) partial[blockIdx.x] = v;
}

__global__ void sumsq_final_kernel(const double* __restrict__ partial, int np, double* out) {
    __shared__ double part[32];
    double s = 0.0;
    for (int i = threadIdx.x; i < np; i += blockDim.x) s += partial[i];
    const double v = block_sum(s, part);
    if (threadIdx.x == 0) out[0] = v;
}

__global__ void scale_columns_kernel(const double* __restrict__ F, int64_t n, int64_t R, const double* __restrict__ sc,
                                     double* __restrict__ out, bool transpose) {
    const int64_t total = n * R;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e % n, c = e / n;
        const double v = F[e] * sc[c];
        if (transpose) out[c + i * R] = v;
        else out[e] = v;
    }
}

int tsqr_block_rows(int64_t cols) {
    const int64_t cap = 20480 / std::max<int64_t>(cols, 1);  // 160 KB of fp64 per block
    return static_cast<int>(std::max<int64_t>(2 * cols, std::min<int64_t>(256, cap)));
}

}  // namespace

#ifdef TS_CHOL_PROBE
extern "C" void tsi_read_chol_probe(long long* out) { cudaMemcpyFromSymbol(out, g_chol_probe, 8 * sizeof(long long)); }
#endif

int max_tsqr_cols() { return 96; }

namespace {
__global__ void atom_sumsq_kernel(const double* __restrict__ cores, const Atom* __restrict__ atoms, int order,
                                  double* __restrict__ out) {
    const Atom& at = atoms[blockIdx.x];
    int64_t e = 1;
    for (int j = 0; j < order; ++j) e *= at.shape[j];
    const double* c = cores + at.core_off;
    __shared__ double part[32];
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < e; i += blockDim.x) s = fma(c[i], c[i], s);
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < blockDim.x / 32 ? part[threadIdx.x] : 0.0;
        v = warp_sum(v);
        if (threadIdx.x == 0) out[blockIdx.x] = v;
    }
}
}  // namespace

void launch_atom_sumsq(const double* cores, const Atom* atoms, int natoms, int order, double* out, CallScratch& sc) {
    if (natoms <= 0) return;
    atom_sumsq_kernel<<<natoms, 256, 0, sc.stream()>>>(cores, atoms, order, out);
    TS_LAUNCH_CHECK();
    sc.launches += 1;
}

TsqrPlan plan_tsqr(double* A, int64_t lda, int64_t rows, int64_t cols, double* Q, int64_t ldq, CallScratch& sc) {
    TsqrPlan plan;
    const int br = tsqr_block_rows(cols);
    double* cur = A;
    int64_t cur_ld = lda, cur_rows = rows;
    struct LevelInfo {
        double* A;
        int64_t ld, rows;
        std::vector<int64_t> row0, brows, roff;
        double* taus;
    };
    std::vector<LevelInfo> info;
    while (true) {
        LevelInfo li;
        li.A = cur;
        li.ld = cur_ld;
        li.rows = cur_rows;
        const int64_t nblk = cur_rows <= br ? 1 : (cur_rows + br - 1) / br;
        int64_t next_rows = 0;
        for (int64_t b = 0; b < nblk; ++b) {
            const int64_t r0 = b * br, rb = std::min<int64_t>(br, cur_rows - r0);
            li.row0.push_back(r0);
            li.brows.push_back(rb);
            li.roff.push_back(next_rows);
            next_rows += std::min<int64_t>(rb, cols);
        }
        li.taus = sc.alloc_n<double>(static_cast<size_t>(nblk * cols));
        double* Rbuf = sc.alloc_n<double>(static_cast<size_t>(std::max<int64_t>(next_rows, 1) * cols));
        std::vector<QrTask> tasks;
        for (int64_t b = 0; b < nblk; ++b) {
            QrTask t{};
            t.A = cur + li.row0[static_cast<size_t>(b)];
            t.lda = cur_ld;
            t.rows = static_cast<int>(li.brows[static_cast<size_t>(b)]);
            t.cols = static_cast<int>(cols);
            t.tau = li.taus + b * cols;
            t.R = Rbuf + li.roff[static_cast<size_t>(b)];
            t.ldr = next_rows;
            tasks.push_back(t);
        }
        plan.levels.push_back(std::move(tasks));
        info.push_back(li);
        if (nblk == 1) {
            plan.Rtop = Rbuf;
            plan.kk = next_rows;
            break;
        }
        cur = Rbuf;
        cur_ld = next_rows;
        cur_rows = next_rows;
    }
    if (Q != nullptr) {
        const int64_t q = std::min(rows, cols);
        // Top-down: level L's Q buffer (rows_L × q); level 0 writes into Q.
        std::vector<double*> qbuf(info.size());
        std::vector<int64_t> qld(info.size());
        for (size_t L = 0; L < info.size(); ++L) {
            if (L == 0) {
                qbuf[L] = Q;
                qld[L] = ldq;
            } else {
                qbuf[L] = sc.alloc_n<double>(static_cast<size_t>(info[L].rows * q));
                qld[L] = info[L].rows;
            }
        }
        for (size_t Li = info.size(); Li-- > 0;) {
            const LevelInfo& li = info[Li];
            std::vector<QrApplyTask> tasks;
            for (size_t b = 0; b < li.row0.size(); ++b) {
                QrApplyTask t{};
                t.V = li.A + li.row0[b];
                t.ldv = li.ld;
                t.tau = li.taus + static_cast<int64_t>(b) * cols;
                t.rows = static_cast<int>(li.brows[b]);
                t.kk = static_cast<int>(std::min<int64_t>(li.brows[b], cols));
                t.q = static_cast<int>(q);
                if (Li + 1 == info.size()) {
                    t.Qin = nullptr;
                    t.Rsign = plan.Rtop;
                    t.ldrs = plan.kk;
                } else {
                    t.Qin = qbuf[Li + 1] + li.roff[b];
                    t.ldqin = qld[Li + 1];
                    t.Rsign = nullptr;
                }
                t.Q = qbuf[Li] + li.row0[b];
                t.ldq = qld[Li];
                tasks.push_back(t);
            }
            plan.applies.push_back(std::move(tasks));
        }
    }
    return plan;
}

void run_tsqr(const std::vector<TsqrPlan*>& plans, CallScratch& sc, bool form_q) {
    size_t nlev = 0, napp = 0;
    for (auto* p : plans) {
        nlev = std::max(nlev, p->levels.size());
        napp = std::max(napp, p->applies.size());
    }
    // Per-device, thread-safe smem attribute (runtime.hpp set_max_smem).
    set_max_smem(tsqr_apply_kernel<4>, 200 * 1024); set_max_smem(tsqr_apply_kernel<6>, 200 * 1024);
    for (size_t L = 0; L < nlev; ++L) {
        std::vector<QrTask> tasks;
        size_t smem = 0;
        for (auto* p : plans)
            if (L < p->levels.size())
                for (const QrTask& t : p->levels[L]) {
                    tasks.push_back(t);
                    smem = std::max(smem, sizeof(double) * static_cast<size_t>(t.rows) * t.cols);
                }
        if (tasks.empty()) continue;
        auto* d = static_cast<const QrTask*>(sc.upload(tasks.data(), tasks.size() * sizeof(QrTask)));
        int mrows = 0, mcols = 0;
        for (const QrTask& t : tasks) {
            mrows = std::max(mrows, t.rows);
            mcols = std::max(mcols, t.cols);
        }
        const unsigned nb = static_cast<unsigned>(tasks.size());
        cudaStream_t st = sc.stream();
        if (mcols <= 64) {
            if (mrows <= 64) tsqr_factor_kernel<2, 4><<<nb, kQrFThreads, 0, st>>>(d);
            else if (mrows <= 128) tsqr_factor_kernel<4, 4><<<nb, kQrFThreads, 0, st>>>(d);
            else tsqr_factor_kernel<8, 4><<<nb, kQrFThreads, 0, st>>>(d);
        } else {
            if (mrows <= 64) tsqr_factor_kernel<2, 6><<<nb, kQrFThreads, 0, st>>>(d);
            else if (mrows <= 128) tsqr_factor_kernel<4, 6><<<nb, kQrFThreads, 0, st>>>(d);
            else tsqr_factor_kernel<8, 6><<<nb, kQrFThreads, 0, st>>>(d);
        }
        TS_LAUNCH_CHECK();
        sc.launches += 1;
    }
    if (!form_q) return;
    // Apply levels are stored top-down per plan; align plans at their top level.
    for (size_t A = 0; A < napp; ++A) {
        std::vector<QrApplyTask> tasks;
        size_t smem = 0;
        for (auto* p : plans) {
            const size_t off = napp - p->applies.size();  // plans with fewer levels start later
            if (A < off) continue;
            for (const QrApplyTask& t : p->applies[A - off]) {
                tasks.push_back(t);
                smem = std::max(smem, sizeof(double) * (static_cast<size_t>(t.rows) * (t.q + 2) + t.kk));
            }
        }
        if (tasks.empty()) continue;
        auto* d = static_cast<const QrApplyTask*>(sc.upload(tasks.data(), tasks.size() * sizeof(QrApplyTask)));
        int mq = 0;
        for (const QrApplyTask& t : tasks) mq = std::max(mq, t.q);
        if (mq <= 64) tsqr_apply_kernel<4><<<static_cast<unsigned>(tasks.size()), kQrThreads, smem, sc.stream()>>>(d);
        else tsqr_apply_kernel<6><<<static_cast<unsigned>(tasks.size()), kQrThreads, smem, sc.stream()>>>(d);
        TS_LAUNCH_CHECK();
        sc.launches += 1;
    }
}

void launch_sym_jacobi(const double* C, int64_t ldc, int n, double* lambda, double* V, CallScratch& sc, int* sweeps) {
    if (launch_sym_jacobi_pp(C, ldc, n, lambda, V, sc, sweeps)) return;  // eig.cu, n ≤ 64
    const size_t np = static_cast<size_t>(n + (n & 1));
    const size_t smem = sizeof(double) * (2 * np * (np + 1) + 2 * np + 3 * np + np) + 16;
    // Per-device, thread-safe smem attribute (runtime.hpp set_max_smem).
    set_max_smem(sym_jacobi_kernel, 200 * 1024);
    sym_jacobi_kernel<<<1, kJacThreads, smem, sc.stream()>>>(C, ldc, n, lambda, V, sweeps);
    TS_LAUNCH_CHECK();
    sc.launches += 1;
}

void launch_gram_check(const double* lam, int q, int cap, const double* resid, int* flag, CallScratch& sc, int count,
                       int64_t strideL) {
    if (count < 1) return;
    gram_check_kernel<<<count, 32, 0, sc.stream()>>>(lam, q, cap, resid, flag, strideL);
    TS_LAUNCH_CHECK();
    sc.launches += 1;
}

void launch_gram_rank_check(const double* lam, int q, int cap, double eps, int order, const double* hss,
                            const double* resid, int expect, int* flag, CallScratch& sc) {
    if (q > kMaxRankRule) throw Error(TS_UNSUPPORTED, "gram_rank_check: q exceeds the device maximum");
    gram_rank_check_kernel<<<1, 32, 0, sc.stream()>>>(lam, q, cap, eps, order, hss, resid, expect, flag);
    TS_LAUNCH_CHECK();
    sc.launches += 1;
}

// R-form condition check (capi.cu stages D/E): κ_F(R)² = trace(YᵀY)·‖R⁻¹‖_F² ≥
// κ₂(Y)²; the R form P = R⁻ᵀ(YᵀF) loses a factor κ(Y) of accuracy, so modes
// with κ_F > 1e4 (error > ~1e-12) get *flag |= 4 (→ Householder TSQR).
__global__ void rform_check_kernel(CholBatch cb) {
    __shared__ double part[32];
    const int b = blockIdx.x, n = cb.n;
    double tr = 0.0, fr = 0.0;
    const double* G = cb.Gd ? cb.Gd[b] : cb.G[b];
    const double* Ri = cb.Rd ? cb.Rd[b] : cb.Rinv[b];
    for (int i = threadIdx.x; i < n; i += blockDim.x) tr += G[i + static_cast<int64_t>(i) * cb.ldg];
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
        const double v = Ri[e % n + static_cast<int64_t>(e / n) * cb.ldri];
        fr = fma(v, v, fr);
    }
    tr = block_sum(tr, part);
    __syncthreads();
    fr = block_sum(fr, part);
    if (threadIdx.x == 0 && !(tr * fr <= 1e8)) atomicOr(cb.Fd ? cb.Fd[b] : cb.flag[b], 4);
}

void launch_rform_check(const CholBatch& cb, int count, CallScratch& sc) {
    if (count <= 0) return;
    rform_check_kernel<<<count, 256, 0, sc.stream()>>>(cb);
    TS_LAUNCH_CHECK();
    sc.launches += 1;
}

void launch_chol_inv(const CholBatch& cb, int count, CallScratch& sc) {
    if (count <= 0) return;
    if (cb.n > 96) throw std::invalid_argument("chol_inv: n > 96");
    const size_t ldc = cb.n <= 32 ? 33 : cb.n <= 48 ? 49 : cb.n <= 64 ? 65 : 97;  // LD of the kernel instance
    const size_t smem = sizeof(double) * (2 * static_cast<size_t>(cb.n) * ldc + cb.n);
    // Per-device, thread-safe smem attribute (runtime.hpp set_max_smem).
    set_max_smem(chol_inv_kernel<32>, 200 * 1024); set_max_smem(chol_inv_kernel<48>, 200 * 1024); set_max_smem(chol_inv_kernel<64>, 200 * 1024); set_max_smem(chol_inv_kernel<96>, 200 * 1024);
    if (cb.n <= 32) chol_inv_kernel<32><<<count, 4 * 32, smem, sc.stream()>>>(cb);  // small sketches: half the threads and rows
    else if (cb.n <= 48) chol_inv_kernel<48><<<count, 4 * 48, smem, sc.stream()>>>(cb);
    else if (cb.n <= 64) chol_inv_kernel<64><<<count, 4 * 64, smem, sc.stream()>>>(cb);
    else chol_inv_kernel<96><<<count, 4 * 96, smem, sc.stream()>>>(cb);
    TS_LAUNCH_CHECK();
    sc.launches += 1;
}

void launch_jacobi_svd(const double* R, int64_t ldr, int m, int nc, double* sigma, double* U, CallScratch& sc) {
    const size_t smem = sizeof(double) * (static_cast<size_t>(m) * nc + static_cast<size_t>(nc) * nc + nc);
    // Per-device, thread-safe smem attribute (runtime.hpp set_max_smem).
    set_max_smem(jacobi_svd_kernel, 200 * 1024);
    jacobi_svd_kernel<<<1, kJacThreads, smem, sc.stream()>>>(R, ldr, m, nc, sigma, U, eig_probe_buffer());
    TS_LAUNCH_CHECK();
    sc.launches += 1;
}

void launch_unfold_t(const double* g, int order, const int64_t* shape, int mode, double* X, CallScratch& sc) {
    UnfoldArgs a{};
    int64_t total = 1;
    for (int j = 0; j < order; ++j) {
        a.shape[j] = shape[j];
        total *= shape[j];
    }
    a.order = order;
    a.mode = mode;
    const int threads = 256;
    const int64_t blocks = std::min<int64_t>((total + threads - 1) / threads, 2048);
    unfold_t_kernel<<<static_cast<unsigned>(std::max<int64_t>(blocks, 1)), threads, 0, sc.stream()>>>(g, a, X, total);
    TS_LAUNCH_CHECK();
    sc.launches += 1;
}

void launch_unfold_t_batched(const double* const* gs, double* const* Xs, int count, int order, const int64_t* shape,
                             int mode, CallScratch& sc) {
    if (count < 1) return;
    UnfoldArgs a{};
    int64_t total = 1;
    for (int j = 0; j < order; ++j) {
        a.shape[j] = shape[j];
        total *= shape[j];
    }
    a.order = order;
    a.mode = mode;
    const int threads = 256;
    const int64_t blocks = std::min<int64_t>((total + threads - 1) / threads, 1024);
    unfold_t_batched_kernel<<<dim3(static_cast<unsigned>(std::max<int64_t>(blocks, 1)), static_cast<unsigned>(count)), threads,
                              0, sc.stream()>>>(gs, a, Xs, total);
    TS_LAUNCH_CHECK();
    sc.launches += 1;
}

void launch_scale_columns(const double* F, int64_t n, int64_t R, const double* scale, double* out, bool transpose,
                          CallScratch& sc) {
    const int threads = 256;
    const int64_t blocks = std::min<int64_t>((n * R + threads - 1) / threads, 4096);
    scale_columns_kernel<<<static_cast<unsigned>(std::max<int64_t>(blocks, 1)), threads, 0, sc.stream()>>>(F, n, R, scale,
                                                                                                         out, transpose);
    TS_LAUNCH_CHECK();
    sc.launches += 1;
}

void launch_sumsq(const double* x, int64_t n, double* out, CallScratch& sc) {
    double* partial = sc.alloc_n<double>(kSumsqBlocks);
    sumsq_partial_kernel<<<kSumsqBlocks, 256, 0, sc.stream()>>>(x, n, partial);
    TS_LAUNCH_CHECK();
    sumsq_final_kernel<<<1, 128, 0, sc.stream()>>>(partial, kSumsqBlocks, out);
    TS_LAUNCH_CHECK();
    sc.launches += 2;
}

namespace {
// Kron stage B epilogue: Wt[c + C·(col + i)] = w · V[l + L·(i + r·t)], c = l + L·t
// (the mode-n unfolding of the atom's sketched block, transposed and scaled).
__global__ void kron_gather_kernel(const KronGather* __restrict__ g, int count, int64_t C, double* __restrict__ Wt,
                                   const double* __restrict__ weights) {
    for (int a = blockIdx.y; a < count; a += gridDim.y) {
        const KronGather d = g[a];
        const double w = weights[d.summand];
        const int64_t total = C * d.r;
        for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
             e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            const int64_t c = e % C, i = e / C;
            const int64_t l = c % d.L, t = c / d.L;
            Wt[c + C * (d.col + i)] = w * d.V[l + d.L * (i + static_cast<int64_t>(d.r) * t)];
        }
    }
}
}  // namespace

void launch_kron_gather(const std::vector<KronGather>& g, int64_t C, double* Wt, const double* weights,
                        CallScratch& sc) {
    if (g.empty()) return;
    int64_t most = 1;
    for (const auto& x : g) most = std::max<int64_t>(most, C * x.r);
    auto* dg = static_cast<KronGather*>(sc.upload(g.data(), sizeof(KronGather) * g.size()));
    const int threads = 256;
    const unsigned bx = static_cast<unsigned>(std::min<int64_t>((most + threads - 1) / threads, 64));
    const unsigned by = static_cast<unsigned>(std::min<size_t>(g.size(), 65535));
    kron_gather_kernel<<<dim3(bx, by), threads, 0, sc.stream()>>>(dg, static_cast<int>(g.size()), C, Wt, weights);
    TS_LAUNCH_CHECK();
    sc.launches += 1;
}

namespace {
// acc[0] += alpha · Σ x_i y_i, one CTA, fixed reduction order (deterministic).
__global__ void __launch_bounds__(256) dot_accumulate_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                                            int64_t n, double alpha, double* __restrict__ acc) {
    __shared__ double part[8];
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s = fma(x[i], y[i], s);
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += part[w];
        acc[0] += alpha * t;
    }
}
}  // namespace

void launch_dot_accumulate(const double* x, const double* y, int64_t n, double alpha, double* acc, CallScratch& sc) {
    dot_accumulate_kernel<<<1, 256, 0, sc.stream()>>>(x, y, n, alpha, acc);
    TS_LAUNCH_CHECK();
    sc.launches += 1;
}

}  // namespace ts
