// eig_trd.cu — the symmetric eigensolver of ST-HOSVD's Gram fast path (stage G)
// for n ≤ 64: ONE kernel, one CTA of 512 threads per problem (batched over
// blockIdx.x for segmented sums).
//
// Reference semantics: sym_eig (src/kernels.cpp:70-86) — symmetrise,
// eigendecompose, eigenpairs in descending order.  Stage G runs one of these
// per mode on the serial tail of every call, so the kernel is built for
// latency: every phase is either a short chain per step with all 16 warps busy,
// or independent per-eigenvector chains with no CTA barrier.
//
//  1. Householder tridiagonalisation QᵀCQ = T (dsytd2 order, lower).  The
//     matrix lives in REGISTERS: thread (i = tid/8, t = tid%8) owns row i,
//     columns t + 8u (shared memory only carries v, p and one partial per
//     warp, so a step is not bound by the shared-memory pipe).  Per reflector:
//     p = τ·A v (8-lane row sums), the rank-2 update A −= v wᵀ + w vᵀ, and the
//     8 lanes of the next row form the next reflector from their registers
//     (one 8-lane reduction, MUFU rsqrt/rcp + Newton) — two CTA barriers per
//     step; warps whose rows are finished skip the step.
//  2. Eigenvalues of T to ~2^-44 of its Gershgorin width by multisection: 8
//     lanes per eigenvalue, 8 shifts per round (9× narrowing), 14 rounds, Sturm
//     counts from the sign bits of the product-form recurrence
//     p_i = (d_i − x)p_{i−1} − e²_{i−1}p_{i−2} (one dependent FMA per step,
//     power-of-two rescaling every 8 steps).  Full accuracy comes from step 5.
//  3. Eigenvectors of T by inverse iteration on the LDLᵀ factorisation of
//     T − λI (thread per eigenvalue, two iterations).
//  4. Back-transformation Z ← H_0 ⋯ H_{n−3} Z: 8 lanes per eigenvector, its
//     rows in registers, no CTA barrier.
//  5. Orthonormality: E = ZᵀZ − I (DMMA); Löwdin steps Z ← Z − ½ZE for small
//     defects (close eigenvalues), modified Gram-Schmidt with completion for
//     collapsed clusters (e.g. the zero eigenvalues of a rank-deficient Gram).
//     Then R = C Z (DMMA), λ_j = z_jᵀ(Cz_j) (Rayleigh
//     quotients: accurate to O(ε‖C‖ + ‖r_j‖²/gap)), the measured residual
//     ‖C Z − ZΛ‖_F (written to *resid; the rank checks use it), and the
//     descending sort.  A non-finite or too large residual sets *flag and the
//     caller recomputes with the Jacobi solver (eig.cu).
#include <cmath>
#include <cstdlib>
#include <string>

#include "kernels.cuh"

namespace ts {
namespace {

constexpr int kEN = 64;               // largest n
constexpr int kEThreads = 512;        // 16 warps
constexpr int kEWarps = kEThreads / 32;
constexpr int kLA = 72;               // row stride of the [row][col] smem matrices
constexpr double kEps = 1.1102230246251565e-16;

struct TrdSmem {
    double A[kEN * kLA];      // matrix during (1); later C for the residual; later R = C Z
    double Z[kEN * kLA];      // eigenvectors [row][col]
    double Lm[kEN * kEN];     // inverse iteration: L_i of eigenvalue j at [i*kEN + j]; later E, Z·E
    double Dinv[kEN * kEN];   //                    1/D_i at [i*kEN + j]
    double V[kEN * kEN];      // reflector k at V[k*kEN + i]: v_i = 0 for i ≤ k, v_{k+1} = 1
    double2 de2[kEN + 8];     // multisection operands (d_i, e²_{i−1}), scaled, padded
    double lamb[kEN];         // multisection eigenvalues (scaled, ascending)
    double tau[kEN], d[kEN], e[kEN], ds[kEN], e2s[kEN], es[kEN], lam[kEN], p[kEN], rowfill[kEN];
    double red[kEWarps];
    double misc[8];
    int rank[kEN];
    int flag;
};

__device__ __forceinline__ double rcp_refined(double x) {  // ≈ correctly rounded 1/x
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    y = y * fma(-x, y, 2.0);
    y = y * fma(-x, y, 2.0);
    return fma(y, fma(-x, y, 1.0), y);
}

__device__ __forceinline__ double sqrt_refined(double x) {  // x > 0
    double rs;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(rs) : "d"(x));
    rs = rs * fma(-0.5 * x, rs * rs, 1.5);
    rs = rs * fma(-0.5 * x, rs * rs, 1.5);
    const double sq = x * rs;
    return fma(0.5 * rs, fma(-sq, sq, x), sq);
}

// 2^-(exponent of m) for m > 0, exactly representable (rescales a pair of
// polynomial values into [1, 2) without rounding).
__device__ __forceinline__ double inv_pow2_of(double m) {
    const int hi = __double2hiint(m);
    const int ex = (hi >> 20) & 0x7ff;  // biased exponent (m is finite, normal here)
    return __hiloint2double((2046 - ex) << 20, 0);
}

// Out(64×64) = op(X)·Y over kLA-strided smem operands with DMMA.8x8x4 (inner
// dimension n, zero beyond); warp w computes the 8×8 output tiles w, w+16, ….
// TransX: op(X)(i,k) = X[k][i].  Out may be given a different stride.
template <bool TransX>
__device__ __forceinline__ void dmma_64(const double* X, const double* Y, double* Out, int ldo, int n) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    for (int tile = warp; tile < 64; tile += kEWarps) {
        const int r0 = 8 * (tile & 7), c0 = 8 * (tile >> 3);
        double c_0 = 0.0, c_1 = 0.0;
        for (int k0 = 0; k0 < n; k0 += 4) {
            const int kk = k0 + t;
            const double a = kk < n ? (TransX ? X[kk * kLA + r0 + g] : X[(r0 + g) * kLA + kk]) : 0.0;
            const double b = kk < n ? Y[kk * kLA + c0 + g] : 0.0;
            dmma884(c_0, c_1, a, b);
        }
        Out[(r0 + g) * ldo + c0 + 2 * t] = c_0;
        Out[(r0 + g) * ldo + c0 + 2 * t + 1] = c_1;
    }
}

__device__ __forceinline__ double block_max(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    v = 0.0;
#pragma unroll
    for (int w = 0; w < kEWarps; ++w) v = fmax(v, red[w]);
    __syncthreads();
    return v;
}

__global__ void __launch_bounds__(kEThreads, 1)
    trd_eig_kernel(const double* __restrict__ Cin, int64_t ldc, int n, double* __restrict__ lambda_out,
                   double* __restrict__ V_out, int* __restrict__ flag_out, double* __restrict__ resid_out,
                   unsigned long long* __restrict__ prof, int64_t strideC, int64_t strideL, int64_t strideV,
                   int variant) {
    {  // batched launches (segmented sums): CTA b solves problem b
        const int64_t b = blockIdx.x;
        Cin += b * strideC;
        lambda_out += b * strideL;
        V_out += b * strideV;
        flag_out += b;
        if (resid_out) resid_out += b;
        if (b > 0) prof = nullptr;
    }
    extern __shared__ __align__(16) unsigned char smraw[];
    TrdSmem& S = *reinterpret_cast<TrdSmem*>(smraw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ri = tid >> 3, rt = tid & 7;  // row ri, columns rt + 8u
    long long tmark = clock64();
    auto phase = [&](int ph) {  // optional phase clocks (TS_EIG_PROFILE): prof[10 + phase]
        if (prof != nullptr && tid == 0) {
            const long long now = clock64();
            prof[10 + ph] = static_cast<unsigned long long>(now - tmark);
            tmark = now;
        }
    };

    // ---- load + symmetrise; zero the padding and the reflector store
    for (int idx = tid; idx < kEN * kEN; idx += kEThreads) {
        const int i = idx & 63, j = idx >> 6;
        S.A[i * kLA + j] = (i < n && j < n) ? 0.5 * (Cin[i + static_cast<int64_t>(j) * ldc] + Cin[j + static_cast<int64_t>(i) * ldc])
                                            : 0.0;
        S.V[idx] = 0.0;
    }
    if (tid == 0) S.flag = 0;
    if (prof && tid == 0) prof[19] = prof[20] = prof[21] = 0;
    if (tid < kEN) {
        S.tau[tid] = 0.0;
        S.e[tid] = 0.0;
        S.d[tid] = 0.0;
    }
    __syncthreads();
    if (n == 1) {
        if (tid == 0) {
            const double c = S.A[0];
            lambda_out[0] = c;
            V_out[0] = 1.0;
            if (resid_out) *resid_out = 0.0;
            if (!isfinite(c)) atomicOr(flag_out, 1);
        }
        return;
    }

    // ---- 1. tridiagonalisation.  A in registers: thread (ri, rt) holds
    // a[u] = A[ri][rt + 8u]; the full symmetric matrix is updated, so row k is
    // column k.  Step k: [row k's 8 lanes form reflector k] → barrier →
    // p = τ·A v (rows > k) → barrier → A −= v wᵀ + w vᵀ, and row k+1's lanes
    // form reflector k+1 straight from their updated registers.
    double a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = S.A[ri * kLA + rt + 8 * u];
    const int gbase = lane & 24;
    const unsigned gm8 = 0xffu << gbase;
    auto reflector = [&](int k) {  // the 8 lanes of row k (ri == k)
        if (variant == 1) {  // timing ablation: no reflector arithmetic
            if (rt == 0) S.tau[k] = 0.0;
            return;
        }
        double ss = 0.0, xa = 0.0, xd = 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int j = rt + 8 * u;
            ss = (j > k + 1) ? fma(a[u], a[u], ss) : ss;
            xa = (j == k + 1) ? a[u] : xa;
            xd = (j == k) ? a[u] : xd;
        }
        ss += __shfl_xor_sync(gm8, ss, 1);
        ss += __shfl_xor_sync(gm8, ss, 2);
        ss += __shfl_xor_sync(gm8, ss, 4);
        const double alpha = __shfl_sync(gm8, xa, gbase + ((k + 1) & 7));
        const double dkk = __shfl_sync(gm8, xd, gbase + (k & 7));
        double tau = 0.0, beta = alpha, scale = 0.0;
        if (ss > 0.0) {
            beta = -copysign(sqrt_refined(fma(alpha, alpha, ss)), alpha);
            tau = fma(-alpha, rcp_refined(beta), 1.0);  // (β − α)/β
            scale = rcp_refined(alpha - beta);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int j = rt + 8 * u;
            S.V[k * kEN + j] = j == k + 1 ? 1.0 : (j > k + 1 ? a[u] * scale : 0.0);
        }
        if (rt == 0) {
            S.tau[k] = tau;
            S.d[k] = dkk;
            S.e[k] = beta;
        }
    };
    long long c_refl = 0, c_mv = 0, c_up = 0, c0_ = 0;
    if (prof && tid == 0) prof[9] = static_cast<unsigned long long>(clock64() - tmark);
    if (n > 2 && ri == 0) reflector(0);
    __syncthreads();
    if (prof && tid == 0) prof[17] = static_cast<unsigned long long>(clock64() - tmark);
    for (int k = 0; k + 2 < n; ++k) {
        if (prof) c0_ = clock64();
        const double tk = S.tau[k];
        const double* vk = S.V + k * kEN;
        const bool wact = 4 * warp + 3 > k && 4 * warp < n;  // warp-uniform: any row in (k, n)
        double pr = 0.0, vi = 0.0;
        const long long m0_ = clock64();
        if (wact && variant != 2) {
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int u = 0; u < 8; u += 2) {
                s0 = fma(a[u], vk[rt + 8 * u], s0);
                s1 = fma(a[u + 1], vk[rt + 8 * u + 8], s1);
            }
            pr = s0 + s1;
            pr += __shfl_xor_sync(0xffffffffu, pr, 1);
            pr += __shfl_xor_sync(0xffffffffu, pr, 2);
            pr += __shfl_xor_sync(0xffffffffu, pr, 4);
            vi = vk[ri];
            pr = ri > k ? tk * pr : 0.0;
            double pv = pr * vi;  // Σ over the warp's 4 rows
            pv += __shfl_xor_sync(0xffffffffu, pv, 8);
            pv += __shfl_xor_sync(0xffffffffu, pv, 16);
            if (lane == 0) S.red[warp] = pv;
        } else if (lane == 0) {
            S.red[warp] = 0.0;
        }
        if (rt == 0) S.p[ri] = pr;
        if (prof && tid == 480) prof[20] += static_cast<unsigned long long>(clock64() - m0_);
        __syncthreads();
        const long long u0_ = clock64();
        if (prof) {
            const long long c1_ = clock64();
            c_mv += c1_ - c0_;
            c0_ = c1_;
        }
        if (wact && variant != 3) {
            double pv2[kEWarps];
#pragma unroll
            for (int w = 0; w < kEWarps; w += 2) {
                const double2 t2 = *reinterpret_cast<const double2*>(&S.red[w]);
                pv2[w] = t2.x;
                pv2[w + 1] = t2.y;
            }
#pragma unroll
            for (int h = kEWarps / 2; h > 0; h >>= 1)
#pragma unroll
                for (int w = 0; w < h; ++w) pv2[w] += pv2[w + h];
            const double K = 0.5 * tk * pv2[0];
            const double wi = fma(-K, vi, pr);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int j = rt + 8 * u;
                const double vj = vk[j];
                const double wj = fma(-K, vj, S.p[j]);
                a[u] -= fma(vi, wj, wi * vj);
            }
        }
        if (prof && tid == 480) prof[21] += static_cast<unsigned long long>(clock64() - u0_);
        if (prof) {
            const long long c1_ = clock64();
            c_up += c1_ - c0_;
            c0_ = c1_;
        }
        if (k + 3 < n && ri == k + 1) {
            const long long r0_ = clock64();
            reflector(k + 1);
            if (prof && rt == 0) prof[19] += static_cast<unsigned long long>(clock64() - r0_);
        }
        __syncthreads();
        if (prof) c_refl += clock64() - c0_;
    }
    if (prof && tid == 0) prof[16] = static_cast<unsigned long long>(clock64() - tmark);
    {  // trailing 2×2 from the registers of rows n-2, n-1
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int j = rt + 8 * u;
            if (ri == n - 2 && j == n - 2) S.d[n - 2] = a[u];
            if (ri == n - 1 && j == n - 1) S.d[n - 1] = a[u];
            if (ri == n - 1 && j == n - 2) S.e[n - 2] = a[u];
        }
    }
    if (prof && tid == 0) {
        prof[5] = static_cast<unsigned long long>(c_refl);
        prof[6] = static_cast<unsigned long long>(c_mv);
        prof[8] = static_cast<unsigned long long>(c_up);
    }
    __syncthreads();
    phase(0);

    // ---- 2. eigenvalues of T (power-of-two scaled), multisection
    if (warp == 0) {
        double lo = 1e300, hi = -1e300;
        for (int i = lane; i < n; i += 32) {
            const double off = (i > 0 ? fabs(S.e[i - 1]) : 0.0) + (i + 1 < n ? fabs(S.e[i]) : 0.0);
            lo = fmin(lo, S.d[i] - off);
            hi = fmax(hi, S.d[i] + off);
        }
        for (int o = 16; o > 0; o >>= 1) {
            lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        const double tn = fmax(fabs(lo), fabs(hi));
        const double sc = tn > 0.0 ? inv_pow2_of(tn) : 1.0;  // tn·sc in [1, 2)
        for (int i = lane; i < kEN; i += 32) {
            const double es = (i + 1 < n) ? S.e[i] * sc : 0.0;
            S.ds[i] = i < n ? S.d[i] * sc : 0.0;
            S.es[i] = es;
            S.e2s[i] = es * es;
            const double ep = (i >= 1 && i < n) ? S.e[i - 1] * sc : 0.0;
            // (d_i, e²_{i−1}); beyond n a decoupled d = 8 > every shift leaves the
            // Sturm signs unchanged, so the count loop needs no bound checks
            S.de2[i] = make_double2(i < n ? S.d[i] * sc : 8.0, ep * ep);
        }
        if (lane < 8) S.de2[kEN + lane] = make_double2(8.0, 0.0);
        if (lane == 0) {
            const double pad = 8.0 * kEps * n;
            S.misc[0] = lo * sc - pad;
            S.misc[1] = hi * sc + pad;
            S.misc[3] = tn;
            S.misc[4] = 1.0 / sc;  // exact: sc is a power of two
        }
    }
    __syncthreads();
    const double tn = S.misc[3];
    const double isc = S.misc[4];
    if (!(tn > 0.0) || !isfinite(tn)) {  // zero matrix (λ = 0, V = I) or non-finite input (flagged)
        for (int idx = tid; idx < n * n; idx += kEThreads) {
            const int i = idx % n, r = idx / n;
            V_out[i + static_cast<int64_t>(r) * n] = i == r ? 1.0 : 0.0;
        }
        if (tid < n) lambda_out[tid] = 0.0;
        if (tid == 0) {
            if (resid_out) *resid_out = 0.0;
            if (!(tn == 0.0)) atomicOr(flag_out, 1);
        }
        return;
    }
    {
        const int j = ri;                      // eigenvalue j (ascending)
        const int jj = j < n ? j : n - 1;
        const unsigned gbase = lane & 24u;     // the 8 lanes of this eigenvalue
        double lo_b = S.misc[0], hi_b = S.misc[1];
        for (int it = 0; it < 14; ++it) {  // 9^14 ≈ 2^44
            const double x = lo_b + (hi_b - lo_b) * (static_cast<double>(rt + 1) * (1.0 / 9.0));
            // number of eigenvalues < x = sign changes of (1, p_1, …, p_n)
            double pm = 1.0, pc = S.ds[0] - x;
            unsigned sg = static_cast<unsigned>(__double2hiint(pc)) >> 31;
            int cnt = static_cast<int>(sg);
            for (int i0 = 1; i0 < n; i0 += 8) {
                double2 q[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) q[u] = S.de2[i0 + u];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const double pn = fma(q[u].x - x, pc, -q[u].y * pm);
                    pm = pc;
                    pc = pn;
                    const unsigned sn = static_cast<unsigned>(__double2hiint(pc)) >> 31;
                    cnt += static_cast<int>(sn ^ sg);
                    sg = sn;
                }
                const double m = fmax(fabs(pc), fabs(pm));
                if (m > 0.0) {
                    const double f = inv_pow2_of(m);
                    pc *= f;
                    pm *= f;
                }
            }
            const unsigned above = (__ballot_sync(0xffffffffu, cnt > jj) >> gbase) & 0xffu;
            const int first = above ? __ffs(above) - 1 : 8;  // first shift with > jj eigenvalues below it
            const double x_hi = __shfl_sync(0xffffffffu, x, gbase + min(first, 7));
            const double x_lo = __shfl_sync(0xffffffffu, x, gbase + max(first - 1, 0));
            if (first < 8) hi_b = x_hi;
            if (first > 0) lo_b = x_lo;
        }
        if (rt == 0 && j < n) S.lam[j] = 0.5 * (lo_b + hi_b);  // scaled
        if (rt == 0 && j < n) S.lamb[j] = 0.5 * (lo_b + hi_b);  // kept: the output if the vectors are rejected
    }
    __syncthreads();
    phase(1);

    // ---- 3. eigenvectors of T: inverse iteration, thread j
    if (tid < n) {
        const int j = tid;
        const double sig = S.lam[j];
        const double pivtol = 4.0 * kEps;
        double Dp = S.ds[0] - sig;
        if (fabs(Dp) < pivtol) Dp = Dp < 0.0 ? -pivtol : pivtol;
        double Di = rcp_refined(Dp);
        S.Dinv[j] = Di;
        for (int i = 0; i + 1 < n; ++i) {
            const double l = S.es[i] * Di;
            S.Lm[i * kEN + j] = l;
            Dp = (S.ds[i + 1] - sig) - l * S.es[i];
            if (fabs(Dp) < pivtol) Dp = Dp < 0.0 ? -pivtol : pivtol;
            Di = rcp_refined(Dp);
            S.Dinv[(i + 1) * kEN + j] = Di;
        }
        for (int i = 0; i < n; ++i) {  // deterministic start vector, distinct per eigenvalue
            const unsigned h = (static_cast<unsigned>(i) * 2654435761u) ^ (static_cast<unsigned>(j + 1) * 40503u);
            S.Z[i * kLA + j] = 1.0 + 0.5 * (static_cast<double>(h & 0xffffu) * (1.0 / 65535.0) - 0.5);
        }
        for (int itr = 0; itr < 2; ++itr) {
            double y = S.Z[j];
            for (int i = 1; i < n; ++i) {
                y = fma(-S.Lm[(i - 1) * kEN + j], y, S.Z[i * kLA + j]);
                S.Z[i * kLA + j] = y;
            }
            double x = y * S.Dinv[(n - 1) * kEN + j];
            S.Z[(n - 1) * kLA + j] = x;
            double m = fabs(x);
            for (int i = n - 2; i >= 0; --i) {
                x = fma(S.Z[i * kLA + j], S.Dinv[i * kEN + j], -S.Lm[i * kEN + j] * x);
                S.Z[i * kLA + j] = x;
                m = fmax(m, fabs(x));
            }
            // normalise (∞-norm first so the 2-norm cannot overflow)
            const double im = m > 0.0 ? rcp_refined(m) : 0.0;
            double nrm = 0.0;
            for (int i = 0; i < n; ++i) {
                const double z = S.Z[i * kLA + j] * im;
                nrm = fma(z, z, nrm);
            }
            const double inv = nrm > 0.0 ? im * rsqrt(nrm) : 0.0;
            for (int i = 0; i < n; ++i) S.Z[i * kLA + j] *= inv;
        }
    }
    __syncthreads();
    phase(2);

    // ---- 4. back-transformation: column ri (eigenvector), rows rt + 8u in registers
    {
        const int col = ri;
        double z[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = rt + 8 * u;
            z[u] = (col < n && i < n) ? S.Z[i * kLA + col] : 0.0;
        }
        for (int k = n - 3; k >= 0; --k) {
            const double* vk = S.V + k * kEN + rt;
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int u = 0; u < 8; u += 2) {
                a0 = fma(vk[8 * u], z[u], a0);
                a1 = fma(vk[8 * u + 8], z[u + 1], a1);
            }
            double sv = a0 + a1;
            sv += __shfl_xor_sync(0xffffffffu, sv, 1);
            sv += __shfl_xor_sync(0xffffffffu, sv, 2);
            sv += __shfl_xor_sync(0xffffffffu, sv, 4);
            sv *= S.tau[k];
#pragma unroll
            for (int u = 0; u < 8; ++u) z[u] = fma(-sv, vk[8 * u], z[u]);
        }
        __syncthreads();  // every column read its inverse-iteration vector
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = rt + 8 * u;
            S.Z[i * kLA + col] = (col < n && i < n) ? z[u] : 0.0;
        }
    }
    __syncthreads();
    phase(3);

    // ---- 5a. re-orthonormalisation (E = ZᵀZ − I)
    double* E = S.Lm;     // kEN-strided scratch below: use kLA layout inside Lm/Dinv (2·4096 ≥ 64·72)
    double* P = S.Dinv;
    bool mgs = false;
    for (int itl = 0; itl < 3; ++itl) {
        dmma_64<true>(S.Z, S.Z, E, kEN, n);
        __syncthreads();
        double emax = 0.0;
        for (int idx = tid; idx < kEN * kEN; idx += kEThreads) {
            const int i = idx & 63, jx = idx >> 6;
            const double v = (i < n && jx < n) ? E[i * kEN + jx] - (i == jx ? 1.0 : 0.0) : 0.0;
            E[i * kEN + jx] = v;
            emax = fmax(emax, fabs(v));
        }
        emax = block_max(emax, S.red);
        if (emax <= 4.0 * kEps * n) break;  // uniform: orthonormal to working precision
        if (!(emax <= 1e-3) || itl == 2) {
            mgs = true;
            break;
        }
        // P = Z·E (Z rows × E), then Z −= ½P
        {
            const int g = lane >> 2, t = lane & 3;
            for (int tile = warp; tile < 64; tile += kEWarps) {
                const int r0 = 8 * (tile & 7), c0 = 8 * (tile >> 3);
                double c_0 = 0.0, c_1 = 0.0;
                for (int k0 = 0; k0 < n; k0 += 4) {
                    const int kk = k0 + t;
                    const double a = kk < n ? S.Z[(r0 + g) * kLA + kk] : 0.0;
                    const double b = kk < n ? E[kk * kEN + c0 + g] : 0.0;
                    dmma884(c_0, c_1, a, b);
                }
                P[(r0 + g) * kEN + c0 + 2 * t] = c_0;
                P[(r0 + g) * kEN + c0 + 2 * t + 1] = c_1;
            }
        }
        __syncthreads();
        for (int idx = tid; idx < kEN * kEN; idx += kEThreads) {
            const int i = idx & 63, jx = idx >> 6;
            if (i < n && jx < n) S.Z[i * kLA + jx] = fma(-0.5, P[i * kEN + jx], S.Z[i * kLA + jx]);
        }
        __syncthreads();
    }
    if (mgs) {  // uniform.  Modified Gram-Schmidt in DESCENDING eigenvalue order (the
                // kept subspace's leading columns keep their span); a collapsed column is
                // completed by the unit vector with the most room outside the fixed ones.
        const int ci = ri;  // group of 8 lanes per column, rows rt + 8u
        if (tid < kEN) S.rowfill[tid] = 0.0;
        __syncthreads();
        for (int jp = n - 1; jp >= 0; --jp) {
            if (warp == 0) {
                double ss = 0.0;
                for (int r2 = lane; r2 < n; r2 += 32) ss = fma(S.Z[r2 * kLA + jp], S.Z[r2 * kLA + jp], ss);
                ss = warp_sum(ss);
                if (lane == 0) S.misc[5] = ss;
            }
            __syncthreads();
            double nrm2 = S.misc[5];
            if (!(nrm2 > 1e-4)) {  // collapsed (< 1% left)
                if (warp == 0) {
                    double best = -1.0;
                    int bm = 0;
                    for (int m = lane; m < n; m += 32) {
                        const double room = 1.0 - S.rowfill[m];
                        if (room > best) {
                            best = room;
                            bm = m;
                        }
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                        const int om = __shfl_xor_sync(0xffffffffu, bm, o);
                        if (ob > best || (ob == best && om < bm)) {
                            best = ob;
                            bm = om;
                        }
                    }
                    if (lane == 0) S.misc[6] = static_cast<double>(bm);
                }
                __syncthreads();
                const int m = static_cast<int>(S.misc[6]);
                if (tid < n) {  // v_r = δ_rm − Σ_{fixed f > jp} z_f[m] z_f[r]
                    double v = tid == m ? 1.0 : 0.0;
                    for (int f = jp + 1; f < n; ++f) v = fma(-S.Z[m * kLA + f], S.Z[tid * kLA + f], v);
                    S.p[tid] = v;
                }
                __syncthreads();
                if (tid < n) S.Z[tid * kLA + jp] = S.p[tid];
                if (warp == 0) {
                    double ss = 0.0;
                    for (int r2 = lane; r2 < n; r2 += 32) ss = fma(S.p[r2], S.p[r2], ss);
                    ss = warp_sum(ss);
                    if (lane == 0) S.misc[5] = ss;
                }
                __syncthreads();
                nrm2 = S.misc[5];
                if (!(nrm2 > 1e-16) && tid == 0) S.flag = 1;  // cannot complete: leave it to Jacobi
            }
            const double inv = nrm2 > 0.0 ? rsqrt(nrm2) : 0.0;
            if (tid < n) {
                const double z = S.Z[tid * kLA + jp] * inv;
                S.Z[tid * kLA + jp] = z;
                S.rowfill[tid] = fma(z, z, S.rowfill[tid]);
            }
            __syncthreads();
            if (ci < jp) {  // project the pivot out of the remaining columns
                double dz = 0.0;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int i = rt + 8 * u;
                    if (i < n) dz = fma(S.Z[i * kLA + jp], S.Z[i * kLA + ci], dz);
                }
                const unsigned gm8 = 0xffu << (lane & 24);  // this column's 8 lanes (the warp may diverge here)
                dz += __shfl_xor_sync(gm8, dz, 1);
                dz += __shfl_xor_sync(gm8, dz, 2);
                dz += __shfl_xor_sync(gm8, dz, 4);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int i = rt + 8 * u;
                    if (i < n) S.Z[i * kLA + ci] = fma(-dz, S.Z[i * kLA + jp], S.Z[i * kLA + ci]);
                }
            }
            __syncthreads();
        }
    }
    phase(4);

    // ---- 5b. R = C Z (C still in A: the tridiagonalisation ran in registers),
    // Rayleigh quotients, residual ‖R − ZΛ‖_F, descending order
    double* R = S.Lm;  // kEN-strided
    {
        const int g = lane >> 2, t = lane & 3;
        for (int tile = warp; tile < 64; tile += kEWarps) {
            const int r0 = 8 * (tile & 7), c0 = 8 * (tile >> 3);
            double c_0 = 0.0, c_1 = 0.0;
            for (int k0 = 0; k0 < n; k0 += 4) {
                const int kk = k0 + t;
                const double a = kk < n ? S.A[(r0 + g) * kLA + kk] : 0.0;
                const double b = kk < n ? S.Z[kk * kLA + c0 + g] : 0.0;
                dmma884(c_0, c_1, a, b);
            }
            R[(r0 + g) * kEN + c0 + 2 * t] = c_0;
            R[(r0 + g) * kEN + c0 + 2 * t + 1] = c_1;
        }
    }
    __syncthreads();
    {  // column j: 8 lanes; λ_j = z_jᵀ r_j, residual² = ‖r_j − λ_j z_j‖²
        const int j = ri;
        double zr = 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = rt + 8 * u;
            if (i < n && j < n) zr = fma(S.Z[i * kLA + j], R[i * kEN + j], zr);
        }
        zr += __shfl_xor_sync(0xffffffffu, zr, 1);
        zr += __shfl_xor_sync(0xffffffffu, zr, 2);
        zr += __shfl_xor_sync(0xffffffffu, zr, 4);
        double r2 = 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = rt + 8 * u;
            if (i < n && j < n) {
                const double r = fma(-zr, S.Z[i * kLA + j], R[i * kEN + j]);
                r2 = fma(r, r, r2);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r2 += __shfl_xor_sync(0xffffffffu, r2, o);
        if (lane == 0) S.red[warp] = r2;
        if (rt == 0 && j < n) S.lam[j] = zr;  // unscaled now
    }
    __syncthreads();
    if (tid < n) {  // rank in descending order (ties: lower index first)
        const double v = S.lam[tid];
        int rk = 0;
        for (int i = 0; i < n; ++i) {
            const double w = S.lam[i];
            rk += (w > v) || (w == v && i < tid);
        }
        S.rank[tid] = rk;
    }
    if (tid == 0) {
        double r2 = 0.0;
        for (int w = 0; w < kEWarps; ++w) r2 += S.red[w];
        const double res = sqrt(r2);
        // Backward-stable methods leave ~n·ε‖C‖; far more means a failure.
        if (!(res <= 1e-12 * tn)) S.flag = 1;
        if (resid_out) *resid_out = res;
    }
    __syncthreads();
    if (tid == 0 && S.flag) atomicOr(flag_out, 1);
    for (int idx = tid; idx < kEN * kEN; idx += kEThreads) {
        const int i = idx & 63, j = idx >> 6;
        if (i < n && j < n) V_out[i + static_cast<int64_t>(S.rank[j]) * n] = S.Z[i * kLA + j];
    }
    // Rejected vectors (an exactly multiple nonzero eigenvalue, say): their
    // Rayleigh quotients mean nothing, the multisection values still do.
    if (tid < n) lambda_out[S.flag ? n - 1 - tid : S.rank[tid]] = S.flag ? S.lamb[tid] * isc : S.lam[tid];
    phase(5);
}

// Eigenvalues only, n ≤ NR (plan stage, src/sketch.cpp:311-312: the eigenvalues
// of the energy-weighted Gram VᵀV; no vectors are needed).  The same register-
// resident tridiagonalisation as trd_eig_kernel with NR/8 columns per thread
// (only the current reflector is kept), then multisection to full precision:
// 16 rounds of 8 shifts (9^16 ≈ 2^51 of the Gershgorin width), λ descending.
template <int NR>
__global__ void __launch_bounds__(NR * 8, 1)
    eigvals_kernel(const double* __restrict__ Cin, int64_t ldc, int n, double* __restrict__ lambda_out) {
    constexpr int NT = NR * 8, NW = NT / 32, CPT = NR / 8;
    __shared__ __align__(16) double V[2][NR];
    __shared__ __align__(16) double P[NR];
    __shared__ __align__(16) double red[NW];
    __shared__ double dd[NR], ee[NR], tau[NR];
    __shared__ __align__(16) double2 de2[NR + 8];
    __shared__ double misc[4];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ri = tid >> 3, rt = tid & 7;
    const int gbase = lane & 24;
    const unsigned gm8 = 0xffu << gbase;
    double a[CPT];
#pragma unroll
    for (int u = 0; u < CPT; ++u) {
        const int j = rt + 8 * u;
        a[u] = (ri < n && j < n) ? 0.5 * (Cin[ri + static_cast<int64_t>(j) * ldc] + Cin[j + static_cast<int64_t>(ri) * ldc])
                                 : 0.0;
    }
    if (n == 1) {
        if (tid == 0) lambda_out[0] = a[0];
        return;
    }
    auto reflector = [&](int k) {  // the 8 lanes of row k; writes V[k & 1]
        double s0 = 0.0, s1 = 0.0, xa = 0.0, xd = 0.0;
#pragma unroll
        for (int u = 0; u < CPT; u += 2) {
            const int j = rt + 8 * u;
            s0 = (j > k + 1) ? fma(a[u], a[u], s0) : s0;
            s1 = (j + 8 > k + 1) ? fma(a[u + 1], a[u + 1], s1) : s1;
            xa = (j == k + 1) ? a[u] : ((j + 8 == k + 1) ? a[u + 1] : xa);
            xd = (j == k) ? a[u] : ((j + 8 == k) ? a[u + 1] : xd);
        }
        double ss = s0 + s1;
        ss += __shfl_xor_sync(gm8, ss, 1);
        ss += __shfl_xor_sync(gm8, ss, 2);
        ss += __shfl_xor_sync(gm8, ss, 4);
        const double alpha = __shfl_sync(gm8, xa, gbase + ((k + 1) & 7));
        const double dkk = __shfl_sync(gm8, xd, gbase + (k & 7));
        double tk = 0.0, beta = alpha, scale = 0.0;
        if (ss > 0.0) {
            beta = -copysign(sqrt_refined(fma(alpha, alpha, ss)), alpha);
            tk = fma(-alpha, rcp_refined(beta), 1.0);
            scale = rcp_refined(alpha - beta);
        }
        double* vb = V[k & 1];
#pragma unroll
        for (int u = 0; u < CPT; ++u) {
            const int j = rt + 8 * u;
            vb[j] = j == k + 1 ? 1.0 : (j > k + 1 ? a[u] * scale : 0.0);
        }
        if (rt == 0) {
            tau[k] = tk;
            dd[k] = dkk;
            ee[k] = beta;
        }
    };
    if (n > 2 && ri == 0) reflector(0);
    __syncthreads();
    for (int k = 0; k + 2 < n; ++k) {
        const double tk = tau[k];
        const double* vk = V[k & 1];
        const bool wact = 4 * warp + 3 > k && 4 * warp < n;
        double pr = 0.0, vi = 0.0;
        if (wact) {
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int u = 0; u < CPT; u += 2) {
                s0 = fma(a[u], vk[rt + 8 * u], s0);
                s1 = fma(a[u + 1], vk[rt + 8 * u + 8], s1);
            }
            pr = s0 + s1;
            pr += __shfl_xor_sync(0xffffffffu, pr, 1);
            pr += __shfl_xor_sync(0xffffffffu, pr, 2);
            pr += __shfl_xor_sync(0xffffffffu, pr, 4);
            vi = vk[ri];
            pr = ri > k ? tk * pr : 0.0;
            double pv = pr * vi;
            pv += __shfl_xor_sync(0xffffffffu, pv, 8);
            pv += __shfl_xor_sync(0xffffffffu, pv, 16);
            if (lane == 0) red[warp] = pv;
        } else if (lane == 0) {
            red[warp] = 0.0;
        }
        if (rt == 0) P[ri] = pr;
        __syncthreads();
        if (wact) {
            double pv2[NW];
#pragma unroll
            for (int w = 0; w < NW; w += 2) {
                const double2 t2 = *reinterpret_cast<const double2*>(&red[w]);
                pv2[w] = t2.x;
                pv2[w + 1] = t2.y;
            }
#pragma unroll
            for (int h = NW / 2; h > 0; h >>= 1)
#pragma unroll
                for (int w = 0; w < h; ++w) pv2[w] += pv2[w + h];
            const double K = 0.5 * tk * pv2[0];
            const double wi = fma(-K, vi, pr);
#pragma unroll
            for (int u = 0; u < CPT; ++u) {
                const int j = rt + 8 * u;
                const double vj = vk[j];
                a[u] -= fma(vi, fma(-K, vj, P[j]), wi * vj);
            }
        }
        if (k + 3 < n && ri == k + 1) reflector(k + 1);
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < CPT; ++u) {  // trailing 2×2
        const int j = rt + 8 * u;
        if (ri == n - 2 && j == n - 2) dd[n - 2] = a[u];
        if (ri == n - 1 && j == n - 1) dd[n - 1] = a[u];
        if (ri == n - 1 && j == n - 2) ee[n - 2] = a[u];
    }
    __syncthreads();
    if (warp == 0) {
        double lo = 1e300, hi = -1e300;
        for (int i = lane; i < n; i += 32) {
            const double off = (i > 0 ? fabs(ee[i - 1]) : 0.0) + (i + 1 < n ? fabs(ee[i]) : 0.0);
            lo = fmin(lo, dd[i] - off);
            hi = fmax(hi, dd[i] + off);
        }
        for (int o = 16; o > 0; o >>= 1) {
            lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        const double tn = fmax(fabs(lo), fabs(hi));
        const double sc = tn > 0.0 && isfinite(tn) ? inv_pow2_of(tn) : 1.0;
        for (int i = lane; i < NR + 8; i += 32) {
            const double ep = (i >= 1 && i < n) ? ee[i - 1] * sc : 0.0;
            de2[i] = make_double2(i < n ? dd[i] * sc : 8.0, ep * ep);
        }
        if (lane == 0) {
            const double pad = 8.0 * kEps * n;
            misc[0] = lo * sc - pad;
            misc[1] = hi * sc + pad;
            misc[2] = tn;
            misc[3] = 1.0 / sc;
        }
    }
    __syncthreads();
    const double tn = misc[2];
    if (!(tn > 0.0) || !isfinite(tn)) {
        if (tid < n) lambda_out[tid] = tn == 0.0 ? 0.0 : tn;  // zero matrix, or NaN/Inf passed through
        return;
    }
    const int j = ri;
    const int jj = j < n ? j : n - 1;
    double lo_b = misc[0], hi_b = misc[1];
    for (int it = 0; it < 16; ++it) {
        const double x = lo_b + (hi_b - lo_b) * (static_cast<double>(rt + 1) * (1.0 / 9.0));
        double pm = 1.0, pc = de2[0].x - x;
        unsigned sg = static_cast<unsigned>(__double2hiint(pc)) >> 31;
        int cnt = static_cast<int>(sg);
        for (int i0 = 1; i0 < n; i0 += 8) {
            double2 q[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) q[u] = de2[i0 + u];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const double pn = fma(q[u].x - x, pc, -q[u].y * pm);
                pm = pc;
                pc = pn;
                const unsigned sn = static_cast<unsigned>(__double2hiint(pc)) >> 31;
                cnt += static_cast<int>(sn ^ sg);
                sg = sn;
            }
            const double m = fmax(fabs(pc), fabs(pm));
            if (m > 0.0) {
                const double f = inv_pow2_of(m);
                pc *= f;
                pm *= f;
            }
        }
        const unsigned above = (__ballot_sync(0xffffffffu, cnt > jj) >> gbase) & 0xffu;
        const int first = above ? __ffs(above) - 1 : 8;
        const double x_hi = __shfl_sync(0xffffffffu, x, gbase + min(first, 7));
        const double x_lo = __shfl_sync(0xffffffffu, x, gbase + max(first - 1, 0));
        if (first < 8) hi_b = x_hi;
        if (first > 0) lo_b = x_lo;
    }
    if (rt == 0 && j < n) lambda_out[n - 1 - j] = 0.5 * (lo_b + hi_b) * misc[3];  // descending, unscaled
}

}  // namespace

bool jacobi_eig_forced() {
    static const bool on = [] {
        const char* e = std::getenv("TS_EIG");
        return e && std::string(e) == "jacobi";
    }();
    return on;
}

bool launch_sym_eigvals(const double* C, int64_t ldc, int n, double* lambda, CallScratch& sc) {
    if (n < 1 || n > 128) return false;
    if (n <= 64) eigvals_kernel<64><<<1, 512, 0, sc.stream()>>>(C, ldc, n, lambda);
    else eigvals_kernel<128><<<1, 1024, 0, sc.stream()>>>(C, ldc, n, lambda);
    TS_LAUNCH_CHECK();
    sc.launches += 1;
    return true;
}

bool launch_sym_trd(const double* C, int64_t ldc, int n, double* lambda, double* V, int* flag, double* resid,
                    CallScratch& sc, int count, int64_t strideC, int64_t strideL, int64_t strideV) {
    if (n < 1 || n > kEN) return false;
    if (count < 1) return true;
    set_max_smem(trd_eig_kernel, static_cast<int>(sizeof(TrdSmem)));
    static const int variant = [] {  // timing ablations of the tridiagonalisation (tools/probe_trd.py)
        const char* e = std::getenv("TS_TRD_VARIANT");
        return e ? std::atoi(e) : 0;
    }();
    trd_eig_kernel<<<count, kEThreads, sizeof(TrdSmem), sc.stream()>>>(C, ldc, n, lambda, V, flag, resid,
                                                                       eig_probe_buffer(), strideC, strideL, strideV,
                                                                       variant);
    TS_LAUNCH_CHECK();
    sc.launches += 1;
    return true;
}

}  // namespace ts
