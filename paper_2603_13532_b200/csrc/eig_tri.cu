// eig_tri.cu — symmetric eigensolver of ST-HOSVD's Gram fast path (stage G) by
// tridiagonalization, for n ≤ 64 in ONE kernel (one CTA):
//
//   1. Householder tridiagonalization Qᵀ C Q = T (LAPACK dsytd2 order, lower),
//      the matrix in shared memory, three CTA barriers per reflector;
//   2. all eigenvalues of T by multisection: each warp brackets four
//      eigenvalues at once (one Sturm-count chain per eigenvalue and lane, 32
//      shifts per eigenvalue and round → 5 bits per round);
//   3. eigenvectors of T by inverse iteration on the LDLᵀ factorisation of
//      T − λI, with Gram-Schmidt inside clusters (|λ_i − λ_j| ≤ 1e-3‖T‖, the
//      dstein rule) so clustered vectors stay orthogonal;
//   4. back-transformation Z ← Q Z, each warp applying all reflectors to its
//      own columns (no CTA barrier);
//   5. an acceptance check on the ORIGINAL matrix: every residual
//      ‖C z − λ z‖ ≤ 1e-13‖C‖_F and |ZᵀZ − I| ≤ 1e-12, else *flag |= 1 and the
//      caller recomputes with the two-sided Jacobi kernel (eig.cu).
//
// Reference semantics are those of sym_eig (src/kernels.cpp:70-86): symmetrise,
// eigendecompose, descending order.  The Jacobi solver needs ~8 sweeps × (n-1)
// rounds whose latency is a dependent rotation chain plus a CTA barrier; this
// path needs (n-2) reflector steps and a fixed number of bisection rounds.
#include <cmath>
#include <cstdlib>
#include <string>

#include "kernels.cuh"

namespace ts {
namespace {

constexpr int kTriThreads = 512;
constexpr int kTriWarps = kTriThreads / 32;
constexpr int kTN = 64;       // largest n
constexpr int kLA = kTN + 1;  // row stride of A and Z (conflict-free column walks)
constexpr double kEps = 1.1102230246251565e-16;

// ~40-bit reciprocal (MUFU approximation + one Newton step): enough for the
// signs of a Sturm sequence.
__device__ __forceinline__ double rcp_newton(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return y * fma(-x, y, 2.0);
}

struct TriSmem {
    double A[kTN * kLA];   // working matrix (full symmetric), row-major [i][j]
    double Z[kTN * kLA];   // eigenvectors, [row][col]
    double V[kTN * kTN];   // reflector k contiguous: V[k * kTN + i], rows k+1..n-1 (v_{k+1} = 1)
    double Dinv[kTN * kTN];  // inverse iteration: 1/D_i of eigenvalue t at [i * kTN + t]
    double Lm[kTN * kTN];    //                    L_i at [i * kTN + t]
    double tau[kTN], d[kTN], e[kTN], e2[kTN], lam[kTN], p[kTN];
    double red[kTriWarps];
    double misc[8];
    int flag;
};

__global__ void __launch_bounds__(kTriThreads, 1) tri_eig_kernel(const double* __restrict__ Cin, int64_t ldc, int n,
                                                                 double* __restrict__ lambda_out,
                                                                 double* __restrict__ V_out, int* __restrict__ flag_out,
                                                                 unsigned long long* __restrict__ prof) {
    extern __shared__ __align__(16) unsigned char smraw[];
    TriSmem& S = *reinterpret_cast<TriSmem*>(smraw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    // ---- load + symmetrise
    for (int idx = tid; idx < n * n; idx += kTriThreads) {
        const int i = idx % n, j = idx / n;
        S.A[i * kLA + j] = 0.5 * (Cin[i + static_cast<int64_t>(j) * ldc] + Cin[j + static_cast<int64_t>(i) * ldc]);
    }
    if (tid == 0) S.flag = 0;
    __syncthreads();
    // Optional phase clocks (TS_EIG_PROFILE): prof[10 + phase] += cycles.
    long long tmark = clock64();
    auto phase = [&](int ph) {
        if (prof != nullptr && tid == 0) {
            const long long now = clock64();
            prof[10 + ph] = static_cast<unsigned long long>(now - tmark);
            tmark = now;
        }
    };

    // ---- 1. tridiagonalization
    for (int k = 0; k + 2 < n; ++k) {
        const int r0 = k + 1;  // first row of the reflector
        if (warp == 0) {
            // x = A[r0.., k]; dlarfg: beta = -sign(x0)‖x‖, tau = (beta - x0)/beta, v = x / (x0 - beta), v0 = 1.
            double ss = 0.0;
            for (int i = r0 + 1 + lane; i < n; i += 32) {
                const double x = S.A[i * kLA + k];
                ss = fma(x, x, ss);
            }
            ss = warp_sum(ss);
            const double x0 = S.A[r0 * kLA + k];
            double tau = 0.0, beta = x0, scale = 0.0;
            if (ss > 0.0) {
                beta = -copysign(sqrt(fma(x0, x0, ss)), x0);
                tau = (beta - x0) / beta;
                scale = 1.0 / (x0 - beta);
            }
            for (int i = r0 + lane; i < n; i += 32) S.V[k * kTN + i] = i == r0 ? 1.0 : S.A[i * kLA + k] * scale;
            if (lane == 0) {
                S.tau[k] = tau;
                S.d[k] = S.A[k * kLA + k];
                S.e[k] = beta;
            }
        }
        __syncthreads();
        // p = tau · A22 v (rows r0..n-1): 8 threads per row, 3-shuffle reduction.
        const double tau = S.tau[k];
        {
            const int i = r0 + (tid >> 3), c = tid & 7;
            double acc = 0.0;
            if (i < n)
                for (int j = r0 + c; j < n; j += 8) acc = fma(S.A[i * kLA + j], S.V[k * kTN + j], acc);
            acc += __shfl_xor_sync(0xffffffffu, acc, 1);
            acc += __shfl_xor_sync(0xffffffffu, acc, 2);
            acc += __shfl_xor_sync(0xffffffffu, acc, 4);
            if (i < n && c == 0) S.p[i] = tau * acc;
        }
        __syncthreads();
        // w = p - (tau/2)(pᵀv) v ; A22 -= v wᵀ + w vᵀ.  Every warp forms pᵀv itself.
        double pv = 0.0;
        for (int j = r0 + lane; j < n; j += 32) pv = fma(S.p[j], S.V[k * kTN + j], pv);
        pv = warp_sum(pv);
        const double K = 0.5 * tau * pv;
        const int m = n - r0;
        for (int idx = tid; idx < m * m; idx += kTriThreads) {
            const int i = r0 + idx / m, j = r0 + idx % m;
            const double vi = S.V[k * kTN + i], vj = S.V[k * kTN + j];
            const double wi = S.p[i] - K * vi, wj = S.p[j] - K * vj;
            S.A[i * kLA + j] -= fma(vi, wj, wi * vj);
        }
        __syncthreads();
    }
    if (tid == 0) {
        if (n >= 2) {
            S.d[n - 2] = S.A[(n - 2) * kLA + (n - 2)];
            S.e[n - 2] = S.A[(n - 1) * kLA + (n - 2)];
        }
        S.d[n - 1] = S.A[(n - 1) * kLA + (n - 1)];
    }
    __syncthreads();
    phase(0);
    if (tid < n - 1) S.e2[tid] = S.e[tid] * S.e[tid];
    if (warp == 0) {
        // Gershgorin bounds and pivmin.
        double lo = 1e300, hi = -1e300, me2 = 0.0;
        for (int i = lane; i < n; i += 32) {
            const double off = (i > 0 ? fabs(S.e[i - 1]) : 0.0) + (i + 1 < n ? fabs(S.e[i]) : 0.0);
            lo = fmin(lo, S.d[i] - off);
            hi = fmax(hi, S.d[i] + off);
            if (i + 1 < n) me2 = fmax(me2, S.e[i] * S.e[i]);
        }
        for (int o = 16; o > 0; o >>= 1) {
            lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
            me2 = fmax(me2, __shfl_xor_sync(0xffffffffu, me2, o));
        }
        if (lane == 0) {
            const double tn = fmax(fabs(lo), fabs(hi));
            const double pad = 2.0 * kEps * tn * n + 1e-300;
            S.misc[0] = lo - pad;
            S.misc[1] = hi + pad;
            S.misc[2] = tn;
            S.misc[3] = 1e-290 * fmax(1.0, me2);
        }
    }
    __syncthreads();

    // ---- 2. eigenvalues: warp w brackets eigenvalues 4w .. 4w+3 (ascending)
    {
        const double tn = S.misc[2], pivmin = S.misc[3];
        const double atol = 2.0 * kEps * tn;
        double a[4], b[4];
        int jj[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            a[u] = S.misc[0];
            b[u] = S.misc[1];
            jj[u] = min(4 * warp + u, n - 1);
        }
        for (int it = 0; it < 24; ++it) {
            bool open = false;
#pragma unroll
            for (int u = 0; u < 4; ++u) open |= (b[u] - a[u]) > fmax(atol, 2.0 * kEps * fmax(fabs(a[u]), fabs(b[u])));
            if (!open) break;  // warp-uniform
            int c[4];
            double sg[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) sg[u] = a[u] + (b[u] - a[u]) * (static_cast<double>(lane + 1) / 33.0);
            // Four independent Sturm chains per lane (instruction-level parallelism).
            {
                double q[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    q[u] = S.d[0] - sg[u];
                    c[u] = q[u] < 0.0;
                }
                for (int i = 1; i < n; ++i) {
                    const double di = S.d[i], ei = S.e2[i - 1];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        if (fabs(q[u]) < pivmin) q[u] = -pivmin;
                        q[u] = (di - sg[u]) - ei * rcp_newton(q[u]);
                        c[u] += q[u] < 0.0;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const unsigned above = __ballot_sync(0xffffffffu, c[u] > jj[u]);
                const double lo_s = __shfl_sync(0xffffffffu, sg[u], max(__ffs(above) - 2, 0));
                const double hi_s = __shfl_sync(0xffffffffu, sg[u], above ? __ffs(above) - 1 : 31);
                if (above == 0u) {
                    a[u] = hi_s;  // every shift is still at or below the eigenvalue
                } else {
                    if (__ffs(above) >= 2) a[u] = lo_s;
                    b[u] = hi_s;
                }
            }
        }
        if (lane == 0) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (4 * warp + u < n) S.lam[4 * warp + u] = 0.5 * (a[u] + b[u]);
        }
    }
    __syncthreads();

    phase(1);
    // ---- 3. eigenvectors of T: inverse iteration, thread t for eigenvalue t
    const double tn = S.misc[2];
    if (tid < n) {
        const int j = tid;
        const double pivtol = kEps * fmax(tn, 1e-300);
        const double sigma = S.lam[j];
        // LDLᵀ of T − σI (no pivoting; zero pivots nudged to ±pivtol).
        double Dp = S.d[0] - sigma;
        if (fabs(Dp) < pivtol) Dp = Dp < 0.0 ? -pivtol : pivtol;
        double Di = 1.0 / Dp;
        S.Dinv[j] = Di;
        for (int i = 0; i + 1 < n; ++i) {
            const double l = S.e[i] * Di;
            S.Lm[i * kTN + j] = l;
            Dp = (S.d[i + 1] - sigma) - l * S.e[i];
            if (fabs(Dp) < pivtol) Dp = Dp < 0.0 ? -pivtol : pivtol;
            Di = 1.0 / Dp;
            S.Dinv[(i + 1) * kTN + j] = Di;
        }
        // Start vector: deterministic, distinct per eigenvalue.
        for (int i = 0; i < n; ++i) {
            const unsigned h = (static_cast<unsigned>(i) * 2654435761u) ^ (static_cast<unsigned>(j + 1) * 40503u);
            S.Z[i * kLA + j] = 1.0 + 0.5 * (static_cast<double>(h & 0xffffu) / 65535.0 - 0.5);
        }
        for (int it = 0; it < 3; ++it) {
            // L y = x, z = D⁻¹ y, Lᵀ x = z, normalise.
            double y = S.Z[j];
            for (int i = 1; i < n; ++i) {
                y = fma(-S.Lm[(i - 1) * kTN + j], y, S.Z[i * kLA + j]);
                S.Z[i * kLA + j] = y;
            }
            double x = y * S.Dinv[(n - 1) * kTN + j];
            S.Z[(n - 1) * kLA + j] = x;
            double nrm = x * x;
            for (int i = n - 2; i >= 0; --i) {
                x = fma(S.Z[i * kLA + j], S.Dinv[i * kTN + j], -S.Lm[i * kTN + j] * x);
                S.Z[i * kLA + j] = x;
                nrm = fma(x, x, nrm);
            }
            const double inv = nrm > 0.0 ? rsqrt(nrm) : 0.0;
            for (int i = 0; i < n; ++i) S.Z[i * kLA + j] *= inv;
        }
    }
    __syncthreads();
    phase(2);
    // Clusters (|λ_{j+1} − λ_j| ≤ 1e-3‖T‖, the dstein rule): classical Gram-Schmidt
    // twice, member by member, against the cluster's earlier vectors.
    {
        const double ortol = 1e-3 * tn;
        for (int j = 1; j < n; ++j) {
            if (!(S.lam[j] - S.lam[j - 1] <= ortol)) continue;  // uniform: lam is shared
            int first = j - 1;
            while (first > 0 && S.lam[first] - S.lam[first - 1] <= ortol) --first;
            for (int pass = 0; pass < 2; ++pass) {
                // d_q = z_qᵀ z_j for q in [first, j): warp per q.
                for (int q = first + warp; q < j; q += kTriWarps) {
                    double dot = 0.0;
                    for (int i = lane; i < n; i += 32) dot = fma(S.Z[i * kLA + q], S.Z[i * kLA + j], dot);
                    dot = warp_sum(dot);
                    if (lane == 0) S.p[q] = dot;
                }
                __syncthreads();
                double zi = 0.0;
                if (tid < n) {
                    zi = S.Z[tid * kLA + j];
                    for (int q = first; q < j; ++q) zi = fma(-S.p[q], S.Z[tid * kLA + q], zi);
                }
                double sq = warp_sum(zi * zi);
                if (lane == 0 && warp < 2) S.red[warp] = sq;
                __syncthreads();
                const double inv = rsqrt(S.red[0] + (n > 32 ? S.red[1] : 0.0));
                if (tid < n) S.Z[tid * kLA + j] = zi * inv;
                __syncthreads();
            }
        }
    }

    phase(3);
    // ---- 4. back-transformation: Z ← H_0 ⋯ H_{n-3} Z, warp w owns columns w, w+16, ...
    {
        int cols[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) cols[u] = min(warp + u * kTriWarps, n - 1);  // duplicates are dropped below
        const int ncols = n > warp ? (n - warp + kTriWarps - 1) / kTriWarps : 0;
        for (int k = n - 3; k >= 0; --k) {
            const int r0 = k + 1;
            double s[4] = {0.0, 0.0, 0.0, 0.0};
            for (int i = r0 + lane; i < n; i += 32) {
                const double v = S.V[k * kTN + i];
#pragma unroll
                for (int u = 0; u < 4; ++u) s[u] = fma(v, S.Z[i * kLA + cols[u]], s[u]);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) s[u] = warp_sum(s[u]) * S.tau[k];
            __syncwarp();
            for (int i = r0 + lane; i < n; i += 32) {
                const double v = S.V[k * kTN + i];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (u < ncols) S.Z[i * kLA + cols[u]] = fma(-s[u], v, S.Z[i * kLA + cols[u]]);
            }
            __syncwarp();
        }
    }
    __syncthreads();

    phase(4);
    // ---- 5. acceptance on the original matrix + output (descending order)
    {
        // The symmetrised C again (the working copy was consumed) and ‖C‖_F.
        double cf = 0.0;
        for (int idx = tid; idx < n * n; idx += kTriThreads) {
            const int i = idx % n, j = idx / n;
            const double v = 0.5 * (Cin[i + static_cast<int64_t>(j) * ldc] + Cin[j + static_cast<int64_t>(i) * ldc]);
            S.A[i * kLA + j] = v;
            cf = fma(v, v, cf);
        }
        cf = warp_sum(cf);
        if (lane == 0) S.red[warp] = cf;
        __syncthreads();
        double cfro = 0.0;
        for (int w = 0; w < kTriWarps; ++w) cfro += S.red[w];
        cfro = sqrt(cfro);
        bool bad = false;
        // Residual of eigenpair j (warp per eigenpair): ‖(C z_j)_i − λ_j z_ij‖.
        for (int j = warp; j < n; j += kTriWarps) {
            double r2 = 0.0;
            for (int i = lane; i < n; i += 32) {
                double acc = -S.lam[j] * S.Z[i * kLA + j];
                for (int t = 0; t < n; ++t) acc = fma(S.A[i * kLA + t], S.Z[t * kLA + j], acc);
                r2 = fma(acc, acc, r2);
            }
            r2 = warp_sum(r2);
            bad |= !(sqrt(r2) <= 1e-13 * cfro + 1e-300);
        }
        // Orthogonality |z_aᵀ z_b − δ_ab| (thread per pair, upper triangle).
        for (int idx = tid; idx < n * n; idx += kTriThreads) {
            const int a_ = idx % n, b_ = idx / n;
            if (a_ > b_) continue;
            double dot = 0.0;
            for (int i = 0; i < n; ++i) dot = fma(S.Z[i * kLA + a_], S.Z[i * kLA + b_], dot);
            bad |= !(fabs(dot - (a_ == b_ ? 1.0 : 0.0)) <= 1e-12);
        }
        if (bad) atomicOr(&S.flag, 1);
        __syncthreads();
        if (tid == 0 && S.flag) atomicOr(flag_out, 1);
        for (int idx = tid; idx < n * n; idx += kTriThreads) {
            const int i = idx % n, r = idx / n;  // output column r = eigenvalue n-1-r
            V_out[i + static_cast<int64_t>(r) * n] = S.Z[i * kLA + (n - 1 - r)];
        }
        if (tid < n) lambda_out[tid] = S.lam[n - 1 - tid];
        __syncthreads();
        phase(5);
    }
}

}  // namespace

bool tri_eig_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("TS_EIG");
        return e && std::string(e) == "tri";  // opt-in: slower than the Jacobi kernel on this GPU
    }();
    return on;
}

bool launch_sym_tridiag(const double* C, int64_t ldc, int n, double* lambda, double* V, int* flag, CallScratch& sc) {
    if (n < 1 || n > kTN) return false;
    set_max_smem(tri_eig_kernel, static_cast<int>(sizeof(TriSmem)));
    tri_eig_kernel<<<1, kTriThreads, sizeof(TriSmem), sc.stream()>>>(C, ldc, n, lambda, V, flag, eig_probe_buffer());
    TS_LAUNCH_CHECK();
    sc.launches += 1;
    return true;
}

}  // namespace ts
