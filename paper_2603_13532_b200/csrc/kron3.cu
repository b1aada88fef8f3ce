// kron3.cu — stage B of the Kronecker sketch for order-3 summands, fused
// (reference src/sketch.cpp:132-140, krp = false).  For atom b with core G
// (r0 × r1 × r2) and M_j = Ω_jᵀU_j (s_j × r_j, the atom's column slice of Z_j),
// the three mode sketches are
//   V0[a0, c1 + s1·c2] = Σ_{a1,a2} G[a0,a1,a2] M1[c1,a1] M2[c2,a2]
//   V1[a1, c0 + s0·c2] = Σ_{a0,a2} G[a0,a1,a2] M0[c0,a0] M2[c2,a2]
//   V2[a2, c0 + s0·c1] = Σ_{a0,a1} M0[c0,a0] G[a0,a1,a2] M1[c1,a1]
// (the mode-n unfolding of G ×_{j≠n} M_j, other modes lowest-first).  Per core
// slice G_s = G[:, :, a2] the CTA forms T = G_s·M1ᵀ (r0 × s1) and U = M0·G_s
// (s0 × r1) once; V0 and V1 accumulate M2[:, a2]-weighted copies of them in
// registers and V2's row a2 is M0·T.  One CTA per atom, slices streamed with
// cp.async (double-buffered); the weighted transposes go straight into Wt_n
// (C_n × R_n).  The generic path (capi.cu kron_stage_b) runs a chain of grouped
// GEMM launches per mode instead.
#include "kernels.cuh"

namespace ts {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxR = 32;   // block ranks
constexpr int kMaxC = 96;   // sketch columns per mode (Π of the other widths)
constexpr int kVPT = kMaxR * kMaxC / kThreads;  // V0 / V1 entries per thread (12)

__global__ void __launch_bounds__(kThreads) kron3_kernel(Kron3Args args) {
    const Atom& at = args.atoms[blockIdx.x];
    const int r0 = at.shape[0], r1 = at.shape[1], r2 = at.shape[2];
    const int s0 = args.s[0], s1 = args.s[1], s2 = args.s[2];
    const int C0 = s1 * s2, C1 = s0 * s2, C2 = s0 * s1;
    const int tid = threadIdx.x;
    extern __shared__ __align__(16) double sm[];
    double* M0 = sm;                 // s0 × r0, [c][a]
    double* M1 = M0 + s0 * r0;       // s1 × r1
    double* M2 = M1 + s1 * r1;       // s2 × r2
    double* Gs = M2 + s2 * r2;       // 2 × r0·r1 (column-major slices)
    double* T = Gs + 2 * r0 * r1;    // r0 × s1, [a0 + r0·c1]
    double* U = T + r0 * s1;         // s0 × r1, [c0 + s0·a1]
    for (int i = tid; i < s0 * r0; i += kThreads) {
        const int c = i % s0, a = i / s0;
        M0[c + s0 * a] = args.Z[0][c + static_cast<int64_t>(at.col[0] + a) * s0];
    }
    for (int i = tid; i < s1 * r1; i += kThreads) {
        const int c = i % s1, a = i / s1;
        M1[c + s1 * a] = args.Z[1][c + static_cast<int64_t>(at.col[1] + a) * s1];
    }
    for (int i = tid; i < s2 * r2; i += kThreads) {
        const int c = i % s2, a = i / s2;
        M2[c + s2 * a] = args.Z[2][c + static_cast<int64_t>(at.col[2] + a) * s2];
    }
    const double* core = args.cores + at.core_off;
    const int slice = r0 * r1;
    auto load_slice = [&](int a2, int buf) {
        const double* src = core + static_cast<int64_t>(a2) * slice;
        for (int i = tid; i < slice; i += kThreads) cp_async8(Gs + buf * slice + i, src + i, 8);
    };
    double v0[kVPT], v1[kVPT];
#pragma unroll
    for (int e = 0; e < kVPT; ++e) v0[e] = v1[e] = 0.0;
    const double w = args.weights[at.summand];
    double* W2 = args.W[2];
    const int64_t ld2 = C2;

    if (r2 > 0) load_slice(0, 0);
    cp_async_commit();
    for (int a2 = 0; a2 < r2; ++a2) {
        const int buf = a2 & 1;
        if (a2 + 1 < r2) load_slice(a2 + 1, buf ^ 1);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        const double* G = Gs + buf * slice;
        // T = G_s · M1ᵀ (r0 × s1) and U = M0 · G_s (s0 × r1).
        for (int i = tid; i < r0 * s1; i += kThreads) {
            const int a0 = i % r0, c1 = i / r0;
            double acc = 0.0;
            for (int a1 = 0; a1 < r1; ++a1) acc = fma(G[a0 + r0 * a1], M1[c1 + s1 * a1], acc);
            T[i] = acc;
        }
        for (int i = tid; i < s0 * r1; i += kThreads) {
            const int c0 = i % s0, a1 = i / s0;
            double acc = 0.0;
            for (int a0 = 0; a0 < r0; ++a0) acc = fma(M0[c0 + s0 * a0], G[a0 + r0 * a1], acc);
            U[i] = acc;
        }
        __syncthreads();
        // V0[a0, c1 + s1·c2] += M2[c2, a2]·T[a0, c1];  V1[a1, c0 + s0·c2] += M2[c2, a2]·U[c0, a1].
#pragma unroll
        for (int e = 0; e < kVPT; ++e) {
            const int i = tid + kThreads * e;
            if (i < r0 * C0) {
                const int a0 = i % r0, c = i / r0, c1 = c % s1, c2 = c / s1;
                v0[e] = fma(M2[c2 + s2 * a2], T[a0 + r0 * c1], v0[e]);
            }
            if (i < r1 * C1) {
                const int a1 = i % r1, c = i / r1, c0 = c % s0, c2 = c / s0;
                v1[e] = fma(M2[c2 + s2 * a2], U[c0 + s0 * a1], v1[e]);
            }
        }
        // Row a2 of V2: (M0 · T)[c0, c1] → Wt_2[c0 + s0·c1, col2 + a2].
        for (int i = tid; i < C2; i += kThreads) {
            const int c0 = i % s0, c1 = i / s0;
            double acc = 0.0;
            for (int a0 = 0; a0 < r0; ++a0) acc = fma(M0[c0 + s0 * a0], T[a0 + r0 * c1], acc);
            W2[i + ld2 * (at.col[2] + a2)] = w * acc;
        }
        __syncthreads();  // T / U / slice buffer reuse
    }
    cp_async_wait<0>();
    double* W0 = args.W[0];
    double* W1 = args.W[1];
#pragma unroll
    for (int e = 0; e < kVPT; ++e) {
        const int i = tid + kThreads * e;
        if (i < r0 * C0) {
            const int a0 = i % r0, c = i / r0;
            W0[c + static_cast<int64_t>(C0) * (at.col[0] + a0)] = w * v0[e];
        }
        if (i < r1 * C1) {
            const int a1 = i % r1, c = i / r1;
            W1[c + static_cast<int64_t>(C1) * (at.col[1] + a1)] = w * v1[e];
        }
    }
}

}  // namespace

bool launch_kron3(const Kron3Args& args, int max_shape, CallScratch& sc) {
    if (args.natoms == 0) return true;
    const int s0 = args.s[0], s1 = args.s[1], s2 = args.s[2];
    if (max_shape > kMaxR || s1 * s2 > kMaxC || s0 * s2 > kMaxC || s0 * s1 > kMaxC) return false;
    const size_t smem = sizeof(double) * (static_cast<size_t>(s0 + s1 + s2) * kMaxR + 2 * kMaxR * kMaxR +
                                          static_cast<size_t>(kMaxR) * (s1 + s0));
    set_max_smem(kron3_kernel, 200 * 1024);
    kron3_kernel<<<static_cast<unsigned>(args.natoms), kThreads, smem, sc.stream()>>>(args);
    TS_LAUNCH_CHECK();
    sc.launches += 1;
    return true;
}

}  // namespace ts
