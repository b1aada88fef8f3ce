// ttm3.cu — stage F1 for order-3 summands: the core projection's first two
// mode products fused per core slice (reference src/sketch.cpp:161-166):
//   T_b[:, :, a2] = w_b · P_0,b · G_b[:, :, a2] · P_1,bᵀ       (q0 × q1 per slice)
// with P_n,b = (Û_nᵀ U_n)[:, cols of atom b].  The result goes straight into
// column col_b[2] + a2 of T_stack (Π q × R_2), whose product with P_2ᵀ (stage F2)
// then sums over all summands as one GEMM.  One CTA per (atom, 8 slices): the
// two projected factor blocks stay in shared memory, each slice streams in via
// cp.async (double-buffered) and both GEMMs of the chain run on DMMA.8x8x4.
#include <algorithm>

#include "kernels.cuh"

namespace ts {
namespace {

constexpr int kThreads = 128;
constexpr int kR = 32;          // padded r0 = r1
constexpr int kQ = 64;          // padded q0 = q1
constexpr int kLQ = kQ + 4;     // [k][m] stride for P0s, Xs, P1s (conflict-free fragments)
constexpr int kLG = kR + 4;     // slice stride ([a1][a0], a0 contiguous)
constexpr int kSPC = 8;         // slices per CTA

__global__ void __launch_bounds__(kThreads) ttm3_kernel(Ttm3Args args) {
    const Atom& at = args.atoms[blockIdx.x];
    const int r0 = at.shape[0], r1 = at.shape[1], r2 = at.shape[2];
    const int s_begin = blockIdx.y * kSPC;
    if (s_begin >= r2) return;
    const int s_end = min(r2, s_begin + kSPC);
    const int q0 = static_cast<int>(args.q[0]), q1 = static_cast<int>(args.q[1]);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;

    extern __shared__ __align__(16) double sm[];
    double* P0s = sm;                   // [a0][i0]  (A of GEMM 1: m = i0, k = a0)
    double* P1s = P0s + kR * kLQ;       // [a1][i1]  (B of GEMM 2: k = a1, n = i1)
    double* Xs = P1s + kR * kLQ;        // [a1][i0]  (A of GEMM 2: m = i0, k = a1)
    double* Gs = Xs + kR * kLQ;         // 2 × [a1][a0] (B of GEMM 1: k = a0, n = a1)
    const double* P0 = args.P[0];
    const double* P1 = args.P[1];
    for (int idx = tid; idx < kR * kQ; idx += kThreads) {
        const int a = idx / kQ, i = idx % kQ;
        P0s[a * kLQ + i] = (a < r0 && i < q0) ? P0[i + static_cast<int64_t>(at.col[0] + a) * q0] : 0.0;
        P1s[a * kLQ + i] = (a < r1 && i < q1) ? P1[i + static_cast<int64_t>(at.col[1] + a) * q1] : 0.0;
    }
    for (int idx = tid; idx < 2 * kR * kLG; idx += kThreads) Gs[idx] = 0.0;
    __syncthreads();
    const double* __restrict__ core = args.cores + at.core_off;
    const int slice = r0 * r1;
    auto load_slice = [&](int a2, int buf) {
        double* dst = Gs + buf * kR * kLG;
        const double* src = core + static_cast<int64_t>(a2) * slice;
        for (int idx = tid; idx < slice; idx += kThreads) {
            const int a0 = idx % r0, a1 = idx / r0;
            cp_async8(dst + a1 * kLG + a0, src + idx, 8);
        }
    };
    const double w = args.weights[at.summand];
    double* __restrict__ T = args.Tstack;
    const int64_t Qp = args.Qp;
    // GEMM 1 tiling: warp w → rows 16w..16w+15 of X (2 groups), all 32 columns (4 groups).
    // GEMM 2 tiling: 2×2 warps of 32×32 over T (64×64).
    const int wm2 = warp & 1, wn2 = warp >> 1;

    // Running maxima of |T| per output (i0, i1) over this CTA's slices, as the high
    // words of the doubles (monotone for non-negative values): the row exponent
    // bounds stage F2's int8 engine needs, without another pass over T_stack.
    const bool track = args.rowexp != nullptr;
    int mxh[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) mxh[i][j][0] = mxh[i][j][1] = 0;

    load_slice(s_begin, 0);
    cp_async_commit();
    for (int a2 = s_begin; a2 < s_end; ++a2) {
        const int buf = (a2 - s_begin) & 1;
        if (a2 + 1 < s_end) load_slice(a2 + 1, buf ^ 1);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        const double* G = Gs + buf * kR * kLG;
        // ---- X = P0b · G_s   (64 × 32, K = 32)
        double x[2][4][2];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) x[i][j][0] = x[i][j][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < kR; kk += 4) {
            double af[2], bf[4];
#pragma unroll
            for (int i = 0; i < 2; ++i) af[i] = P0s[(kk + t) * kLQ + warp * 16 + i * 8 + g];
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = G[(j * 8 + g) * kLG + kk + t];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma884(x[i][j][0], x[i][j][1], af[i], bf[j]);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) Xs[(j * 8 + 2 * t + h) * kLQ + warp * 16 + i * 8 + g] = x[i][j][h];
        __syncthreads();
        // ---- T_s = X · P1bᵀ   (64 × 64, K = 32)
        double acc[4][4][2];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < kR; kk += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = Xs[(kk + t) * kLQ + wm2 * 32 + i * 8 + g];
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = P1s[(kk + t) * kLQ + wn2 * 32 + j * 8 + g];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
        double* out = T + static_cast<int64_t>(at.col[2] + a2) * Qp;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int i0 = wm2 * 32 + i * 8 + g, i1 = wn2 * 32 + j * 8 + 2 * t + h;
                    const double val = w * acc[i][j][h];
                    if (i0 < q0 && i1 < q1) out[i0 + static_cast<int64_t>(i1) * q0] = val;
                    if (track) mxh[i][j][h] = max(mxh[i][j][h], __double2hiint(val) & 0x7fffffff);
                }
        __syncthreads();  // Xs / slice buffer reuse
    }
    cp_async_wait<0>();
    if (track) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int i0 = wm2 * 32 + i * 8 + g, i1 = wn2 * 32 + j * 8 + 2 * t + h;
                    if (i0 >= q0 || i1 >= q1) continue;
                    // biased exponent b: 2^(b-1023) ≤ max < 2^(b-1022); zero / subnormal → the floor
                    const int bexp = mxh[i][j][h] >> 20;
                    const int e = bexp > 0 ? max(bexp - 1022, kOzExpFloor) : kOzExpFloor;
                    // kTtmExpBuckets copies of the bounds (bucket = atom mod 16) keep the first
                    // wave's same-address atomics short; launch_reduce_exponents folds them.
                    int* slot = args.rowexp + (blockIdx.x % kTtmExpBuckets) * args.Qp + i0 + static_cast<int64_t>(i1) * q0;
                    if (e > *reinterpret_cast<volatile int*>(slot)) atomicMax(slot, e);
                }
    }
}

}  // namespace

bool launch_ttm3(const Ttm3Args& args, int max_shape, int max_r2, CallScratch& sc) {
    if (args.natoms == 0) return true;
    if (max_shape > kR || args.q[0] > kQ || args.q[1] > kQ) return false;
    const size_t smem = sizeof(double) * (3 * kR * kLQ + 2 * kR * kLG);
    // Per-device, thread-safe smem attribute (runtime.hpp set_max_smem).
    set_max_smem(ttm3_kernel, static_cast<int>(smem));
    dim3 grid(static_cast<unsigned>(args.natoms), static_cast<unsigned>((max_r2 + kSPC - 1) / kSPC));
    ttm3_kernel<<<grid, kThreads, smem, sc.stream()>>>(args);
    TS_LAUNCH_CHECK();
    sc.launches += 1;
    return true;
}

}  // namespace ts
