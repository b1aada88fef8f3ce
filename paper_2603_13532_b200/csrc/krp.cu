// krp.cu — stage B on DMMA tensor cores: core × implicit Khatri-Rao product.
//
// For atom b (one core block of one summand) and mode n (reference
// src/sketch.cpp:117-131):
//   V_n(a, c) = Σ_J G_b,(n)(a, J) · K_n(J, c),   K_n(J, c) = Π_{j≠n} M_j(col_b[j] + a_j(J), c)
// with J enumerating the other modes lowest-first (the unfolding's column order,
// src/dense_tensor.cpp:145-164) and M_j = (Ω_jᵀ U_j)ᵀ stored as Z_j (s × R_j).
// One CTA per (atom, mode, 64 sketch columns): the M_j slices sit in shared
// memory, each 16-row chunk of K_n is generated there (never in HBM), the
// matching 16 columns of G_(n) are gathered from the core (prefetched into
// registers one chunk ahead), and the product runs on DMMA.8x8x4.  The result
// is stored transposed, Wt_n (s × R_n), so stage C reads both of its operands
// along their non-reduction dimension (gemm_tma.cu MN scheme).
#include <algorithm>
#include <cstdlib>

#include "../../include/tucksum_cuda.h"
#include "kernels.cuh"

namespace ts {
namespace {

constexpr int kThreads = 128;
constexpr int kCT = 64;   // sketch columns per CTA
constexpr int kJC = 16;   // K_n rows (complement indices) per chunk
constexpr int kGS = kJC + 4;   // Gs row stride ([a][J], J contiguous)
constexpr int kKS = kCT + 4;   // Ks row stride ([J][c], c contiguous)

template <int RT>
struct KrpCfg {
    static constexpr int WM = 32;
    static constexpr int WN = RT == 64 ? 32 : 16;
    static constexpr int WARPS_M = RT / WM;
    static constexpr int GPT = RT * kJC / kThreads;  // gathered core values per thread per chunk
};

template <int RT>
__global__ void __launch_bounds__(kThreads) krp_dmma_kernel(KrpArgs args) {
    using Cfg = KrpCfg<RT>;
    constexpr int WM = Cfg::WM, WN = Cfg::WN;
    const Atom& at = args.atoms[blockIdx.x];
    const int n = blockIdx.y;
    // blockIdx.z = column chunk × splits + split: split `sp` takes its share of
    // the complement chunks (split-J, partials summed in split order afterwards).
    const int sp = static_cast<int>(blockIdx.z) % args.splits;
    const int c0 = (static_cast<int>(blockIdx.z) / args.splits) * kCT;
    const int order = args.order, s = args.s;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp % Cfg::WARPS_M, wn = warp / Cfg::WARPS_M;

    int shape[kMaxOrder], col[kMaxOrder];
    int64_t gstride[kMaxOrder];
    int64_t st = 1;
    for (int j = 0; j < order; ++j) {
        shape[j] = at.shape[j];
        col[j] = at.col[j];
        gstride[j] = st;
        st *= shape[j];
    }
    const int rn = shape[n];
    int64_t jtot = 1;
    for (int j = 0; j < order; ++j)
        if (j != n) jtot *= shape[j];
    const int64_t nall = (jtot + kJC - 1) / kJC;
    const int64_t ch_begin = nall * sp / args.splits, ch_end = nall * (sp + 1) / args.splits;
    const int64_t nchunks = ch_end - ch_begin;

    extern __shared__ __align__(16) double sm[];
    int moff[kMaxOrder];
    int msum = 0;
    for (int j = 0; j < order; ++j) {
        moff[j] = msum;
        if (j != n) msum += shape[j] * kCT;
    }
    double* Ms = sm;                          // Σ_{j≠n} r_j × CT ([a][c])
    double* Ks = Ms + msum;                   // kJC × kKS
    double* Gs = Ks + kJC * kKS;              // RT × kGS
    int64_t* Goff = reinterpret_cast<int64_t*>(Gs + RT * kGS);  // 2 × kJC (double-buffered)
    int* Idx = reinterpret_cast<int*>(Goff + 2 * kJC);           // 2 × kJC × kMaxOrder

    for (int j = 0; j < order; ++j) {
        if (j == n) continue;
        const double* Z = args.Z[j];
        for (int idx = tid; idx < shape[j] * kCT; idx += kThreads) {
            const int a = idx / kCT, c = idx % kCT;
            const int cg = c0 + c;
            Ms[moff[j] + idx] = cg < s ? Z[cg + static_cast<int64_t>(col[j] + a) * s] : 0.0;
        }
    }
    const double w = args.weights[at.summand];
    const double* __restrict__ core = args.cores + at.core_off;
    // Unsplit: the weighted result goes straight to Wt_n; split: partial sums
    // (already weighted) go to this split's slab of the workspace.
    double* Wn = args.splits == 1 ? args.W[n] : args.Wpart[n] + static_cast<int64_t>(sp) * args.R[n] * s;

    auto decode = [&](int64_t chunk, int buf) {
        if (tid < kJC) {
            const int64_t J = chunk * kJC + tid;
            int64_t off = -1;
            if (J < jtot) {
                int64_t rem = J;
                off = 0;
                for (int j = 0; j < order; ++j) {
                    if (j == n) continue;
                    const int aj = static_cast<int>(rem % shape[j]);
                    rem /= shape[j];
                    off += aj * gstride[j];
                    Idx[(buf * kJC + tid) * kMaxOrder + j] = aj;
                }
            }
            Goff[buf * kJC + tid] = off;
        }
    };
    // Gathered core element e of this thread for a chunk: threads run along J
    // (contiguous for n != 0) or along a (contiguous for n == 0).
    auto gather = [&](int buf, int a0, double (&gv)[Cfg::GPT]) {
#pragma unroll
        for (int e = 0; e < Cfg::GPT; ++e) {
            const int idx = tid + e * kThreads;
            const int a = n == 0 ? idx % RT : idx / kJC;
            const int jj = n == 0 ? idx / RT : idx % kJC;
            const int64_t off = Goff[buf * kJC + jj];
            gv[e] = (off >= 0 && a0 + a < rn) ? core[off + (a0 + a) * gstride[n]] : 0.0;
        }
    };

    for (int a0 = 0; a0 < rn; a0 += RT) {
        double acc[WM / 8][WN / 8][2];
#pragma unroll
        for (int i = 0; i < WM / 8; ++i)
#pragma unroll
            for (int j = 0; j < WN / 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        double gv[Cfg::GPT];
        __syncthreads();
        decode(ch_begin, 0);
        __syncthreads();
        gather(0, a0, gv);
        for (int64_t ch = 0; ch < nchunks; ++ch) {
            const int buf = static_cast<int>(ch & 1);
            // Stage this chunk: gathered core values → Gs, generated KRP rows → Ks.
#pragma unroll
            for (int e = 0; e < Cfg::GPT; ++e) {
                const int idx = tid + e * kThreads;
                const int a = n == 0 ? idx % RT : idx / kJC;
                const int jj = n == 0 ? idx / RT : idx % kJC;
                Gs[a * kGS + jj] = gv[e];
            }
            for (int idx = tid; idx < kJC * kCT; idx += kThreads) {
                const int jj = idx / kCT, c = idx % kCT;
                double v = 0.0;
                if (Goff[buf * kJC + jj] >= 0) {
                    v = 1.0;
                    for (int j = 0; j < order; ++j) {
                        if (j == n) continue;
                        v *= Ms[moff[j] + Idx[(buf * kJC + jj) * kMaxOrder + j] * kCT + c];
                    }
                }
                Ks[jj * kKS + c] = v;
            }
            if (ch + 1 < nchunks) decode(ch_begin + ch + 1, buf ^ 1);
            __syncthreads();
            if (ch + 1 < nchunks) gather(buf ^ 1, a0, gv);  // prefetch the next chunk during the MMAs
#pragma unroll
            for (int kk = 0; kk < kJC; kk += 4) {
                double af[WM / 8], bf[WN / 8];
#pragma unroll
                for (int i = 0; i < WM / 8; ++i) af[i] = Gs[(wm * WM + i * 8 + g) * kGS + kk + t];
#pragma unroll
                for (int j = 0; j < WN / 8; ++j) bf[j] = Ks[(kk + t) * kKS + wn * WN + j * 8 + g];
#pragma unroll
                for (int i = 0; i < WM / 8; ++i)
#pragma unroll
                    for (int j = 0; j < WN / 8; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
            }
            __syncthreads();
        }
#pragma unroll
        for (int i = 0; i < WM / 8; ++i)
#pragma unroll
            for (int j = 0; j < WN / 8; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int a = a0 + wm * WM + i * 8 + g;
                    const int cg = c0 + wn * WN + j * 8 + 2 * t + h;
                    if (a < rn && cg < s) Wn[cg + static_cast<int64_t>(col[n] + a) * s] = w * acc[i][j][h];
                }
    }
}

// ---------------------------------------------------------------------------
// Order-3 specialisation (all block ranks ≤ 32): per core slice G_s = G[:, :, a2]
//   T0 = G_s · M1   (r0 × s)   →  V0 += M2(a2, :) ⊙ T0,   V2(a2, :) = colsum(M0 ⊙ T0)
//   T1 = G_sᵀ · M0  (r1 × s)   →  V1 += M2(a2, :) ⊙ T1
// i.e. the three mode contractions of src/sketch.cpp:117-130 share the two
// slice GEMMs (4·r³·s flops per atom instead of 6·r³·s) and no Khatri-Rao row
// is ever formed.  One CTA per (atom, 64 sketch columns); warps own 16 columns
// each; core slices stream through a cp.async double buffer.
constexpr int k3Rows = 32;            // padded r0 = r1
constexpr int k3GLD = k3Rows + 4;     // slice row stride (conflict-free both ways)
constexpr int k3MLD = kCT + 4;        // M0 / M1 row stride

__global__ void __launch_bounds__(kThreads) krp3_dmma_kernel(KrpArgs args) {
    const Atom& at = args.atoms[blockIdx.x];
    const int c0 = blockIdx.y * kCT;
    const int s = args.s;
    const int r0 = at.shape[0], r1 = at.shape[1], r2 = at.shape[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int cw = warp * 16;  // this warp's 16 columns within the chunk

    extern __shared__ __align__(16) double sm[];
    double* M0s = sm;                       // 32 × k3MLD
    double* M1s = M0s + k3Rows * k3MLD;     // 32 × k3MLD
    double* Gs = M1s + k3Rows * k3MLD;      // 2 × 32 × k3GLD
    double* M2s = Gs + 2 * k3Rows * k3GLD;  // r2 × kCT
    const double* Z0 = args.Z[0];
    const double* Z1 = args.Z[1];
    const double* Z2 = args.Z[2];
    for (int idx = tid; idx < k3Rows * kCT; idx += kThreads) {
        const int a = idx / kCT, c = idx % kCT, cg = c0 + c;
        M0s[a * k3MLD + c] = (a < r0 && cg < s) ? Z0[cg + static_cast<int64_t>(at.col[0] + a) * s] : 0.0;
        M1s[a * k3MLD + c] = (a < r1 && cg < s) ? Z1[cg + static_cast<int64_t>(at.col[1] + a) * s] : 0.0;
    }
    for (int idx = tid; idx < r2 * kCT; idx += kThreads) {
        const int a = idx / kCT, c = idx % kCT, cg = c0 + c;
        M2s[idx] = cg < s ? Z2[cg + static_cast<int64_t>(at.col[2] + a) * s] : 0.0;
    }
    // Zero the slice buffers once: padded rows / columns stay zero.
    for (int idx = tid; idx < 2 * k3Rows * k3GLD; idx += kThreads) Gs[idx] = 0.0;
    __syncthreads();
    const double* __restrict__ core = args.cores + at.core_off;
    const int slice = r0 * r1;
    auto load_slice = [&](int a2, int buf) {
        double* dst = Gs + buf * k3Rows * k3GLD;
        const double* src = core + static_cast<int64_t>(a2) * slice;
        for (int idx = tid; idx < slice; idx += kThreads) {
            const int i = idx % r0, j = idx / r0;  // G_s(i, j) column-major
            cp_async8(dst + i + j * k3GLD, src + idx, 8);
        }
    };

    double v0[4][2][2], v1[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) v0[i][j][0] = v0[i][j][1] = v1[i][j][0] = v1[i][j][1] = 0.0;
    const double w = args.weights[at.summand];
    double* W2 = args.W[2];

    if (r2 > 0) load_slice(0, 0);
    cp_async_commit();
    for (int a2 = 0; a2 < r2; ++a2) {
        const int buf = a2 & 1;
        if (a2 + 1 < r2) load_slice(a2 + 1, buf ^ 1);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        const double* G = Gs + buf * k3Rows * k3GLD;
        double t0[4][2][2], t1[4][2][2];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) t0[i][j][0] = t0[i][j][1] = t1[i][j][0] = t1[i][j][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < k3Rows; kk += 4) {
            double a0f[4], a1f[4], b1f[2], b0f[2];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                a0f[i] = G[(8 * i + g) + (kk + t) * k3GLD];  // G_s(a0, a1):  m = a0, k = a1
                a1f[i] = G[(kk + t) + (8 * i + g) * k3GLD];  // G_sᵀ(a1, a0): m = a1, k = a0
            }
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                b1f[j] = M1s[(kk + t) * k3MLD + cw + 8 * j + g];
                b0f[j] = M0s[(kk + t) * k3MLD + cw + 8 * j + g];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    dmma884(t0[i][j][0], t0[i][j][1], a0f[i], b1f[j]);
                    dmma884(t1[i][j][0], t1[i][j][1], a1f[i], b0f[j]);
                }
        }
        // Fold the slice into the three mode sketches.
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = cw + 8 * j + 2 * t + h;
                const double m2 = M2s[a2 * kCT + c];
                double part = 0.0;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    v0[i][j][h] = fma(t0[i][j][h], m2, v0[i][j][h]);
                    v1[i][j][h] = fma(t1[i][j][h], m2, v1[i][j][h]);
                    part = fma(M0s[(8 * i + g) * k3MLD + c], t0[i][j][h], part);
                }
                part += __shfl_xor_sync(0xffffffffu, part, 4);
                part += __shfl_xor_sync(0xffffffffu, part, 8);
                part += __shfl_xor_sync(0xffffffffu, part, 16);
                const int cg = c0 + c;
                if (g == 0 && cg < s) W2[cg + static_cast<int64_t>(at.col[2] + a2) * s] = w * part;
            }
        __syncthreads();
    }
    cp_async_wait<0>();
    double* W0 = args.W[0];
    double* W1 = args.W[1];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int a = 8 * i + g;
                const int cg = c0 + cw + 8 * j + 2 * t + h;
                if (cg >= s) continue;
                if (a < r0) W0[cg + static_cast<int64_t>(at.col[0] + a) * s] = w * v0[i][j][h];
                if (a < r1) W1[cg + static_cast<int64_t>(at.col[1] + a) * s] = w * v1[i][j][h];
            }
}

// Order 4, the krp3 idea one level deeper: for each (a2, a3) core slice G_s
// (r0 × r1) two DMMA slice GEMMs t0 = G_s·M1 and t1 = G_sᵀ·M0 serve all four
// modes — V0 += t0·(M2[a2]∘M3[a3]), V1 += t1·(M2[a2]∘M3[a3]) and, with
// x = Σ_a0 M0∘t0, V2[a2] += x∘M3[a3], V3[a3] += x∘M2[a2] (V2 / V3 accumulate in
// shared memory, one column per thread) — 4·r0·r1·s flops per slice instead
// of the generic kernel's 4·(r⁴·s) per atom and mode.  One CTA per (atom, 64
// sketch columns, a3 range); a3 ranges split the slice loop for few atoms
// (partials summed by krp_split_reduce, deterministic).
__global__ void __launch_bounds__(kThreads) krp4_dmma_kernel(KrpArgs args) {
    const Atom& at = args.atoms[blockIdx.x];
    const int c0 = blockIdx.y * kCT;
    const int s = args.s;
    const int r0 = at.shape[0], r1 = at.shape[1], r2 = at.shape[2], r3 = at.shape[3];
    const int sp = blockIdx.z;
    const int per = (r3 + args.splits - 1) / args.splits;
    const int a3b = sp * per, a3e = min(r3, a3b + per);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int cw = warp * 16;

    extern __shared__ __align__(16) double sm[];
    double* M0s = sm;                        // 32 × k3MLD
    double* M1s = M0s + k3Rows * k3MLD;      // 32 × k3MLD
    double* Gs = M1s + k3Rows * k3MLD;       // 2 × 32 × k3GLD
    double* M2s = Gs + 2 * k3Rows * k3GLD;   // r2 × kCT
    double* M3s = M2s + r2 * kCT;            // r3 × kCT
    double* V2s = M3s + r3 * kCT;            // r2 × kCT
    double* V3s = V2s + r2 * kCT;            // r3 × kCT
    for (int idx = tid; idx < k3Rows * kCT; idx += kThreads) {
        const int a = idx / kCT, c = idx % kCT, cg = c0 + c;
        M0s[a * k3MLD + c] = (a < r0 && cg < s) ? args.Z[0][cg + static_cast<int64_t>(at.col[0] + a) * s] : 0.0;
        M1s[a * k3MLD + c] = (a < r1 && cg < s) ? args.Z[1][cg + static_cast<int64_t>(at.col[1] + a) * s] : 0.0;
    }
    for (int idx = tid; idx < r2 * kCT; idx += kThreads) {
        const int a = idx / kCT, c = idx % kCT, cg = c0 + c;
        M2s[idx] = cg < s ? args.Z[2][cg + static_cast<int64_t>(at.col[2] + a) * s] : 0.0;
        V2s[idx] = 0.0;
    }
    for (int idx = tid; idx < r3 * kCT; idx += kThreads) {
        const int a = idx / kCT, c = idx % kCT, cg = c0 + c;
        M3s[idx] = cg < s ? args.Z[3][cg + static_cast<int64_t>(at.col[3] + a) * s] : 0.0;
        V3s[idx] = 0.0;
    }
    for (int idx = tid; idx < 2 * k3Rows * k3GLD; idx += kThreads) Gs[idx] = 0.0;
    __syncthreads();
    const double* __restrict__ core = args.cores + at.core_off;
    const int slice = r0 * r1;
    const int nsl = (a3e - a3b) * r2;  // slices (a2, a3) of this CTA, a2 fastest
    auto load_slice = [&](int li, int buf) {
        const int a2 = li % r2, a3 = a3b + li / r2;
        double* dst = Gs + buf * k3Rows * k3GLD;
        const double* src = core + static_cast<int64_t>(a2 + r2 * a3) * slice;
        for (int idx = tid; idx < slice; idx += kThreads) {
            const int i = idx % r0, j = idx / r0;
            cp_async8(dst + i + j * k3GLD, src + idx, 8);
        }
    };
    double v0[4][2][2], v1[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) v0[i][j][0] = v0[i][j][1] = v1[i][j][0] = v1[i][j][1] = 0.0;

    if (nsl > 0) load_slice(0, 0);
    cp_async_commit();
    for (int li = 0; li < nsl; ++li) {
        const int buf = li & 1;
        const int a2 = li % r2, a3 = a3b + li / r2;
        if (li + 1 < nsl) load_slice(li + 1, buf ^ 1);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        const double* G = Gs + buf * k3Rows * k3GLD;
        double t0[4][2][2], t1[4][2][2];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) t0[i][j][0] = t0[i][j][1] = t1[i][j][0] = t1[i][j][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < k3Rows; kk += 4) {
            double a0f[4], a1f[4], b1f[2], b0f[2];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                a0f[i] = G[(8 * i + g) + (kk + t) * k3GLD];
                a1f[i] = G[(kk + t) + (8 * i + g) * k3GLD];
            }
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                b1f[j] = M1s[(kk + t) * k3MLD + cw + 8 * j + g];
                b0f[j] = M0s[(kk + t) * k3MLD + cw + 8 * j + g];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    dmma884(t0[i][j][0], t0[i][j][1], a0f[i], b1f[j]);
                    dmma884(t1[i][j][0], t1[i][j][1], a1f[i], b0f[j]);
                }
        }
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = cw + 8 * j + 2 * t + h;
                const double m2 = M2s[a2 * kCT + c], m3 = M3s[a3 * kCT + c];
                const double m23 = m2 * m3;
                double part = 0.0;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    v0[i][j][h] = fma(t0[i][j][h], m23, v0[i][j][h]);
                    v1[i][j][h] = fma(t1[i][j][h], m23, v1[i][j][h]);
                    part = fma(M0s[(8 * i + g) * k3MLD + c], t0[i][j][h], part);
                }
                part += __shfl_xor_sync(0xffffffffu, part, 4);
                part += __shfl_xor_sync(0xffffffffu, part, 8);
                part += __shfl_xor_sync(0xffffffffu, part, 16);
                if (g == 0) {  // column c belongs to this lane alone
                    V2s[a2 * kCT + c] = fma(part, m3, V2s[a2 * kCT + c]);
                    V3s[a3 * kCT + c] = fma(part, m2, V3s[a3 * kCT + c]);
                }
            }
        __syncthreads();
    }
    cp_async_wait<0>();
    const double w = args.weights[at.summand];
    double* Wout[4];
#pragma unroll
    for (int n = 0; n < 4; ++n)
        Wout[n] = args.splits == 1 ? args.W[n] : args.Wpart[n] + static_cast<int64_t>(sp) * args.R[n] * s;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int a = 8 * i + g;
                const int cg = c0 + cw + 8 * j + 2 * t + h;
                if (cg >= s) continue;
                if (a < r0) Wout[0][cg + static_cast<int64_t>(at.col[0] + a) * s] = w * v0[i][j][h];
                if (a < r1) Wout[1][cg + static_cast<int64_t>(at.col[1] + a) * s] = w * v1[i][j][h];
            }
    for (int idx = tid; idx < r2 * kCT; idx += kThreads) {
        const int a = idx / kCT, cg = c0 + idx % kCT;
        if (cg < s) Wout[2][cg + static_cast<int64_t>(at.col[2] + a) * s] = w * V2s[idx];
    }
    for (int idx = tid; idx < r3 * kCT; idx += kThreads) {
        const int a = idx / kCT, cg = c0 + idx % kCT;
        if (cg < s) Wout[3][cg + static_cast<int64_t>(at.col[3] + a) * s] = w * V3s[idx];
    }
}

}  // namespace

// Wt_n = Σ_split Wpart[split] in split order (deterministic).
__global__ void krp_split_reduce(KrpArgs args) {
    const int n = blockIdx.y;
    const int64_t total = args.R[n] * args.s;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double v = 0.0;
        for (int sp = 0; sp < args.splits; ++sp) v += args.Wpart[n][sp * total + e];
        args.W[n][e] = v;
    }
}

void launch_krp_contract(const KrpArgs& args_in, int max_shape, CallScratch& sc) {
    KrpArgs args = args_in;
    args.splits = 1;
    if (args.natoms == 0) return;
    static const bool use3 = [] {
        const char* e = std::getenv("TS_KRP_GENERIC");
        return !(e && e[0] == '1');
    }();
    if (use3 && args.order == 3 && max_shape <= k3Rows) {
        const size_t smem =
            sizeof(double) * (2 * k3Rows * k3MLD + 2 * k3Rows * k3GLD + static_cast<size_t>(max_shape) * kCT);
        // Per-device, thread-safe smem attribute (runtime.hpp set_max_smem).
        set_max_smem(krp3_dmma_kernel, 120 * 1024);
        dim3 grid(static_cast<unsigned>(args.natoms), static_cast<unsigned>((args.s + kCT - 1) / kCT));
        krp3_dmma_kernel<<<grid, kThreads, smem, sc.stream()>>>(args);
        TS_LAUNCH_CHECK();
        sc.launches += 1;
        return;
    }
    if (use3 && args.order == 4 && max_shape <= k3Rows) {
        // a3 splits so that few atoms still cover the SMs (about two waves)
        const int cchunks4 = (args.s + kCT - 1) / kCT;
        const int64_t base4 = static_cast<int64_t>(args.natoms) * cchunks4;
        args.splits = static_cast<int>(std::clamp<int64_t>((2 * 148 + base4 - 1) / base4, 1, std::max(1, max_shape)));
        if (args.splits > 1)
            for (int n = 0; n < 4; ++n)
                args.Wpart[n] = sc.alloc_n<double>(static_cast<size_t>(args.splits * args.R[n] * args.s));
        const size_t smem = sizeof(double) * (2 * k3Rows * k3MLD + 2 * k3Rows * k3GLD + 4 * static_cast<size_t>(max_shape) * kCT);
        set_max_smem(krp4_dmma_kernel, 160 * 1024);
        dim3 grid(static_cast<unsigned>(args.natoms), static_cast<unsigned>(cchunks4), static_cast<unsigned>(args.splits));
        krp4_dmma_kernel<<<grid, kThreads, smem, sc.stream()>>>(args);
        TS_LAUNCH_CHECK();
        sc.launches += 1;
        if (args.splits > 1) {
            krp_split_reduce<<<dim3(64, 4), 256, 0, sc.stream()>>>(args);
            TS_LAUNCH_CHECK();
            sc.launches += 1;
        }
        return;
    }
    const int RT = max_shape <= 32 ? 32 : 64;
    const size_t smem = sizeof(double) * (static_cast<size_t>(max_shape) * args.order * kCT + kJC * kKS + RT * kGS) +
                        sizeof(int64_t) * 2 * kJC + sizeof(int) * 2 * kJC * kMaxOrder;
    // Few (atom, mode, column-chunk) CTAs each walking a long complement (order
    // ≥ 4: Π_{j≠n} r_j KRP rows) leave most of the 148 SMs idle; split the
    // complement so the grid covers about two waves.
    const int cchunks = (args.s + kCT - 1) / kCT;
    const int64_t base = static_cast<int64_t>(args.natoms) * args.order * cchunks;
    std::int64_t most = 1;
    for (int j = 0; j < args.order; ++j) most *= max_shape;
    most /= std::max(1, max_shape);
    const int64_t nall = (most + kJC - 1) / kJC;
    args.splits = static_cast<int>(std::clamp<int64_t>((2 * 148 + base - 1) / base, 1, std::max<int64_t>(1, nall / 8)));
    if (args.splits > 1) {
        for (int n = 0; n < args.order; ++n)
            args.Wpart[n] = sc.alloc_n<double>(static_cast<size_t>(args.splits * args.R[n] * args.s));
    }
    dim3 grid(static_cast<unsigned>(args.natoms), static_cast<unsigned>(args.order),
              static_cast<unsigned>(cchunks * args.splits));
    // Thread-safe one-time setup (the attribute call must not run inside a CUDA
    // graph capture of a later call).
    set_max_smem(krp_dmma_kernel<32>, 200 * 1024); set_max_smem(krp_dmma_kernel<64>, 200 * 1024);
    if (smem > 200 * 1024) throw Error(TS_UNSUPPORTED, "stage B: block ranks too large for shared memory");
    if (RT == 32) krp_dmma_kernel<32><<<grid, kThreads, smem, sc.stream()>>>(args);
    else krp_dmma_kernel<64><<<grid, kThreads, smem, sc.stream()>>>(args);
    TS_LAUNCH_CHECK();
    sc.launches += 1;
    if (args.splits > 1) {
        krp_split_reduce<<<dim3(64, static_cast<unsigned>(args.order)), 256, 0, sc.stream()>>>(args);
        TS_LAUNCH_CHECK();
        sc.launches += 1;
    }
}

}  // namespace ts
