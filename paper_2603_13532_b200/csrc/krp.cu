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
    const int c0 = blockIdx.z * kCT;
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
    const int64_t nchunks = (jtot + kJC - 1) / kJC;

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
    double* Wn = args.W[n];

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
        decode(0, 0);
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
            if (ch + 1 < nchunks) decode(ch + 1, buf ^ 1);
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

}  // namespace

void launch_krp_contract(const KrpArgs& args, int max_shape, CallScratch& sc) {
    if (args.natoms == 0) return;
    const int RT = max_shape <= 32 ? 32 : 64;
    const size_t smem = sizeof(double) * (static_cast<size_t>(max_shape) * args.order * kCT + kJC * kKS + RT * kGS) +
                        sizeof(int64_t) * 2 * kJC + sizeof(int) * 2 * kJC * kMaxOrder;
    dim3 grid(static_cast<unsigned>(args.natoms), static_cast<unsigned>(args.order),
              static_cast<unsigned>((args.s + kCT - 1) / kCT));
    auto go = [&](auto kern) {
        TS_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        kern<<<grid, kThreads, smem, sc.stream()>>>(args);
        TS_LAUNCH_CHECK();
    };
    if (RT == 32) go(krp_dmma_kernel<32>);
    else go(krp_dmma_kernel<64>);
    sc.launches += 1;
}

}  // namespace ts
