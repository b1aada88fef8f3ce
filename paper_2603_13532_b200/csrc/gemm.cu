// gemm.cu — grouped/batched/split-K fp64 DMMA GEMM for sm_100a (see gemm.cuh).
//
// CTA tile BM×BN, K-step BK, multi-stage cp.async pipeline into padded shared
// memory; each warp owns a WM×WN sub-tile computed with DMMA.8x8x4.  Shared-
// memory rows are padded to a stride ≡ 4 (mod 16) doubles, which makes every
// fragment load (8 rows × 4 k, or 4 k × 8 cols) hit 16 distinct 8-byte bank
// pairs per half-warp, whichever operand dimension is contiguous.
#include <algorithm>
#include <cstring>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "gemm.cuh"

namespace ts {
namespace {

// Copies a ROWS×CONT tile: element (r, c) = g[(row0 + r) * ld + col0 + c]
// → s[r * SS + c], zero-filling outside [0, row_lim) × [0, col_lim).
template <int ROWS, int CONT, int SS, int NTHREADS, int VEC>
__device__ __forceinline__ void load_tile(double* s, const double* __restrict__ g, int64_t ld, int row0, int col0,
                                          int row_lim, int col_lim) {
    constexpr int CV = CONT / VEC;
    constexpr int TOTAL = ROWS * CV;
#pragma unroll 4
    for (int idx = threadIdx.x; idx < TOTAL; idx += NTHREADS) {
        const int r = idx / CV, c = (idx % CV) * VEC;
        const int gr = row0 + r, gc = col0 + c;
        double* dst = s + r * SS + c;
        if constexpr (VEC == 2) {
            const int nvalid = (gr < row_lim) ? max(0, min(2, col_lim - gc)) : 0;
            const double* src = nvalid ? g + static_cast<int64_t>(gr) * ld + gc : g;
            cp_async16(dst, src, nvalid * 8);
        } else {
            const bool ok = gr < row_lim && gc < col_lim;
            cp_async8(dst, ok ? g + static_cast<int64_t>(gr) * ld + gc : g, ok ? 8 : 0);
        }
    }
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool AK, bool BKM>
struct GemmCfg {
    static constexpr int kThreads = (BM / WM) * (BN / WN) * 32;
    static constexpr int kARows = AK ? BM : BK, kACont = AK ? BK : BM;
    static constexpr int kBRows = BKM ? BN : BK, kBCont = BKM ? BK : BN;
    static constexpr int kASS = kACont + 4, kBSS = kBCont + 4;
    static constexpr int kAStage = kARows * kASS, kBStage = kBRows * kBSS;
    static constexpr size_t kSmemBytes = sizeof(double) * STAGES * (kAStage + kBStage);
};

// Launches of up to kPackDescs groups carry their descriptors as a
// __grid_constant__ kernel parameter instead of a scratch upload (inside a CUDA
// graph every upload is a memcpy node serialised in front of its kernel).
constexpr int kPackDescs = 16;
struct GemmPack {
    GemmDesc d[kPackDescs];
    int red[kPackDescs];
};

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool AK, bool BKM, int VEC>
__device__ __forceinline__ void gemm_body(const GemmDesc* __restrict__ descs, int ngroups) {
    using Cfg = GemmCfg<BM, BN, BK, WM, WN, STAGES, AK, BKM>;
    constexpr int NT = Cfg::kThreads;
    constexpr int ASS = Cfg::kASS, BSS = Cfg::kBSS;
    extern __shared__ __align__(16) double smem[];
    double* sA = smem;
    double* sB = smem + STAGES * Cfg::kAStage;

    // Group lookup: last group whose unit_begin <= blockIdx.x.
    const int64_t unit = blockIdx.x;
    int lo = 0, hi = ngroups - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (descs[mid].unit_begin <= unit) lo = mid;
        else hi = mid - 1;
    }
    const GemmDesc& d = descs[lo];
    const int M = d.M, N = d.N, K = d.K;
    const int tiles_m = d.tiles_m, tiles_n = d.tiles_n, splits = d.splits;
    int64_t local = unit - d.unit_begin;
    const int tm = static_cast<int>(local % tiles_m);
    local /= tiles_m;
    const int tn = static_cast<int>(local % tiles_n);
    local /= tiles_n;
    const int sp = static_cast<int>(local % splits);
    const int b = static_cast<int>(local / splits);
    const double* __restrict__ A = d.A + b * d.sA;
    const double* __restrict__ B = d.B + b * d.sB;
    const int64_t lda = d.lda, ldb = d.ldb;
    const int m0 = tm * BM, n0 = tn * BN;
    const int kbeg = sp * d.k_per_split;
    const int kend = min(K, kbeg + d.k_per_split);
    const int nk = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp % (BM / WM), wn = warp / (BM / WM);

    double acc[WM / 8][WN / 8][2];
#pragma unroll
    for (int i = 0; i < WM / 8; ++i)
#pragma unroll
        for (int j = 0; j < WN / 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    auto load_stage = [&](int st, int k0) {
        if constexpr (AK) load_tile<BM, BK, ASS, NT, VEC>(sA + st * Cfg::kAStage, A, lda, m0, k0, M, kend);
        else load_tile<BK, BM, ASS, NT, VEC>(sA + st * Cfg::kAStage, A, lda, k0, m0, kend, M);
        if constexpr (BKM) load_tile<BN, BK, BSS, NT, VEC>(sB + st * Cfg::kBStage, B, ldb, n0, k0, N, kend);
        else load_tile<BK, BN, BSS, NT, VEC>(sB + st * Cfg::kBStage, B, ldb, k0, n0, kend, N);
    };

#pragma unroll
    for (int st = 0; st < STAGES - 1; ++st) {
        if (st < nk) load_stage(st, kbeg + st * BK);
        cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        const int nxt = kt + STAGES - 1;
        if (nxt < nk) load_stage(nxt % STAGES, kbeg + nxt * BK);
        cp_async_commit();
        const double* a_s = sA + (kt % STAGES) * Cfg::kAStage;
        const double* b_s = sB + (kt % STAGES) * Cfg::kBStage;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[WM / 8], bf[WN / 8];
#pragma unroll
            for (int i = 0; i < WM / 8; ++i) {
                const int m = wm * WM + i * 8 + g, k = kk + t;
                af[i] = AK ? a_s[m * ASS + k] : a_s[k * ASS + m];
            }
#pragma unroll
            for (int j = 0; j < WN / 8; ++j) {
                const int n = wn * WN + j * 8 + g, k = kk + t;
                bf[j] = BKM ? b_s[n * BSS + k] : b_s[k * BSS + n];
            }
#pragma unroll
            for (int i = 0; i < WM / 8; ++i)
#pragma unroll
                for (int j = 0; j < WN / 8; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
    }
    cp_async_wait<0>();

    // Epilogue: thread owns C[m][n], C[m][n+1] of each 8×8 sub-tile.
    if (splits == 1) {
        double* __restrict__ C = d.C + b * d.sC;
        const int64_t ldc = d.ldc;
        const double alpha = d.alpha, beta = d.beta;
#pragma unroll
        for (int i = 0; i < WM / 8; ++i)
#pragma unroll
            for (int j = 0; j < WN / 8; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int m = m0 + wm * WM + i * 8 + g, n = n0 + wn * WN + j * 8 + 2 * t + h;
                    if (m < M && n < N) {
                        double* c = C + m + static_cast<int64_t>(n) * ldc;
                        *c = beta == 0.0 ? alpha * acc[i][j][h] : alpha * acc[i][j][h] + beta * *c;
                    }
                }
    } else {
        double* __restrict__ W = d.ws + (static_cast<int64_t>(b) * splits + sp) * static_cast<int64_t>(M) * N;
#pragma unroll
        for (int i = 0; i < WM / 8; ++i)
#pragma unroll
            for (int j = 0; j < WN / 8; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int m = m0 + wm * WM + i * 8 + g, n = n0 + wn * WN + j * 8 + 2 * t + h;
                    if (m < M && n < N) W[m + static_cast<int64_t>(n) * M] = acc[i][j][h];
                }
    }
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool AK, bool BKM, int VEC>
__global__ void __launch_bounds__(GemmCfg<BM, BN, BK, WM, WN, STAGES, AK, BKM>::kThreads)
    gemm_kernel(const GemmDesc* __restrict__ descs, int ngroups) {
    gemm_body<BM, BN, BK, WM, WN, STAGES, AK, BKM, VEC>(descs, ngroups);
}
template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool AK, bool BKM, int VEC>
__global__ void __launch_bounds__(GemmCfg<BM, BN, BK, WM, WN, STAGES, AK, BKM>::kThreads)
    gemm_kernel_pk(const __grid_constant__ GemmPack pk, int ngroups) {
    gemm_body<BM, BN, BK, WM, WN, STAGES, AK, BKM, VEC>(pk.d, ngroups);
}

// Sums the split-K partials of group red[blockIdx.y] in split order.
__device__ __forceinline__ void splitk_reduce_body(const GemmDesc* __restrict__ descs, const int* __restrict__ red);
__global__ void splitk_reduce(const GemmDesc* __restrict__ descs, const int* __restrict__ red) {
    splitk_reduce_body(descs, red);
}
__global__ void splitk_reduce_pk(const __grid_constant__ GemmPack pk) { splitk_reduce_body(pk.d, pk.red); }
__device__ __forceinline__ void splitk_reduce_body(const GemmDesc* __restrict__ descs, const int* __restrict__ red) {
    const GemmDesc& d = descs[red[blockIdx.y]];
    const int64_t mn = static_cast<int64_t>(d.M) * d.N;
    const int64_t total = mn * d.batch;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t b = e / mn, r = e % mn;
        const int m = static_cast<int>(r % d.M), n = static_cast<int>(r / d.M);
        const double* w = d.ws + b * d.splits * mn + r;
        double s = 0.0;
        // Split order is fixed (deterministic); loads are batched 8 at a time so
        // their L2 latencies overlap instead of serialising on the running sum.
        const double* src = w;
        int sp = 0;
        for (; sp + 8 <= d.splits; sp += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = src[(sp + u) * mn];
#pragma unroll
            for (int u = 0; u < 8; ++u) s += v[u];
        }
        for (; sp < d.splits; ++sp) s += src[sp * mn];
        double* c = d.C + b * d.sC + m + static_cast<int64_t>(n) * d.ldc;
        *c = d.beta == 0.0 ? d.alpha * s : d.alpha * s + d.beta * *c;
    }
}

// ---------------------------------------------------------------- tile configurations
// Runtime-selectable CTA tiles (TS_GEMM_CFG_{TN,NN,NT} override the defaults).
struct TileCfg {
    int bm, bn, bk;
};
constexpr TileCfg kCfgs[] = {
    {64, 64, 16},   // 0: 4 warps of 32×32, 4 stages
    {128, 64, 16},  // 1: 8 warps of 32×32, 3 stages
    {64, 128, 16},  // 2: 8 warps of 32×32, 3 stages
    {64, 64, 32},   // 3: 4 warps of 32×32, 3 stages
    {128, 64, 16},  // 4: 4 warps of 64×32, 3 stages
    {64, 128, 16},  // 5: 4 warps of 32×64, 3 stages
};
constexpr int kNumCfgs = sizeof(kCfgs) / sizeof(kCfgs[0]);

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool AK, bool BKM, int VEC>
void launch_kernel(const GemmDesc* d_descs, const GemmPack* pk, int ngroups, int64_t units, cudaStream_t stream) {
    using Cfg = GemmCfg<BM, BN, BK, WM, WN, STAGES, AK, BKM>;
    if (pk) {
        auto kern = gemm_kernel_pk<BM, BN, BK, WM, WN, STAGES, AK, BKM, VEC>;
        set_max_smem(kern, static_cast<int>(Cfg::kSmemBytes));
        kern<<<static_cast<unsigned>(units), Cfg::kThreads, Cfg::kSmemBytes, stream>>>(*pk, ngroups);
    } else {
        auto kern = gemm_kernel<BM, BN, BK, WM, WN, STAGES, AK, BKM, VEC>;
        set_max_smem(kern, static_cast<int>(Cfg::kSmemBytes));
        kern<<<static_cast<unsigned>(units), Cfg::kThreads, Cfg::kSmemBytes, stream>>>(d_descs, ngroups);
    }
    TS_LAUNCH_CHECK();
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool AK, bool BKM>
int occupancy_of() {
    using Cfg = GemmCfg<BM, BN, BK, WM, WN, STAGES, AK, BKM>;
    auto kern2 = gemm_kernel<BM, BN, BK, WM, WN, STAGES, AK, BKM, 2>;
    set_max_smem(kern2, static_cast<int>(Cfg::kSmemBytes));  // per device
    static const int occ = [&] {  // thread-safe one-time query (same on every B200)
        int o = 0;
        TS_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern2, Cfg::kThreads, Cfg::kSmemBytes));
        return std::max(o, 1);
    }();
    return occ;
}

template <bool AK, bool BKM>
struct Dispatch {
    static int occupancy(int cfg) {
        switch (cfg) {
            case 1: return occupancy_of<128, 64, 16, 32, 32, 3, AK, BKM>();
            case 2: return occupancy_of<64, 128, 16, 32, 32, 3, AK, BKM>();
            case 3: return occupancy_of<64, 64, 32, 32, 32, 3, AK, BKM>();
            case 4: return occupancy_of<128, 64, 16, 64, 32, 3, AK, BKM>();
            case 5: return occupancy_of<64, 128, 16, 32, 64, 3, AK, BKM>();
            default: return occupancy_of<64, 64, 16, 32, 32, 4, AK, BKM>();
        }
    }
    template <int VEC>
    static void launch(int cfg, const GemmDesc* d, const GemmPack* pk, int ng, int64_t units, cudaStream_t st) {
        switch (cfg) {
            case 1: return launch_kernel<128, 64, 16, 32, 32, 3, AK, BKM, VEC>(d, pk, ng, units, st);
            case 2: return launch_kernel<64, 128, 16, 32, 32, 3, AK, BKM, VEC>(d, pk, ng, units, st);
            case 3: return launch_kernel<64, 64, 32, 32, 32, 3, AK, BKM, VEC>(d, pk, ng, units, st);
            case 4: return launch_kernel<128, 64, 16, 64, 32, 3, AK, BKM, VEC>(d, pk, ng, units, st);
            case 5: return launch_kernel<64, 128, 16, 32, 64, 3, AK, BKM, VEC>(d, pk, ng, units, st);
            default: return launch_kernel<64, 64, 16, 32, 32, 4, AK, BKM, VEC>(d, pk, ng, units, st);
        }
    }
};

int config_for(Layout layout) {
    static int cfg[3] = {-2, -2, -2};
    const int li = static_cast<int>(layout);
    if (cfg[li] == -2) {
        const char* names[3] = {"TS_GEMM_CFG_TN", "TS_GEMM_CFG_NN", "TS_GEMM_CFG_NT"};
        const int defaults[3] = {0, 0, 0};
        const char* e = std::getenv(names[li]);
        int v = e ? std::atoi(e) : defaults[li];
        if (v < 0 || v >= kNumCfgs) v = defaults[li];
        cfg[li] = v;
    }
    return cfg[li];
}

int occupancy(Layout layout, int cfg) {
    switch (layout) {
        case Layout::TN: return Dispatch<true, true>::occupancy(cfg);
        case Layout::NN: return Dispatch<false, true>::occupancy(cfg);
        default: return Dispatch<false, false>::occupancy(cfg);
    }
}

// Splits K so the launch fills whole waves of CTA slots: maximise
// units / (waves × slots), preferring fewer splits within 3 %.
int choose_splits(int64_t tiles, int64_t slots, int K, int bk) {
    const int maxs = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(64, K / (4 * bk))));
    double best = -1.0;
    int best_s = 1;
    std::vector<double> eff(static_cast<size_t>(maxs) + 1, 0.0);
    for (int s = 1; s <= maxs; ++s) {
        const int64_t u = tiles * s;
        const int64_t waves = (u + slots - 1) / slots;
        // Small problems: more splits also shorten each CTA's serial K loop.
        eff[static_cast<size_t>(s)] = static_cast<double>(u) / static_cast<double>(waves * slots);
        best = std::max(best, eff[static_cast<size_t>(s)]);
    }
    for (int s = 1; s <= maxs; ++s)
        if (eff[static_cast<size_t>(s)] >= best - 0.03) {
            best_s = s;
            break;
        }
    return best_s;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

int launch_grouped_gemm(Layout layout, const std::vector<GemmProblem>& probs, CallScratch& sc, int num_sms) {
    {
        int launched = 0;
        if (probs.size() <= 16 && launch_tma_gemm(layout, probs, sc, num_sms, &launched)) return launched;
    }
    const int cfg = config_for(layout);
    const TileCfg tc = kCfgs[cfg];
    const int64_t slots = static_cast<int64_t>(num_sms) * occupancy(layout, cfg);
    std::vector<GemmDesc> descs;
    descs.reserve(probs.size());
    int64_t units = 0;
    bool vec2 = true;
    size_t ws_elems = 0;
    std::vector<int> red;
    int64_t total_tiles = 0;
    for (const GemmProblem& p : probs)
        if (p.M > 0 && p.N > 0 && p.batch > 0)
            total_tiles += static_cast<int64_t>((p.M + tc.bm - 1) / tc.bm) * ((p.N + tc.bn - 1) / tc.bn) * p.batch;
    for (const GemmProblem& p : probs) {
        if (p.M <= 0 || p.N <= 0 || p.batch <= 0) continue;
        GemmDesc d{};
        d.A = p.A;
        d.B = p.B;
        d.C = p.C;
        d.lda = p.lda;
        d.ldb = p.ldb;
        d.ldc = p.ldc;
        d.sA = p.sA;
        d.sB = p.sB;
        d.sC = p.sC;
        d.M = p.M;
        d.N = p.N;
        d.K = p.K;
        d.batch = p.batch;
        d.alpha = p.alpha;
        d.beta = p.beta;
        d.tiles_m = (p.M + tc.bm - 1) / tc.bm;
        d.tiles_n = (p.N + tc.bn - 1) / tc.bn;
        const int64_t tiles = static_cast<int64_t>(d.tiles_m) * d.tiles_n * p.batch;
        // Split decision on the whole launch (groups share the waves); every group
        // gets the same split factor, applied only when its K is long enough.
        int splits = p.K > 4 * tc.bk ? choose_splits(total_tiles, slots, p.K, tc.bk) : 1;
        int kps = (p.K + splits - 1) / splits;
        kps = ((kps + tc.bk - 1) / tc.bk) * tc.bk;
        if (kps <= 0) kps = tc.bk;
        splits = std::max(1, (p.K + kps - 1) / kps);
        d.splits = splits;
        d.k_per_split = kps;
        d.unit_begin = units;
        units += tiles * splits;
        if (splits > 1) {
            red.push_back(static_cast<int>(descs.size()));
            ws_elems += static_cast<size_t>(p.M) * p.N * p.batch * splits;
        }
        vec2 = vec2 && aligned16(p.A) && aligned16(p.B) && (p.lda % 2 == 0) && (p.ldb % 2 == 0) &&
               (p.sA % 2 == 0) && (p.sB % 2 == 0);
        descs.push_back(d);
    }
    if (descs.empty()) return 0;
    if (ws_elems > 0) {
        double* ws = sc.alloc_n<double>(ws_elems);
        size_t off = 0;
        for (int gi : red) {
            GemmDesc& d = descs[static_cast<size_t>(gi)];
            d.ws = ws + off;
            off += static_cast<size_t>(d.M) * d.N * d.batch * d.splits;
        }
    }
    const int ng = static_cast<int>(descs.size());
    const bool packed = ng <= kPackDescs;
    GemmPack pack;
    const GemmPack* pk = nullptr;
    const GemmDesc* d_descs = nullptr;
    if (packed) {
        std::memset(&pack, 0, sizeof(pack));
        std::memcpy(pack.d, descs.data(), descs.size() * sizeof(GemmDesc));
        for (size_t i = 0; i < red.size(); ++i) pack.red[i] = red[i];
        pk = &pack;
    } else {
        d_descs = static_cast<const GemmDesc*>(sc.upload(descs.data(), descs.size() * sizeof(GemmDesc)));
    }
    cudaStream_t st = sc.stream();
    switch (layout) {
        case Layout::TN:
            vec2 ? Dispatch<true, true>::launch<2>(cfg, d_descs, pk, ng, units, st)
                 : Dispatch<true, true>::launch<1>(cfg, d_descs, pk, ng, units, st);
            break;
        case Layout::NN:
            vec2 ? Dispatch<false, true>::launch<2>(cfg, d_descs, pk, ng, units, st)
                 : Dispatch<false, true>::launch<1>(cfg, d_descs, pk, ng, units, st);
            break;
        case Layout::NT:
            vec2 ? Dispatch<false, false>::launch<2>(cfg, d_descs, pk, ng, units, st)
                 : Dispatch<false, false>::launch<1>(cfg, d_descs, pk, ng, units, st);
            break;
    }
    int launched = 1;
    if (!red.empty()) {
        int64_t maxel = 0;
        for (int gi : red) {
            const GemmDesc& d = descs[static_cast<size_t>(gi)];
            maxel = std::max<int64_t>(maxel, static_cast<int64_t>(d.M) * d.N * d.batch);
        }
        const int threads = 256;
        const int64_t blocks = std::min<int64_t>((maxel + threads - 1) / threads, 4LL * num_sms);
        const dim3 rgrid(static_cast<unsigned>(std::max<int64_t>(blocks, 1)), static_cast<unsigned>(red.size()));
        if (packed) {
            splitk_reduce_pk<<<rgrid, threads, 0, st>>>(pack);
        } else {
            const int* d_red = static_cast<const int*>(sc.upload(red.data(), red.size() * sizeof(int)));
            splitk_reduce<<<rgrid, threads, 0, st>>>(d_descs, d_red);
        }
        TS_LAUNCH_CHECK();
        ++launched;
    }
    sc.launches += launched;
    return launched;
}

}  // namespace ts
