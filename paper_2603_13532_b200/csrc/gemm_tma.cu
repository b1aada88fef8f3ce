// gemm_tma.cu — warp-specialised fp64 GEMM: TMA → 128B-swizzled shared memory →
// DMMA.8x8x4, synchronised with mbarriers (no CTA-wide barrier in the main loop).
//
// Used for the big stacked contractions of the KRP sum (stages A, C, E, F2, the
// CholeskyQR Grams and Q updates, the ST-HOSVD Grams and the output GEMM) when
// the operands satisfy TMA's alignment rules; gemm.cu's cp.async kernel covers
// everything else (odd leading dimensions, the many-group per-atom TTMs).
//
// One producer warp (one elected lane) streams 64×16 A and B tiles with
// cp.async.bulk.tensor into a STAGES-deep ring; four consumer warps (2×2, 32×32
// each) wait on the stage's "full" mbarrier, run 64 DMMAs, and release the stage
// through its "empty" mbarrier.
//
// Two fragment schemes, both bank-conflict free on the 128B swizzle (16-byte
// chunk c of line r stored at chunk c ^ (r & 7)) with 16-byte LDS:
//   KK (TN layout: A and B both k-contiguous; lines = m or n, 16 k per line):
//      thread (g,t) reads chunks 2t, 2t+1 of line g → k = 4t..4t+3, so DMMA q
//      of the 16-k stage uses k = 4t + q for both operands.
//   MN (NN with B stored n-contiguous, NT: lines = k, 16 m (or n) per line):
//      thread (g,t) reads chunk ch(g) of line kk + t → the m pair
//      (2ch(g), 2ch(g)+1): one load feeds two DMMAs (even / odd rows) with the
//      natural k mapping; ch(g) = ((g&1)<<2) | (g>>1) keeps each 8-lane phase on
//      8 distinct chunks.  The epilogue undoes the row / column permutation.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "gemm.cuh"
#include "tma.cuh"

namespace ts {
namespace {

constexpr int kBM = 64, kBN = 64, kBK = 16;
constexpr int kStages = 6;
constexpr int kConsumerWarps = 4;
constexpr int kThreads = (kConsumerWarps + 1) * 32;
constexpr int kTileBytes = kBM * kBK * 8;  // 8 KB per operand per stage
constexpr size_t kSmemBytes = 1024 + static_cast<size_t>(kStages) * 2 * kTileBytes + 2 * kStages * 8;

struct alignas(64) TmaGroup {
    CUtensorMap ta;  // A operand map
    CUtensorMap tb;  // B operand map
    double* C;
    double* ws;
    int64_t ldc;
    int M, N, K;
    int splits, tiles_m, tiles_n, k_per_split;
    double alpha, beta;
    int64_t unit_begin;
};

__device__ __forceinline__ void lds128(unsigned addr, double& x, double& y) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(x), "=d"(y) : "r"(addr));
}
__device__ __forceinline__ int chunk_of(int g) { return ((g & 1) << 2) | (g >> 1); }

// Launches of up to kPackGroups groups carry their descriptors (tensor maps
// included) as a __grid_constant__ kernel parameter instead of a scratch upload:
// inside a CUDA graph every upload is a memcpy node serialised in front of its
// kernel (a call has ~30 of them).
constexpr int kPackGroups = 8;
struct TmaPack {
    TmaGroup g[kPackGroups];
    int red[kPackGroups];
};

template <bool MN>
__device__ __forceinline__ void gemm_tma_body(const TmaGroup* __restrict__ groups, int ngroups) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* tilesA = smem;
    unsigned char* tilesB = smem + kStages * kTileBytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * kStages * kTileBytes);
    uint64_t* empty = full + kStages;

    const int64_t unit = blockIdx.x;
    int lo = 0, hi = ngroups - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (groups[mid].unit_begin <= unit) lo = mid;
        else hi = mid - 1;
    }
    const TmaGroup& G = groups[lo];
    const int M = G.M, N = G.N, K = G.K;
    int64_t local = unit - G.unit_begin;
    const int tm = static_cast<int>(local % G.tiles_m);
    local /= G.tiles_m;
    const int tn = static_cast<int>(local % G.tiles_n);
    const int sp = static_cast<int>(local / G.tiles_n);
    const int m0 = tm * kBM, n0 = tn * kBN;
    const int kbeg = sp * G.k_per_split;
    const int kend = min(K, kbeg + G.k_per_split);
    const int nk = kend > kbeg ? (kend - kbeg + kBK - 1) / kBK : 0;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    }
    __syncthreads();

    if (warp == kConsumerWarps) {
        // ---------------- producer
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&G.ta)));
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&G.tb)));
            for (int kt = 0; kt < nk; ++kt) {
                const int s = kt % kStages;
                const int use = kt / kStages;
                if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);
                mbar_expect_tx(&full[s], 2 * kTileBytes);
                const int k0 = kbeg + kt * kBK;
                unsigned char* a = tilesA + s * kTileBytes;
                unsigned char* b = tilesB + s * kTileBytes;
                if constexpr (!MN) {
                    tma_load_2d(a, &G.ta, k0, m0, &full[s]);
                    tma_load_2d(b, &G.tb, k0, n0, &full[s]);
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        tma_load_2d(a + q * 2048, &G.ta, m0 + 16 * q, k0, &full[s]);
                        tma_load_2d(b + q * 2048, &G.tb, n0 + 16 * q, k0, &full[s]);
                    }
                }
            }
        }
        return;
    }

    // ---------------- consumers: 2×2 warps of 32×32
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp & 1, wn = warp >> 1;
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const unsigned baseA = smem_u32(tilesA), baseB = smem_u32(tilesB);

    for (int kt = 0; kt < nk; ++kt) {
        const int s = kt % kStages;
        mbar_wait(&full[s], (kt / kStages) & 1);
        const unsigned sa = baseA + s * kTileBytes, sb = baseB + s * kTileBytes;
        if constexpr (!MN) {
            // KK: lines are m (A) / n (B); 4 DMMAs per (i, j) over the 16-k stage.
            double a[4][4], b[4][4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int r = wm * 32 + i * 8 + g;  // r & 7 == g
                lds128(sa + r * 128 + (((2 * t) ^ g) << 4), a[i][0], a[i][1]);
                lds128(sa + r * 128 + (((2 * t + 1) ^ g) << 4), a[i][2], a[i][3]);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int r = wn * 32 + j * 8 + g;
                lds128(sb + r * 128 + (((2 * t) ^ g) << 4), b[j][0], b[j][1]);
                lds128(sb + r * 128 + (((2 * t + 1) ^ g) << 4), b[j][2], b[j][3]);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i][q], b[j][q]);
        } else {
            // MN: lines are k; sub-tiles of 16 m (n) at 2 KB strides.
            const int cg = chunk_of(g);
#pragma unroll
            for (int kk = 0; kk < kBK; kk += 4) {
                const int line = kk + t;
                const unsigned off = line * 128 + ((cg ^ (line & 7)) << 4);
                double a[4], b[4];  // [2*sub + parity]
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    lds128(sa + (wm * 2 + u) * 2048 + off, a[2 * u], a[2 * u + 1]);
                    lds128(sb + (wn * 2 + u) * 2048 + off, b[2 * u], b[2 * u + 1]);
                }
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }

    // ---------------- epilogue
    const bool direct = G.splits == 1;
    double* __restrict__ C = G.C;
    const int64_t ldc = G.ldc;
    double* __restrict__ W = direct ? nullptr : G.ws + static_cast<int64_t>(sp) * M * N;
    const double alpha = G.alpha, beta = G.beta;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                int m, n;
                if constexpr (!MN) {
                    m = m0 + wm * 32 + i * 8 + g;
                    n = n0 + wn * 32 + j * 8 + 2 * t + h;
                } else {
                    m = m0 + wm * 32 + (i >> 1) * 16 + 2 * chunk_of(g) + (i & 1);
                    n = n0 + wn * 32 + (j >> 1) * 16 + 2 * chunk_of(2 * t + h) + (j & 1);
                }
                if (m < M && n < N) {
                    if (direct) {
                        double* c = C + m + static_cast<int64_t>(n) * ldc;
                        *c = beta == 0.0 ? alpha * acc[i][j][h] : alpha * acc[i][j][h] + beta * *c;
                    } else {
                        W[m + static_cast<int64_t>(n) * M] = acc[i][j][h];
                    }
                }
            }
}

template <bool MN>
__global__ void __launch_bounds__(kThreads, 1) gemm_tma_kernel(const TmaGroup* __restrict__ groups, int ngroups) {
    gemm_tma_body<MN>(groups, ngroups);
}
template <bool MN>
__global__ void __launch_bounds__(kThreads, 1) gemm_tma_kernel_pk(const __grid_constant__ TmaPack pk, int ngroups) {
    gemm_tma_body<MN>(pk.g, ngroups);
}

__device__ __forceinline__ void tma_splitk_reduce_body(const TmaGroup* __restrict__ groups, const int* __restrict__ red);
__global__ void tma_splitk_reduce(const TmaGroup* __restrict__ groups, const int* __restrict__ red) {
    tma_splitk_reduce_body(groups, red);
}
__global__ void tma_splitk_reduce_pk(const __grid_constant__ TmaPack pk) { tma_splitk_reduce_body(pk.g, pk.red); }

__device__ __forceinline__ void tma_splitk_reduce_body(const TmaGroup* __restrict__ groups, const int* __restrict__ red) {
    const TmaGroup& d = groups[red[blockIdx.y]];
    const int64_t mn = static_cast<int64_t>(d.M) * d.N;
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < mn;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int m = static_cast<int>(r % d.M), n = static_cast<int>(r / d.M);
        double s = 0.0;
        // Split order is fixed (deterministic); loads are batched 8 at a time so
        // their L2 latencies overlap instead of serialising on the running sum.
        const double* src = d.ws + r;
        int sp = 0;
        for (; sp + 8 <= d.splits; sp += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = src[(sp + u) * mn];
#pragma unroll
            for (int u = 0; u < 8; ++u) s += v[u];
        }
        for (; sp < d.splits; ++sp) s += src[sp * mn];
        double* c = d.C + m + static_cast<int64_t>(n) * d.ldc;
        *c = d.beta == 0.0 ? d.alpha * s : d.alpha * s + d.beta * *c;
    }
}

bool ok16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

bool tma_gemm_enabled() {
    static const int en = [] {  // thread-safe one-time read
        const char* e = std::getenv("TS_GEMM_TMA");
        return (e && e[0] == '0') ? 0 : 1;
    }();
    return en == 1 && encode_fn() != nullptr;
}

// Returns false (nothing launched) when the problems do not fit the TMA kernel.
bool launch_tma_gemm(Layout layout, const std::vector<GemmProblem>& probs, CallScratch& sc, int num_sms, int* launched) {
    *launched = 0;
    if (!tma_gemm_enabled() || layout == Layout::NN) return false;  // NN handled as MN with an n-contiguous B only
    const bool mn = layout == Layout::NT;
    std::vector<TmaGroup> groups;
    int64_t units = 0;
    int64_t total_tiles = 0;
    for (const GemmProblem& p : probs) {
        if (p.M <= 0 || p.N <= 0) continue;
        if (p.batch != 1) return false;
        if (!ok16(p.A) || !ok16(p.B) || (p.lda & 1) || (p.ldb & 1)) return false;
        total_tiles += static_cast<int64_t>((p.M + kBM - 1) / kBM) * ((p.N + kBN - 1) / kBN);
    }
    if (total_tiles == 0) return true;
    set_max_smem(gemm_tma_kernel<false>, static_cast<int>(kSmemBytes));  // per device
    set_max_smem(gemm_tma_kernel<true>, static_cast<int>(kSmemBytes));
    set_max_smem(gemm_tma_kernel_pk<false>, static_cast<int>(kSmemBytes));
    set_max_smem(gemm_tma_kernel_pk<true>, static_cast<int>(kSmemBytes));
    static const int occ = [] {  // thread-safe one-time query (same on every B200)
        int o = 0;
        TS_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, gemm_tma_kernel<false>, kThreads, kSmemBytes));
        return std::max(o, 1);
    }();
    const int64_t slots = static_cast<int64_t>(num_sms) * occ;
    size_t ws_elems = 0;
    std::vector<int> red;
    for (const GemmProblem& p : probs) {
        if (p.M <= 0 || p.N <= 0) continue;
        TmaGroup gdesc;
        std::memset(&gdesc, 0, sizeof(gdesc));
        // KK (TN): A stored K×M (k contiguous, ld lda), B stored K×N.
        // MN (NT): A stored M×K (m contiguous), B stored N×K (n contiguous).
        bool okA, okB;
        if (!mn) {
            okA = make_map(&gdesc.ta, p.A, p.K, p.M, p.lda, kBM);
            okB = make_map(&gdesc.tb, p.B, p.K, p.N, p.ldb, kBN);
        } else {
            okA = make_map(&gdesc.ta, p.A, p.M, p.K, p.lda, kBK);
            okB = make_map(&gdesc.tb, p.B, p.N, p.K, p.ldb, kBK);
        }
        if (!okA || !okB) return false;
        gdesc.C = p.C;
        gdesc.ldc = p.ldc;
        gdesc.M = p.M;
        gdesc.N = p.N;
        gdesc.K = p.K;
        gdesc.alpha = p.alpha;
        gdesc.beta = p.beta;
        gdesc.tiles_m = (p.M + kBM - 1) / kBM;
        gdesc.tiles_n = (p.N + kBN - 1) / kBN;
        const int64_t tiles = static_cast<int64_t>(gdesc.tiles_m) * gdesc.tiles_n;
        // Wave-quantisation-aware split-K over the whole launch (see gemm.cu).
        int splits = 1;
        if (p.K > 4 * kBK) {
            const int maxs = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(64, p.K / (4 * kBK))));
            double best = -1.0;
            std::vector<double> eff(static_cast<size_t>(maxs) + 1, 0.0);
            for (int s = 1; s <= maxs; ++s) {
                const int64_t u = total_tiles * s;
                const int64_t waves = (u + slots - 1) / slots;
                eff[static_cast<size_t>(s)] = static_cast<double>(u) / static_cast<double>(waves * slots);
                best = std::max(best, eff[static_cast<size_t>(s)]);
            }
            for (int s = 1; s <= maxs; ++s)
                if (eff[static_cast<size_t>(s)] >= best - 0.03) {
                    splits = s;
                    break;
                }
        }
        int kps = (p.K + splits - 1) / splits;
        kps = std::max(kBK, ((kps + kBK - 1) / kBK) * kBK);
        splits = std::max(1, (p.K + kps - 1) / kps);
        gdesc.splits = splits;
        gdesc.k_per_split = kps;
        gdesc.unit_begin = units;
        units += tiles * splits;
        if (splits > 1) {
            red.push_back(static_cast<int>(groups.size()));
            ws_elems += static_cast<size_t>(p.M) * p.N * splits;
        }
        groups.push_back(gdesc);
    }
    if (!ws_elems) {
    } else {
        double* ws = sc.alloc_n<double>(ws_elems);
        size_t off = 0;
        for (int gi : red) {
            TmaGroup& d = groups[static_cast<size_t>(gi)];
            d.ws = ws + off;
            off += static_cast<size_t>(d.M) * d.N * d.splits;
        }
    }
    const int ng = static_cast<int>(groups.size());
    const bool packed = ng <= kPackGroups;
    TmaPack pk;
    const TmaGroup* d_groups = nullptr;
    if (packed) {
        std::memset(&pk, 0, sizeof(pk));
        std::memcpy(pk.g, groups.data(), groups.size() * sizeof(TmaGroup));
        for (size_t i = 0; i < red.size(); ++i) pk.red[i] = red[i];
    } else {
        d_groups = static_cast<const TmaGroup*>(sc.upload(groups.data(), groups.size() * sizeof(TmaGroup)));
    }
    if (sc.before_next_gemm) {
        TS_CUDA_CHECK(cudaEventRecord(sc.before_next_gemm, sc.stream()));
        sc.before_next_gemm = nullptr;
    }
    const unsigned grid = static_cast<unsigned>(units);
    if (packed) {
        if (mn) gemm_tma_kernel_pk<true><<<grid, kThreads, kSmemBytes, sc.stream()>>>(pk, ng);
        else gemm_tma_kernel_pk<false><<<grid, kThreads, kSmemBytes, sc.stream()>>>(pk, ng);
    } else {
        if (mn) gemm_tma_kernel<true><<<grid, kThreads, kSmemBytes, sc.stream()>>>(d_groups, ng);
        else gemm_tma_kernel<false><<<grid, kThreads, kSmemBytes, sc.stream()>>>(d_groups, ng);
    }
    TS_LAUNCH_CHECK();
    if (sc.after_next_gemm) {
        TS_CUDA_CHECK(cudaEventRecord(sc.after_next_gemm, sc.stream()));
        sc.after_next_gemm = nullptr;
    }
    *launched = 1;
    if (!red.empty()) {
        int64_t maxel = 0;
        for (int gi : red) maxel = std::max<int64_t>(maxel, static_cast<int64_t>(groups[static_cast<size_t>(gi)].M) * groups[static_cast<size_t>(gi)].N);
        const int64_t blocks = std::min<int64_t>((maxel + 255) / 256, 4LL * num_sms);
        const dim3 rgrid(static_cast<unsigned>(std::max<int64_t>(blocks, 1)), static_cast<unsigned>(red.size()));
        if (packed) {
            tma_splitk_reduce_pk<<<rgrid, 256, 0, sc.stream()>>>(pk);
        } else {
            const int* d_red = static_cast<const int*>(sc.upload(red.data(), red.size() * sizeof(int)));
            tma_splitk_reduce<<<rgrid, 256, 0, sc.stream()>>>(d_groups, d_red);
        }
        TS_LAUNCH_CHECK();
        *launched = 2;
    }
    sc.launches += *launched;
    return true;
}

}  // namespace ts
