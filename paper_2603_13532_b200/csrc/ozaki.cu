// ozaki.cu — FP64 GEMM C = α·AᵀB on the int8 tcgen05 tensor cores (Ozaki
// splitting), for the KRP sum's HBM-heavy contractions whose long operand is
// the stacked factor matrix F (stage A: Zᵀ = Fᵀ Ω; stage E: Ptᵀ = Fᵀ Y).
//
// FP64 on sm_100a has no tcgen05 kind: the only FP64 tensor instruction is the
// warp-level DMMA, whose 37 TFLOP/s makes stages A/C/E compute-bound (0.77 ms
// each at config 5, 90 % of that peak).  Reading F once from HBM takes ~0.23 ms.
// Splitting every fp64 value into byte "digits" turns the product into a short
// sum of exact integer GEMMs, which the 5th-generation tensor cores run at
// 4.5 POPS with int32 accumulators in TMEM:
//
//   x_A = rint(a · 2^(54 − e_A))   (e_A: the exponent bound of a's column of F,
//                                   computed once per upload; |x_A| < 2^54)
//   x_A = Σ_{t=0..6} d_t 2^(8(6−t)),   balanced signed byte digits d_t ∈ [−128, 127]
//   a·b ≈ Σ_{i+j ≤ 6} (d_i^A d_j^B) 2^(e_A + e_B − 12 − 8(i+j))
//
// The 28 byte products with i + j ≤ 6 (the others weigh < 2^-56 of the leading
// one) go to 7 int32 accumulators (one per i + j, TMEM columns 64·w); a split
// of K ≤ 16384 cannot overflow them (7 · 128² · 16384 < 2^31).  All digits are
// signed, so slice i of A meets slices 0..6−i of B in ONE MMA with B's slices
// concatenated along N (their accumulators are consecutive column blocks): 10
// MMAs per 32-K step instead of 28.  The epilogue combines the accumulators
// exactly in two int64 halves.  Measured error ≤ 1e-16 of Σ|a||b|
// (tools/ozaki_probe.py) — below an fp64 GEMM's own rounding.
//
// Kernel: one CTA per (128 columns of F, K split), 192 threads.
//   warp 4 (producer): TMA of the fp64 F tile (4 boxes of 16 K × 128 columns,
//     128-byte swizzle, double-buffered) and a bulk copy of the pre-sliced B
//     operand (7 × 64 rows × 64 bytes, already in the UMMA layout);
//   warps 0-3 (converters, thread = row of Fᵀ): fp64 → 7 byte slices, written
//     in the K-major 64-byte-swizzled UMMA layout; later the epilogue (TMEM →
//     registers → fp64);
//   warp 5: allocates TMEM (512 columns) and issues the 56 tcgen05.mma.kind::i8
//     of a chunk from one elected lane; tcgen05.commit releases the slices.
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "gemm.cuh"
#include "kernels.cuh"
#include "tma.cuh"
#include "tucksum_cuda.h"

namespace ts {
namespace {

constexpr int kOzM = 128;                    // tile rows (columns of F)
constexpr int kOzN = 64;                     // B columns (padded)
constexpr int kOzKC = 32;                    // K per chunk = one MMA K step (32 int8)
constexpr int kOzS = 7;                      // byte slices
constexpr int kOzConv = 256;                 // converter threads: (row, 16-K half)
constexpr int kOzThreads = kOzConv + 64;     // + producer warp + MMA warp
constexpr int kFStages = 3;
constexpr int kFBox = 16 * kOzM * 8;         // one 16-K box of fp64: 16 KB
constexpr int kFStage = 2 * kFBox;           // 32 KB
constexpr int kASlice = kOzM * kOzKC;        // 4 KB
constexpr int kBSlice = kOzN * kOzKC;        // 2 KB
constexpr int kAStage = kOzS * kASlice;      // 28 KB
constexpr int kBStage = kOzS * kBSlice;      // 14 KB
constexpr int kOffA = kFStages * kFStage;    // 96 KB
constexpr int kOffB = kOffA + 2 * kAStage;   // 152 KB
constexpr int kOffBar = kOffB + 2 * kBStage;  // 180 KB
constexpr size_t kOzSmem = 1024 + kOffBar + 256;
// TS variant (F digits staged in TMEM, not shared memory): no A stages, so the
// fp64 ring is 5 deep; TMEM columns 448..503 hold one chunk's 7 digit slices
// (8 columns of 4 bytes each = 32 K per row).
constexpr int kFStagesTS = 5;
constexpr int kOffBTS = kFStagesTS * kFStage;     // 160 KB
constexpr int kOffBarTS = kOffBTS + 2 * kBStage;  // 188 KB
constexpr size_t kOzSmemTS = 1024 + kOffBarTS + 256;
constexpr int kTmemA = kOzS * kOzN;               // first TMEM column of the digit slices
constexpr int kOzMaxK = 16384;               // int32 headroom: 7 · 128² · K < 2^31

// TS_OZAKI_TRACE=1: clock64 stamps of CTA 0's chunks 8..11 (converter thread 0
// and the MMA thread), printed by ts_debug_ozaki_gemm (tools/ozaki_stageA.py).
__device__ long long g_oz_trace[64];
// Same switch: per-chunk start clocks of four CTAs (block 0, 200, 400, 570) in
// [i][0..95], and [i][96..99] = kernel entry, loop start, loop end, epilogue end.
__device__ long long g_oz_trace2[4][100];

struct alignas(64) OzGroup {
    CUtensorMap fa;        // F: dims {K (contiguous), M}, box {16, 128}, 128B swizzle
    const uint8_t* bsl;    // B slices: [K/32 chunks][7][64 rows × 32 B, UMMA K-major SW32 image]
    const int* aexp;       // per column of F
    const int* bexp;       // per column of B
    double* C;             // out(m, n) at C[n + m·ldc]
    double* ws;            // split partials [split][M][64]
    int64_t ldc;
    int M, N, K;
    int splits, tiles_m, k_per_split;
    int a_mn;              // F stored M-contiguous (stage C: F_n as the n × R left operand)
    int c_colmajor;        // out(m, n) at C[m + n·ldc] instead of C[n + m·ldc]
    double alpha, beta;
    int64_t unit_begin;
};

// Byte offset of (row, k) in a K-major, 32-byte-swizzled tile of 32-byte rows
// (Swizzle<1,4,3>: address bit 4 ^= bit 7).
__host__ __device__ __forceinline__ unsigned sw32(unsigned row, unsigned k) {
    return row * 32u + ((((k >> 4) ^ (row >> 2)) & 1u) << 4) + (k & 15u);
}

// Exponent bound e (max |x| < 2^e) from the largest high word of |x| seen: the
// floor for zero / subnormal vectors, kOzExpBad when a NaN or Inf was among the
// values (their high words compare above every finite one), so the products
// come out NaN like an FP64 GEMM's would instead of as finite garbage.
constexpr int kOzExpBad = 1 << 20;
__device__ __forceinline__ int exp_bound_of(int max_hi) {
    const int b = max_hi >> 20;  // biased exponent: 2^(b-1023) ≤ max < 2^(b-1022)
    return b == 0 ? kOzExpFloor : (b == 0x7ff ? kOzExpBad : max(b - 1022, kOzExpFloor));
}
__device__ __forceinline__ int abs_hi(double x) { return __double2hiint(x) & 0x7fffffff; }

__device__ __forceinline__ double pow2(int e) {  // 2^e, normal range
    return __hiloint2double((e + 1023) << 20, 0);
}

__device__ __forceinline__ uint64_t umma_desc_sw32(unsigned saddr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);  // start address
    d |= static_cast<uint64_t>(1) << 16;                    // LBO (unused for swizzled K-major)
    d |= static_cast<uint64_t>(256 >> 4) << 32;             // SBO: 8 rows × 32 B
    d |= static_cast<uint64_t>(1) << 46;                    // version (sm_100)
    d |= static_cast<uint64_t>(6) << 61;                    // SWIZZLE_32B
    return d;
}

__device__ __forceinline__ uint32_t idesc_s8(int n) {
    return (2u << 4) | (1u << 7) | (1u << 10)           // S32 accumulate, A and B signed int8, K-major
           | (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(kOzM >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// Same with the A operand read from tensor memory (lane = row, 4 K bytes per column).
__device__ __forceinline__ void mma_i8_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void tmem_st4(uint32_t taddr, unsigned a, unsigned b, unsigned c, unsigned d) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(taddr), "r"(a), "r"(b), "r"(c),
                 "r"(d)
                 : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// Balanced signed byte digits of 4 values: x = round(v·2^(54−e)) for the column
// (row) exponent bound e (|v| < 2^e, so |x| < 2^54 — the balanced range is
// ±0x7F7F…7F ≈ ±0.996·2^55, a full 2^55 would overflow); y = x + 0x80…80
// (7 bytes) lies in [0, 2^56) and byte t of y, minus 128, is digit t — i.e. byte
// XOR 0x80 as int8.  Word t holds digit t (t = 0: the top, weight 2^48) of each
// value, value u in byte u.
//
// INTEGER ONLY.  FP64 instructions (DMUL, DFMA, F2I.S64.F64) issue ~14× slower
// while tcgen05 MMAs are running on the SM (tools/i8_mma_rate.cu: 2.2 → 30.9
// cycles per warp instruction per SMSP; integer ALU ops are unaffected), which
// serialised conversion and MMAs.  With v = ±M·2^(E−1075) (M the 53-bit
// significand), x = ±((M·4 >> sh) + 1) >> 1 for sh = e + 1022 − E ≥ 0 — round
// half away from zero; zeros and subnormals (E = 0) shift out (e ≥ −900).
// cexp = e + 1022.
__device__ __forceinline__ void transpose_digits(const unsigned* hi, const unsigned* lo, unsigned* w);

// The same digits through the FP64 pipe (DMUL + F2I.S64.F64, round to nearest
// even): fewer instructions, for code that runs while no MMA is in flight.
// scale = 2^(54 − e).
__device__ __forceinline__ void digits4_fp(const double* v, double scale, unsigned* w) {
    unsigned hi[4], lo[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const unsigned long long y = static_cast<unsigned long long>(__double2ll_rn(v[u] * scale)) + 0x80808080808080ull;
        hi[u] = static_cast<unsigned>(y >> 32);
        lo[u] = static_cast<unsigned>(y);
    }
    transpose_digits(hi, lo, w);
}

__device__ __forceinline__ void digits4(const double* v, int cexp, unsigned* w) {
    unsigned hi[4], lo[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const unsigned vh = static_cast<unsigned>(__double2hiint(v[u])), vl = static_cast<unsigned>(__double2loint(v[u]));
        const unsigned sh = min(static_cast<unsigned>(cexp) - ((vh >> 20) & 0x7ffu), 63u);
        const unsigned mh = (vh & 0xfffffu) | 0x100000u;
        const unsigned long long m4 = ((static_cast<unsigned long long>(mh) << 32) | vl) << 2;
        unsigned long long y = ((m4 >> sh) + 1ull) >> 1;
        const unsigned long long neg = static_cast<unsigned long long>(static_cast<long long>(static_cast<int>(vh) >> 31));
        y = ((y ^ neg) - neg) + 0x80808080808080ull;
        hi[u] = static_cast<unsigned>(y >> 32);
        lo[u] = static_cast<unsigned>(y);
    }
    transpose_digits(hi, lo, w);
}

// 4 × 7 byte transpose: two PRMT stages (pairs, then quads), then the XOR.
__device__ __forceinline__ void transpose_digits(const unsigned* hi, const unsigned* lo, unsigned* w) {
    const unsigned l01a = __byte_perm(lo[0], lo[1], 0x5140), l01b = __byte_perm(lo[0], lo[1], 0x7362);
    const unsigned l23a = __byte_perm(lo[2], lo[3], 0x5140), l23b = __byte_perm(lo[2], lo[3], 0x7362);
    const unsigned h01a = __byte_perm(hi[0], hi[1], 0x5140), h01b = __byte_perm(hi[0], hi[1], 0x7362);
    const unsigned h23a = __byte_perm(hi[2], hi[3], 0x5140), h23b = __byte_perm(hi[2], hi[3], 0x7362);
    w[0] = __byte_perm(h01b, h23b, 0x5410) ^ 0x80808080u;  // byte 6
    w[1] = __byte_perm(h01a, h23a, 0x7632) ^ 0x80808080u;  // byte 5
    w[2] = __byte_perm(h01a, h23a, 0x5410) ^ 0x80808080u;  // byte 4
    w[3] = __byte_perm(l01b, l23b, 0x7632) ^ 0x80808080u;  // byte 3
    w[4] = __byte_perm(l01b, l23b, 0x5410) ^ 0x80808080u;  // byte 2
    w[5] = __byte_perm(l01a, l23a, 0x7632) ^ 0x80808080u;  // byte 1
    w[6] = __byte_perm(l01a, l23a, 0x5410) ^ 0x80808080u;  // byte 0
}

// kIntGroups (TS): how many of a thread's four 4-value groups are converted with
// integer instructions while the previous chunk's MMAs run; the rest go through
// the FP64 pipe after those MMAs retired (FP64 issue is ~14× slower under MMAs).
// Up to kOzPack groups travel as a __grid_constant__ kernel parameter (no
// descriptor upload = no memcpy node in front of the kernel inside a CUDA graph).
constexpr int kOzPack = 8;
struct OzPack {
    OzGroup g[kOzPack];
    int red[kOzPack];
};

template <bool kTS, int kIntGroups>
__device__ __forceinline__ void ozaki_gemm_body(const OzGroup* __restrict__ groups, int ngroups, int variant) {
    constexpr int kFStages = kTS ? kFStagesTS : ts::kFStages;
    constexpr int kOffB = kTS ? kOffBTS : ts::kOffB;
    constexpr int kOffBar = kTS ? kOffBarTS : ts::kOffBar;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* f_full = reinterpret_cast<uint64_t*>(smem + kOffBar);  // [kFStages]
    uint64_t* f_empty = f_full + kFStages;                             // [kFStages]
    uint64_t* b_full = f_empty + kFStages;                             // [2]
    uint64_t* a_full = b_full + 2;                                     // [2]
    uint64_t* mma_done = a_full + 2;                                   // [2]
    uint64_t* acc_full = mma_done + 2;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(acc_full + 1);

    const int tslot = blockIdx.x == 0 ? 0 : blockIdx.x == 200 ? 1 : blockIdx.x == 400 ? 2 : blockIdx.x == 570 ? 3 : -1;
    const bool tr2 = variant == 9 && tslot >= 0 && threadIdx.x == 0;
    if (tr2) g_oz_trace2[tslot][96] = clock64();
    const int64_t unit = blockIdx.x;
    int lo = 0, hi = ngroups - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (groups[mid].unit_begin <= unit) lo = mid;
        else hi = mid - 1;
    }
    const OzGroup& G = groups[lo];
    const int64_t local = unit - G.unit_begin;
    const int tm = static_cast<int>(local % G.tiles_m);
    const int sp = static_cast<int>(local / G.tiles_m);
    const int m0 = tm * kOzM;
    const int kbeg = sp * G.k_per_split;
    const int kend = min(G.K, kbeg + G.k_per_split);
    const int nk = (kend - kbeg + kOzKC - 1) / kOzKC;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kFStages; ++s) {
            mbar_init(&f_full[s], 1);
            mbar_init(&f_empty[s], kOzConv);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&b_full[s], 1);
            mbar_init(&a_full[s], kTS ? kOzConv / 32 : 1);
            mbar_init(&mma_done[s], 1);
        }
        mbar_init(acc_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    constexpr int kProdWarp = kOzConv / 32, kMmaWarp = kProdWarp + 1;
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_holder)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = *tmem_holder;

    if (warp == kProdWarp) {
        if (lane == 0) {  // producer: fp64 F tiles (TMA) and pre-sliced B (bulk copy)
            const uint8_t* bsrc = G.bsl + static_cast<int64_t>(kbeg / kOzKC) * kBStage;
            for (int c = 0; c < nk; ++c) {
                const int s = c % kFStages;
                if (c >= kFStages) mbar_wait(&f_empty[s], ((c / kFStages) - 1) & 1);
                mbar_expect_tx(&f_full[s], kFStage);
                const int k0 = kbeg + c * kOzKC;
                if (G.a_mn) {  // 8 boxes of 16 m × 32 k (m contiguous)
                    for (int b = 0; b < 8; ++b)
                        tma_load_2d(smem + s * kFStage + b * (kFStage / 8), &G.fa, m0 + 16 * b, k0, &f_full[s]);
                } else {       // 2 boxes of 16 k × 128 m (k contiguous)
                    tma_load_2d(smem + s * kFStage, &G.fa, k0, m0, &f_full[s]);
                    tma_load_2d(smem + s * kFStage + kFBox, &G.fa, k0 + 16, m0, &f_full[s]);
                }
                // TS: the small operand's slices are fetched by converter thread 0 right
                // after it saw the previous chunk's MMAs retire, so this warp's fp64
                // ring runs ahead of the MMAs by its full depth (coupling the two
                // loads here kept only ~one chunk of F in flight per SM).
                if (kTS || variant == 1) continue;
                const int s2 = c & 1;
                if (c >= 2) mbar_wait(&mma_done[s2], ((c >> 1) - 1) & 1);  // B stage free again
                mbar_expect_tx(&b_full[s2], kBStage);
                bulk_load(smem + kOffB + s2 * kBStage, bsrc + static_cast<int64_t>(c) * kBStage, kBStage, &b_full[s2]);
            }
        }
    } else if (warp == kMmaWarp) {
        if (lane == 0 && variant == 1) mma_commit(acc_full);
        if (lane == 0 && variant != 1) {  // MMA issuer: per chunk 10 MMAs — slice i of A against slices
                          // 0..6-i of B concatenated along N (their accumulators
                          // w = i..6 are consecutive TMEM column blocks)
            const unsigned a_base = smem_u32(smem + (kTS ? 0 : kOffA)), b_base = smem_u32(smem + kOffB);
            for (int c = 0; c < nk; ++c) {
                const int s2 = c & 1;
                // TS: one digit stage in TMEM (phase flips every chunk); SS: two in shared memory
                const bool tr = variant == 9 && blockIdx.x == 0 && c >= 8 && c < 12;
                // B arrived a chunk ago; the digits are the late operand, so wait for them last
                mbar_wait(&b_full[s2], (c >> 1) & 1);
                if (tr) g_oz_trace[(c - 8) * 16 + 9] = clock64();
                if (kTS) mbar_wait(&a_full[0], c & 1);
                else mbar_wait(&a_full[s2], (c >> 1) & 1);
                if (tr) g_oz_trace[(c - 8) * 16 + 8] = clock64();
                asm volatile("tcgen05.fence::after_thread_sync;\n");
                const unsigned ab = a_base + s2 * kAStage, bb = b_base + s2 * kBStage;
#pragma unroll
                for (int i = 0; i < (variant == 2 ? 0 : variant == 4 ? 1 : kOzS); ++i) {
                    const int ntot = kOzN * (kOzS - i);
                    const uint32_t acc = (c > 0 || i > 0) ? 1u : 0u;
                    const int n1 = min(ntot, 256);
                    if (kTS) {
                        const uint32_t ta = tmem + static_cast<uint32_t>(kTmemA + 8 * i);
                        mma_i8_ts(tmem + static_cast<uint32_t>(kOzN * i), ta, umma_desc_sw32(bb), idesc_s8(n1), acc);
                        if (ntot > 256)
                            mma_i8_ts(tmem + static_cast<uint32_t>(kOzN * i + 256), ta, umma_desc_sw32(bb + 4 * kBSlice),
                                      idesc_s8(ntot - 256), acc);
                    } else {
                        const uint64_t da = umma_desc_sw32(ab + i * kASlice);
                        mma_i8(tmem + static_cast<uint32_t>(kOzN * i), da, umma_desc_sw32(bb), idesc_s8(n1), acc);
                        if (ntot > 256)
                            mma_i8(tmem + static_cast<uint32_t>(kOzN * i + 256), da, umma_desc_sw32(bb + 4 * kBSlice),
                                   idesc_s8(ntot - 256), acc);
                    }
                }
                mma_commit(&mma_done[s2]);
                if (tr) g_oz_trace[(c - 8) * 16 + 10] = clock64();
            }
            mma_commit(acc_full);
        }
    } else {  // warps 0-7: converters (thread = row, 16-K half), then the epilogue
        const int row = threadIdx.x & (kOzM - 1), g = threadIdx.x >> 7;
        const int ea_raw = (m0 + row < G.M) ? G.aexp[m0 + row] : 0;
        const int ea = ea_raw == kOzExpBad ? 0 : ea_raw;  // a NaN / Inf row: its outputs are NaN (epilogue)
        const int cexp = ea + 1022;
        const double scale = pow2(54 - ea);
        const uint8_t* bsrc = G.bsl + static_cast<int64_t>(kbeg / kOzKC) * kBStage;
        auto load_b = [&](int c) {  // pre-sliced small operand of chunk c → B stage c & 1
            mbar_expect_tx(&b_full[c & 1], kBStage);
            bulk_load(smem + kOffB + (c & 1) * kBStage, bsrc + static_cast<int64_t>(c) * kBStage, kBStage, &b_full[c & 1]);
        };
        if (kTS && threadIdx.x == 0 && variant != 1 && nk > 0) load_b(0);
        for (int c = 0; c < nk; ++c) {
            const int s = c % kFStages, s2 = c & 1;
            const bool tr = variant == 9 && blockIdx.x == 0 && threadIdx.x == 0 && c >= 8 && c < 12;
            if (tr) g_oz_trace[(c - 8) * 16 + 0] = clock64();
            if (tr2 && c < 96) g_oz_trace2[tslot][c] = clock64();
            if (tr2 && c == 0) g_oz_trace2[tslot][97] = clock64();
            mbar_wait(&f_full[s], (c / kFStages) & 1);
            if (tr) g_oz_trace[(c - 8) * 16 + 1] = clock64();
            double v[16];
            if (G.a_mn) {  // box row/16: line k (32 lines of 128 B), element row%16 in it
                const unsigned base = smem_u32(smem + s * kFStage + (row >> 4) * (kFStage / 8));
                const int e = row & 15;
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    const int k = 16 * g + u;
                    v[u] = lds64(base + k * 128 + ((((e >> 1) ^ (k & 7)) << 4) | ((e & 1) << 3)));
                }
            } else {
                const unsigned base = smem_u32(smem + s * kFStage + g * kFBox) + row * 128;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const double2 t2 = lds128(base + ((q ^ (row & 7)) << 4));
                    v[2 * q] = t2.x;
                    v[2 * q + 1] = t2.y;
                }
            }
            mbar_arrive(&f_empty[s]);
            if (variant == 1) continue;
            unsigned wq[4][kOzS];
            if (kTS) {
                // Integer-converted groups first: they overlap the previous chunk's MMAs.
#pragma unroll
                for (int qd = 0; qd < kIntGroups; ++qd) digits4(v + 4 * qd, cexp, wq[qd]);
                if (tr) g_oz_trace[(c - 8) * 16 + 2] = clock64();
                // The single TMEM digit stage is free once the previous chunk's MMAs
                // retired; from here until this chunk's MMAs start the FP64 pipe runs
                // at full speed, so the remaining groups take the short FP64 route.
                if (c >= 1) mbar_wait(&mma_done[(c - 1) & 1], ((c - 1) >> 1) & 1);
                if (tr) g_oz_trace[(c - 8) * 16 + 3] = clock64();
                asm volatile("tcgen05.fence::after_thread_sync;\n");
#pragma unroll
                for (int qd = kIntGroups; qd < 4; ++qd) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) asm volatile("" : "+d"(v[4 * qd + u]));  // keep it after the wait
                    digits4_fp(v + 4 * qd, scale, wq[qd]);
                }
                // Digits go straight to tensor memory: this thread's row is TMEM lane
                // `row`, its 16 K bytes of slice t are columns kTmemA + 8t + 4g .. +3.
                const uint32_t ta = tmem + (static_cast<uint32_t>(32 * (warp & 3)) << 16) + static_cast<uint32_t>(kTmemA + 4 * g);
                if (tr) g_oz_trace[(c - 8) * 16 + 4] = clock64() + (wq[3][0] & 0);  // after the FP64 groups
#pragma unroll
                for (int t = 0; t < (variant == 3 ? 0 : kOzS); ++t)
                    tmem_st4(ta + static_cast<uint32_t>(8 * t), wq[0][t], wq[1][t], wq[2][t], wq[3][t]);
                asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
                if (tr) g_oz_trace[(c - 8) * 16 + 5] = clock64();
                asm volatile("tcgen05.fence::before_thread_sync;\n");
                __syncwarp();
                if (lane == 0) mbar_arrive(&a_full[0]);
                if (tr) g_oz_trace[(c - 8) * 16 + 6] = clock64();
                // off the critical path: the next chunk's small-operand slices (their
                // stage was chunk c−1's, whose MMAs retired above)
                if (threadIdx.x == 0 && c + 1 < nk) load_b(c + 1);
                __syncwarp();
                continue;
            }
#pragma unroll
            for (int qd = 0; qd < 4; ++qd) digits4(v + 4 * qd, cexp, wq[qd]);
            if (c >= 2) mbar_wait(&mma_done[s2], ((c >> 1) - 1) & 1);  // A stage free again
            unsigned char* as = smem + kOffA + s2 * kAStage;
#pragma unroll
            for (int t = 0; t < (variant == 3 ? 0 : kOzS); ++t) {
                const unsigned addr = smem_u32(as + t * kASlice + sw32(row, 16 * g));
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(wq[0][t]), "r"(wq[1][t]),
                             "r"(wq[2][t]), "r"(wq[3][t]));
            }
            // The converters' generic-proxy stores must be visible to the tensor
            // core (async proxy): a named barrier over the converters, then ONE
            // proxy fence (fences are cumulative) and one arrival.
            asm volatile("bar.sync 1, %0;\n" ::"n"(kOzConv) : "memory");
            if (threadIdx.x == 0) {
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                mbar_arrive(&a_full[s2]);
            }
        }
        // ---- epilogue: row `row` (TMEM lane 32·(warp % 4) + lane), column groups
        // 4g..4g+3 of 8.  S = Σ_w acc_w 2^(8(6-w)) combined exactly in two int64
        // halves (u·2^32 + t), then a·b = S · 2^(e_A + e_B − 60).
        if (tr2) g_oz_trace2[tslot][98] = clock64();
        mbar_wait(acc_full, 0);
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        const int m = m0 + row;
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(32 * (warp & 3)) << 16);
        // the group's fields in registers (the TMEM-load asm's memory clobber would reload them)
        const int n_cols = G.N, c_colmajor = G.c_colmajor;
        const int* __restrict__ bexp = G.bexp;
        double* const Cout = G.C;
        const int64_t ldc = G.ldc;
        const double alpha = G.alpha, beta = G.beta;
        double* const ws_row = G.splits > 1 ? G.ws + (static_cast<int64_t>(sp) * G.M + m) * kOzN : nullptr;
#pragma unroll 1
        for (int q = 4 * g; q < 4 * g + 4; ++q) {
            uint32_t r[kOzS][8];
#pragma unroll
            for (int w = 0; w < kOzS; ++w)
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                             : "=r"(r[w][0]), "=r"(r[w][1]), "=r"(r[w][2]), "=r"(r[w][3]), "=r"(r[w][4]), "=r"(r[w][5]),
                               "=r"(r[w][6]), "=r"(r[w][7])
                             : "r"(lane_base + static_cast<uint32_t>(kOzN * w + 8 * q)));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            if (m < G.M) {
                double val[8];
#pragma unroll
                for (int cc = 0; cc < 8; ++cc) {
                    const int n = 8 * q + cc;
                    const long long u = (static_cast<long long>(static_cast<int>(r[0][cc])) << 16) +
                                        (static_cast<long long>(static_cast<int>(r[1][cc])) << 8) +
                                        static_cast<long long>(static_cast<int>(r[2][cc]));
                    const long long t = (static_cast<long long>(static_cast<int>(r[3][cc])) << 24) +
                                        (static_cast<long long>(static_cast<int>(r[4][cc])) << 16) +
                                        (static_cast<long long>(static_cast<int>(r[5][cc])) << 8) +
                                        static_cast<long long>(static_cast<int>(r[6][cc]));
                    const int be = n < n_cols ? bexp[n] : 0;
                    const double sc2 = (ea_raw == kOzExpBad || be == kOzExpBad) ? __longlong_as_double(0x7ff8000000000000ll)
                                                                                : pow2(ea + be - 60);
                    val[cc] = n < n_cols ? fma(static_cast<double>(u), 4294967296.0, static_cast<double>(t)) * sc2 : 0.0;
                }
                if (ws_row != nullptr) {  // split partial: this row's 64 bytes of the [m][64] block, 16 B at a time
                    double2* dst = reinterpret_cast<double2*>(ws_row + 8 * q);
#pragma unroll
                    for (int cc = 0; cc < 8; cc += 2) dst[cc >> 1] = make_double2(val[cc], val[cc + 1]);
                } else {
#pragma unroll
                    for (int cc = 0; cc < 8; ++cc) {
                        const int n = 8 * q + cc;
                        if (n >= n_cols) continue;
                        double* cp = c_colmajor ? Cout + m + static_cast<int64_t>(n) * ldc : Cout + n + static_cast<int64_t>(m) * ldc;
                        *cp = beta == 0.0 ? alpha * val[cc] : alpha * val[cc] + beta * *cp;
                    }
                }
            }
        }
    }
    if (tr2) g_oz_trace2[tslot][99] = clock64();
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == kMmaWarp) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

template <bool kTS, int kIntGroups>
__global__ void __launch_bounds__(kOzThreads, 1) ozaki_gemm_kernel(const OzGroup* __restrict__ groups, int ngroups,
                                                                   int variant) {
    ozaki_gemm_body<kTS, kIntGroups>(groups, ngroups, variant);
}
template <bool kTS, int kIntGroups>
__global__ void __launch_bounds__(kOzThreads, 1) ozaki_gemm_kernel_pk(const __grid_constant__ OzPack pk, int ngroups,
                                                                      int variant) {
    ozaki_gemm_body<kTS, kIntGroups>(pk.g, ngroups, variant);
}

__device__ __forceinline__ void ozaki_splitk_reduce_body(const OzGroup* __restrict__ groups, const int* __restrict__ red);
__global__ void ozaki_splitk_reduce(const OzGroup* __restrict__ groups, const int* __restrict__ red) {
    ozaki_splitk_reduce_body(groups, red);
}
__global__ void ozaki_splitk_reduce_pk(const __grid_constant__ OzPack pk) { ozaki_splitk_reduce_body(pk.g, pk.red); }

__device__ __forceinline__ void ozaki_splitk_reduce_body(const OzGroup* __restrict__ groups, const int* __restrict__ red) {
    const OzGroup& d = groups[red[blockIdx.y]];
    const int64_t mn = static_cast<int64_t>(d.M) * kOzN;
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < mn;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int m = static_cast<int>(r / kOzN), n = static_cast<int>(r % kOzN);
        if (n >= d.N) continue;
        double s = 0.0;
        for (int sp = 0; sp < d.splits; ++sp) s += d.ws[sp * mn + r];  // fixed order: deterministic
        double* c = d.c_colmajor ? d.C + m + static_cast<int64_t>(n) * d.ldc : d.C + n + static_cast<int64_t>(m) * d.ldc;
        *c = d.beta == 0.0 ? d.alpha * s : d.alpha * s + d.beta * *c;
    }
}

// exp[j] = e with max_i |X[j·ld + i·es]| < 2^e: a block per vector j of `rows`
// elements (es = 1: the columns of a column-major matrix; es = ld of the
// stored matrix, ld = 1: its rows).
__global__ void col_exponent_kernel(const double* __restrict__ X, int64_t ld, int64_t rows, int64_t es,
                                    int* __restrict__ out) {
    const int j = blockIdx.x;
    const double* c = X + static_cast<int64_t>(j) * ld;
    int mx = 0;
    for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) mx = max(mx, abs_hi(c[i * es]));
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    __shared__ int red[32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) mx = max(mx, red[w]);
        out[j] = exp_bound_of(mx);
    }
}

// exp[i] = e with max_j |X[i, j]| < 2^e (column-major rows × cols, ld): a block
// per 32 rows, 32 column lanes per row (lane y takes columns y, y + 32, …; a warp
// reads 32 consecutive rows = 256 contiguous bytes), shared-memory max over lanes.
__global__ void __launch_bounds__(1024) row_exponent_kernel(const double* __restrict__ X, int64_t ld, int64_t rows,
                                                            int64_t cols, int* __restrict__ out) {
    __shared__ int red[32][33];
    const int64_t i = blockIdx.x * 32LL + threadIdx.x;
    int mx = 0;
    if (i < rows) {
        const double* x = X + i;
        int64_t j = threadIdx.y;
        for (; j + 96 < cols; j += 128) {  // four independent loads in flight
            const int a = abs_hi(x[j * ld]), b = abs_hi(x[(j + 32) * ld]);
            const int c = abs_hi(x[(j + 64) * ld]), d = abs_hi(x[(j + 96) * ld]);
            mx = max(max(mx, max(a, b)), max(c, d));
        }
        for (; j < cols; j += 32) mx = max(mx, abs_hi(x[j * ld]));
    }
    red[threadIdx.y][threadIdx.x] = mx;
    __syncthreads();
    if (threadIdx.y == 0 && i < rows) {
#pragma unroll
        for (int y = 1; y < 32; ++y) mx = max(mx, red[y][threadIdx.x]);
        out[i] = exp_bound_of(mx);
    }
}

__global__ void fill_exponent_kernel(int* __restrict__ out, int64_t n) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) out[i] = kOzExpFloor;
}

__global__ void reduce_exponent_kernel(int* __restrict__ e, int64_t n, int buckets) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    int m = e[i];
    for (int b = 1; b < buckets; ++b) m = max(m, e[b * n + i]);
    e[i] = m;
}

// B operand (K × N column-major, ld, N ≤ 64) → 7 balanced byte digits in the
// UMMA smem image per 32-K chunk; thread = (chunk, column n, 16-K group).
__global__ void ozaki_slice_b_kernel(const double* __restrict__ B, int64_t ldb, int K, int N, const int* __restrict__ bexp,
                                     uint8_t* __restrict__ out, int nchunks, int trans) {
    const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t total = static_cast<int64_t>(nchunks) * kOzN * 2;
    if (tid >= total) return;
    const int g = static_cast<int>(tid & 1);
    const int n = static_cast<int>((tid >> 1) % kOzN);
    const int c = static_cast<int>(tid / (2 * kOzN));
    const double scale = (n < N && bexp[n] != kOzExpBad) ? pow2(54 - bexp[n]) : 0.0;
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
        const int k = c * kOzKC + 16 * g + u;
        v[u] = (n < N && k < K) ? (trans ? B[n + static_cast<int64_t>(k) * ldb] : B[k + static_cast<int64_t>(n) * ldb]) : 0.0;
    }
    unsigned wq[4][kOzS];
#pragma unroll
    for (int qd = 0; qd < 4; ++qd) digits4_fp(v + 4 * qd, scale, wq[qd]);
    uint8_t* base = out + static_cast<int64_t>(c) * kBStage;
#pragma unroll
    for (int t = 0; t < kOzS; ++t)
        *reinterpret_cast<uint4*>(base + t * kBSlice + sw32(static_cast<unsigned>(n), static_cast<unsigned>(16 * g))) =
            make_uint4(wq[0][t], wq[1][t], wq[2][t], wq[3][t]);
}

// Exponents + slices of several small operands in ONE launch (stages C, E and F2
// prepare one per mode on every call): block (n, p) handles column n of operand
// p — the column's exponent bound by a block reduction, then its 7 digit planes.
struct OzPrep {
    const double* B;
    int64_t ldb;
    int K, N, trans, nchunks;
    int* exp;
    uint8_t* slices;
};

struct OzPrepPack {
    OzPrep p[kOzPack];
};

__global__ void __launch_bounds__(256) ozaki_prepare_b_kernel(const __grid_constant__ OzPrepPack preps) {
    const OzPrep& P = preps.p[blockIdx.y];
    const int n = blockIdx.x;
    const bool live = n < P.N;
    const int64_t es = P.trans ? P.ldb : 1;  // element stride along k
    const double* col = P.B + (P.trans ? static_cast<int64_t>(n) : static_cast<int64_t>(n) * P.ldb);
    __shared__ int red[8];
    __shared__ int s_exp;
    int mx = 0;
    if (live)
        for (int k = threadIdx.x; k < P.K; k += 256) mx = max(mx, abs_hi(col[k * es]));
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) mx = max(mx, red[w]);
        const int e = exp_bound_of(mx);
        s_exp = e;
        P.exp[n] = e;
    }
    __syncthreads();
    const double scale = (live && s_exp != kOzExpBad) ? pow2(54 - s_exp) : 0.0;
    for (int idx = threadIdx.x; idx < 2 * P.nchunks; idx += 256) {
        const int c = idx >> 1, g = idx & 1;
        double v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int k = c * kOzKC + 16 * g + u;
            v[u] = (live && k < P.K) ? col[k * es] : 0.0;
        }
        unsigned wq[4][kOzS];
#pragma unroll
        for (int qd = 0; qd < 4; ++qd) digits4_fp(v + 4 * qd, scale, wq[qd]);
        uint8_t* base = P.slices + static_cast<int64_t>(c) * kBStage;
#pragma unroll
        for (int t = 0; t < kOzS; ++t)
            *reinterpret_cast<uint4*>(base + t * kBSlice + sw32(static_cast<unsigned>(n), static_cast<unsigned>(16 * g))) =
                make_uint4(wq[0][t], wq[1][t], wq[2][t], wq[3][t]);
    }
}

}  // namespace

// TS_OZAKI_TS=0: the F digits go through shared memory (SS MMAs) instead of TMEM.
static bool ozaki_ts() {
    static const int en = [] {
        const char* e = std::getenv("TS_OZAKI_TS");
        return (e && e[0] == '0') ? 0 : 1;
    }();
    return en == 1;
}

// TS_OZAKI_INT_GROUPS=0..4: the integer / FP64 split of the in-kernel conversion (default 2).
static int ozaki_int_groups() {
    static const int n = [] {
        const char* e = std::getenv("TS_OZAKI_INT_GROUPS");
        return e ? std::atoi(e) : 2;
    }();
    return n;
}

bool ozaki_enabled() {
    static const int en = [] {
        const char* e = std::getenv("TS_OZAKI");
        return (e && e[0] == '0') ? 0 : 1;
    }();
    return en == 1 && encode_fn() != nullptr;
}

void launch_row_exponents(const double* X, int64_t ld, int64_t rows, int64_t cols, int* out, CallScratch& sc) {
    if (rows <= 0) return;
    row_exponent_kernel<<<static_cast<unsigned>((rows + 31) / 32), dim3(32, 32), 0, sc.stream()>>>(X, ld, rows, cols, out);
    TS_LAUNCH_CHECK();
    sc.launches += 1;
}

void launch_fill_exponents(int* out, int64_t n, CallScratch& sc) {
    if (n <= 0) return;
    fill_exponent_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, sc.stream()>>>(out, n);
    TS_LAUNCH_CHECK();
    sc.launches += 1;
}

void launch_reduce_exponents(int* e, int64_t n, int buckets, CallScratch& sc) {
    if (n <= 0 || buckets <= 1) return;
    reduce_exponent_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, sc.stream()>>>(e, n, buckets);
    TS_LAUNCH_CHECK();
    sc.launches += 1;
}

void launch_col_exponents(const double* X, int64_t ld, int64_t rows, int64_t cols, int* out, CallScratch& sc) {
    if (cols <= 0) return;
    col_exponent_kernel<<<static_cast<unsigned>(cols), 256, 0, sc.stream()>>>(X, ld, rows, 1, out);
    TS_LAUNCH_CHECK();
    sc.launches += 1;
}

size_t ozaki_b_bytes(int K) { return static_cast<size_t>((K + kOzKC - 1) / kOzKC) * kBStage; }

OzOperand prepare_ozaki_b(const double* B, int64_t ldb, int K, int N, CallScratch& sc, bool trans) {
    OzOperand o{};
    if (N > kOzN) throw Error(TS_UNSUPPORTED, "ozaki: B has more than 64 columns");
    o.exp = sc.alloc_n<int>(static_cast<size_t>(kOzN));
    o.slices = sc.alloc_n<uint8_t>(ozaki_b_bytes(K));
    o.K = K;
    o.N = N;
    prepare_ozaki_b_into(B, ldb, K, N, o, sc, trans);
    return o;
}

void prepare_ozaki_b_into(const double* B, int64_t ldb, int K, int N, const OzOperand& o, CallScratch& sc, bool trans) {
    if (N > kOzN) throw Error(TS_UNSUPPORTED, "ozaki: B has more than 64 columns");
    const int nchunks = (K + kOzKC - 1) / kOzKC;
    if (trans) {  // B(k, n) = stored[n + k·ld]: the stored matrix's rows, a block each
        col_exponent_kernel<<<static_cast<unsigned>(N), 256, 0, sc.stream()>>>(B, 1, K, ldb, o.exp);
        TS_LAUNCH_CHECK();
        sc.launches += 1;
    } else {
        launch_col_exponents(B, ldb, K, N, o.exp, sc);
    }
    const int64_t threads = static_cast<int64_t>(nchunks) * kOzN * 2;
    ozaki_slice_b_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, sc.stream()>>>(B, ldb, K, N, o.exp,
                                                                                             o.slices, nchunks, trans ? 1 : 0);
    TS_LAUNCH_CHECK();
    sc.launches += 1;
}

std::vector<OzOperand> prepare_ozaki_b_batch(const std::vector<OzSmall>& reqs, CallScratch& sc) {
    std::vector<OzOperand> out(reqs.size());
    std::vector<OzPrep> preps(reqs.size());
    for (size_t i = 0; i < reqs.size(); ++i) {
        const OzSmall& r = reqs[i];
        if (r.N > kOzN) throw Error(TS_UNSUPPORTED, "ozaki: B has more than 64 columns");
        OzOperand& o = out[i];
        o.exp = sc.alloc_n<int>(static_cast<size_t>(kOzN));
        o.slices = sc.alloc_n<uint8_t>(ozaki_b_bytes(r.K));
        o.K = r.K;
        o.N = r.N;
        preps[i] = OzPrep{r.B, r.ldb, r.K, r.N, r.trans ? 1 : 0, (r.K + kOzKC - 1) / kOzKC, o.exp, o.slices};
    }
    for (size_t i0 = 0; i0 < reqs.size(); i0 += kOzPack) {  // descriptors as a kernel parameter, ≤ 8 per launch
        const size_t cnt = std::min<size_t>(kOzPack, reqs.size() - i0);
        OzPrepPack pk;
        std::memset(&pk, 0, sizeof(pk));
        std::memcpy(pk.p, preps.data() + i0, cnt * sizeof(OzPrep));
        ozaki_prepare_b_kernel<<<dim3(kOzN, static_cast<unsigned>(cnt)), 256, 0, sc.stream()>>>(pk);
        TS_LAUNCH_CHECK();
        sc.launches += 1;
    }
    return out;
}

// K splits of a launch with `tiles` 128-column tiles (one CTA per SM): the count
// (≥ min_splits for the int32 headroom, ≥ 24 chunks each) that wastes the least
// of the last wave, charging each CTA about four chunk-times of pipeline fill
// and epilogue.  Config 5 (192 tiles, 256 chunks): 3 splits = 3.89 waves.
static int pick_splits(int64_t tiles, int kchunks, int min_splits, int num_sms) {
    static const int forced = [] {
        const char* e = std::getenv("TS_OZAKI_SPLITS");
        return e ? std::atoi(e) : 0;
    }();
    if (forced > 0) return std::max(forced, min_splits);
    int best = min_splits;
    double best_eff = -1.0;
    for (int s = min_splits; s <= 16; ++s) {
        const int cps = (kchunks + s - 1) / s;
        if (s > min_splits && cps < 24) break;
        const int64_t units = tiles * ((kchunks + cps - 1) / cps);
        const int64_t waves = (units + num_sms - 1) / num_sms;
        const double eff = static_cast<double>(units) / static_cast<double>(waves * num_sms) * cps / (cps + 4.0);
        if (eff > best_eff + 1e-9) {
            best_eff = eff;
            best = s;
        }
    }
    return best;
}

bool launch_ozaki_gemm(const std::vector<OzProblem>& probs, CallScratch& sc, int num_sms, int* launched) {
    *launched = 0;
    if (!ozaki_enabled()) return false;
    for (const OzProblem& p : probs)
        if (p.M > 0 && (p.B.N > kOzN || (reinterpret_cast<uintptr_t>(p.F) & 15u) || (p.ldf & 1))) return false;
    set_max_smem(ozaki_gemm_kernel_pk<false, 4>, static_cast<int>(kOzSmem));
    set_max_smem(ozaki_gemm_kernel_pk<true, 0>, static_cast<int>(kOzSmemTS));
    set_max_smem(ozaki_gemm_kernel_pk<true, 1>, static_cast<int>(kOzSmemTS));
    set_max_smem(ozaki_gemm_kernel_pk<true, 2>, static_cast<int>(kOzSmemTS));
    set_max_smem(ozaki_gemm_kernel_pk<true, 3>, static_cast<int>(kOzSmemTS));
    set_max_smem(ozaki_gemm_kernel_pk<true, 4>, static_cast<int>(kOzSmemTS));
    set_max_smem(ozaki_gemm_kernel<false, 4>, static_cast<int>(kOzSmem));
    set_max_smem(ozaki_gemm_kernel<true, 0>, static_cast<int>(kOzSmemTS));
    set_max_smem(ozaki_gemm_kernel<true, 1>, static_cast<int>(kOzSmemTS));
    set_max_smem(ozaki_gemm_kernel<true, 2>, static_cast<int>(kOzSmemTS));
    set_max_smem(ozaki_gemm_kernel<true, 3>, static_cast<int>(kOzSmemTS));
    set_max_smem(ozaki_gemm_kernel<true, 4>, static_cast<int>(kOzSmemTS));
    std::vector<OzGroup> groups;
    std::vector<int> red;
    int64_t units = 0, tiles = 0;
    for (const OzProblem& p : probs)
        if (p.M > 0) tiles += (p.M + kOzM - 1) / kOzM;
    size_t ws_elems = 0;
    for (const OzProblem& p : probs) {
        if (p.M <= 0) continue;
        OzGroup g;
        std::memset(&g, 0, sizeof(g));
        if (p.a_mn ? !make_map_box(&g.fa, p.F, p.M, p.K, p.ldf, 16, kOzKC) : !make_map(&g.fa, p.F, p.K, p.M, p.ldf, kOzM))
            return false;
        g.a_mn = p.a_mn ? 1 : 0;
        g.c_colmajor = p.c_colmajor ? 1 : 0;
        g.bsl = p.B.slices;
        g.aexp = p.aexp;
        g.bexp = p.B.exp;
        g.C = p.C;
        g.ldc = p.ldc;
        g.M = p.M;
        g.N = p.B.N;
        g.K = p.K;
        g.alpha = p.alpha;
        g.beta = p.beta;
        g.tiles_m = (p.M + kOzM - 1) / kOzM;
        // K splits: ≤ kOzMaxK per split (int32 headroom), then enough units for
        // about three waves over the SMs (one CTA per SM), at least 32 chunks each.
        const int kchunks = (p.K + kOzKC - 1) / kOzKC;
        const int splits = pick_splits(tiles, kchunks, std::max(1, (p.K + kOzMaxK - 1) / kOzMaxK), num_sms);
        const int cps = (kchunks + splits - 1) / splits;
        g.k_per_split = cps * kOzKC;
        g.splits = (kchunks + cps - 1) / cps;
        g.unit_begin = units;
        units += static_cast<int64_t>(g.tiles_m) * g.splits;
        if (g.splits > 1) {
            red.push_back(static_cast<int>(groups.size()));
            ws_elems += static_cast<size_t>(g.splits) * p.M * kOzN;
        }
        groups.push_back(g);
    }
    if (groups.empty()) return true;
    if (ws_elems) {
        double* ws = sc.alloc_n<double>(ws_elems);
        size_t off = 0;
        for (int gi : red) {
            OzGroup& d = groups[static_cast<size_t>(gi)];
            d.ws = ws + off;
            off += static_cast<size_t>(d.splits) * d.M * kOzN;
        }
    }
    const int ng = static_cast<int>(groups.size());
    const bool packed = ng <= kOzPack;
    OzPack pk;
    const OzGroup* d_groups = nullptr;
    if (packed) {
        std::memset(&pk, 0, sizeof(pk));
        std::memcpy(pk.g, groups.data(), groups.size() * sizeof(OzGroup));
        for (size_t i = 0; i < red.size(); ++i) pk.red[i] = red[i];
    } else {
        d_groups = static_cast<const OzGroup*>(sc.upload(groups.data(), groups.size() * sizeof(OzGroup)));
    }
    if (sc.before_next_gemm) {
        TS_CUDA_CHECK(cudaEventRecord(sc.before_next_gemm, sc.stream()));
        sc.before_next_gemm = nullptr;
    }
    static const int variant = [] {  // timing ablations (tools/ozaki_probe.py)
        const char* e = std::getenv("TS_OZAKI_VARIANT");
        return e ? std::atoi(e) : 0;
    }();
    const unsigned grid = static_cast<unsigned>(units);
#define TS_OZ_LAUNCH(TSF, IG, SMEM)                                                                              \
    do {                                                                                                         \
        if (packed) ozaki_gemm_kernel_pk<TSF, IG><<<grid, kOzThreads, SMEM, sc.stream()>>>(pk, ng, variant);       \
        else ozaki_gemm_kernel<TSF, IG><<<grid, kOzThreads, SMEM, sc.stream()>>>(d_groups, ng, variant);           \
    } while (0)
    if (!ozaki_ts()) {
        TS_OZ_LAUNCH(false, 4, kOzSmem);
    } else {
        switch (ozaki_int_groups()) {
            case 0: TS_OZ_LAUNCH(true, 0, kOzSmemTS); break;
            case 1: TS_OZ_LAUNCH(true, 1, kOzSmemTS); break;
            case 3: TS_OZ_LAUNCH(true, 3, kOzSmemTS); break;
            case 4: TS_OZ_LAUNCH(true, 4, kOzSmemTS); break;
            default: TS_OZ_LAUNCH(true, 2, kOzSmemTS); break;
        }
    }
#undef TS_OZ_LAUNCH
    TS_LAUNCH_CHECK();
    if (sc.after_next_gemm) {
        TS_CUDA_CHECK(cudaEventRecord(sc.after_next_gemm, sc.stream()));
        sc.after_next_gemm = nullptr;
    }
    *launched = 1;
    if (variant == 9) {
        long long tr[64];
        TS_CUDA_CHECK(cudaStreamSynchronize(sc.stream()));
        TS_CUDA_CHECK(cudaMemcpyFromSymbol(tr, g_oz_trace, sizeof(tr)));
        for (int c = 0; c < 4; ++c) {
            const long long* r = tr + 16 * c;
            const long long b0 = tr[0];
            std::fprintf(stderr,
                         "oz-trace chunk %d: conv start %lld f_full %lld int %lld mma_done(c-1) %lld fp %lld st %lld arrive %lld | "
                         "mma: a_full %lld b_full %lld issued %lld\n",
                         8 + c, r[0] - b0, r[1] - b0, r[2] - b0, r[3] - b0, r[4] - b0, r[5] - b0, r[6] - b0, r[8] - b0,
                         r[9] - b0, r[10] - b0);
        }
    }
    if (variant == 9) {
        long long t2[4][100];
        TS_CUDA_CHECK(cudaMemcpyFromSymbol(t2, g_oz_trace2, sizeof(t2)));
        for (int i = 0; i < 4; ++i) {
            const long long* r = t2[i];
            std::fprintf(stderr, "oz-trace2 cta-slot %d: entry->loop %lld loop %lld (acc wait+epilogue) %lld; chunk periods:", i,
                         r[97] - r[96], r[98] - r[97], r[99] - r[98]);
            for (int c = 1; c < 86; c += 6) std::fprintf(stderr, " %lld", r[c] - r[c - 1]);
            std::fprintf(stderr, "\n");
        }
    }
    if (!red.empty()) {
        int64_t maxel = 0;
        for (int gi : red) maxel = std::max<int64_t>(maxel, static_cast<int64_t>(groups[static_cast<size_t>(gi)].M) * kOzN);
        const int64_t blocks = std::min<int64_t>((maxel + 255) / 256, 4LL * num_sms);
        const dim3 rgrid(static_cast<unsigned>(std::max<int64_t>(blocks, 1)), static_cast<unsigned>(red.size()));
        if (packed) {
            ozaki_splitk_reduce_pk<<<rgrid, 256, 0, sc.stream()>>>(pk);
        } else {
            const int* d_red = static_cast<const int*>(sc.upload(red.data(), red.size() * sizeof(int)));
            ozaki_splitk_reduce<<<rgrid, 256, 0, sc.stream()>>>(d_groups, d_red);
        }
        TS_LAUNCH_CHECK();
        *launched = 2;
    }
    sc.launches += *launched;
    return true;
}

}  // namespace ts
