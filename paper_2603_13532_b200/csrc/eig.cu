// eig.cu — small symmetric eigensolver for ST-HOSVD's Gram fast path (stage G).
//
// Parallel two-sided Jacobi (reference semantics of sym_eig, src/kernels.cpp:70-86:
// symmetrise, eigendecompose, descending order) for n ≤ 64, in two kernels:
//
//  1. jacobi_values_kernel (one CTA) iterates on the matrix only.  A Jacobi round
//     must stream the whole matrix through shared memory, so a round costs what
//     that traffic costs; keeping the eigenvectors out of the loop and the
//     matrix in its upper triangle halves it.  Layout (all addresses fixed):
//       * positions 0..np-1 hold the players of a round-robin tournament; pair i
//         of every round is the position pair (2i, 2i+1); after each round the
//         players move by the circle-method permutation
//           dest(0) = 0, dest(1) = 2, dest(2i) = 2i+2 (1 ≤ i ≤ k-2),
//           dest(2k-2) = 2k-1, dest(2i+1) = 2i-1 (i ≥ 1),   k = np/2,
//         so over np-1 rounds every two players meet once (one sweep);
//       * warp i owns the row pair of pair i, lane j the column pair of pair j
//         (j ≥ i: upper triangle): two 16-byte loads give the 2×2 block, R_iᵀ·B·R_j
//         is formed in registers and stored at the permuted positions of the
//         next (ping-pong) buffer, transposed where the permutation crosses the
//         diagonal.
//     Every round's rotations are appended to a global log.
//  2. jacobi_vectors_kernel replays the log on the identity, one warp per row of
//     V across many SMs (rows evolve independently; the column permutation is a
//     pair of lane shifts), then writes the eigenpairs in descending order.
#include <cmath>
#include <cstdlib>

#include "kernels.cuh"

namespace ts {
namespace {

constexpr int kWorkWarps = 15;                 // worker warps of the values kernel (464 blocks at n = 64)
constexpr int kValWarps = kWorkWarps + 1;      // + the pivot warp
constexpr int kValThreads = 32 * kValWarps;
constexpr int kMaxNp = 64;
constexpr int kMaxSweeps = 40;

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

// θ = (b - a)/(2g), t = sign(θ)/(|θ| + sqrt(1 + θ²)), c = 1/sqrt(1 + t²), s = t·c;
// t from ~20-bit MUFU approximations, c Newton-refined so every rotation is
// orthogonal to working precision.
__device__ __forceinline__ void rotation(double a, double b, double g, double& c, double& s) {
    const double theta = (b - a) * rcp_approx(2.0 * g);
    const double at = fabs(theta);
    double t;
    if (at > 1e150) {
        t = 0.5 * rcp_approx(theta);
    } else {
        const double u = fma(theta, theta, 1.0);
        t = copysign(rcp_approx(at + u * rsqrt_approx(u)), theta);
    }
    const double w = fma(t, t, 1.0);
    double r = rsqrt_approx(w);
    r = r * fma(-0.5 * w, r * r, 1.5);
    r = r * fma(-0.5 * w, r * r, 1.5);
    c = r;
    s = t * c;
}

__device__ __forceinline__ int dest_of(int pos, int k) {
    if (pos == 0) return 0;
    if (pos == 1) return 2;
    if ((pos & 1) == 0) return pos == 2 * k - 2 ? 2 * k - 1 : pos + 2;
    return pos - 2;
}

// Storage of position (r, c), r ≤ c: even columns in the first half-row, odd in
// the second, so a warp's 8-byte accesses along a row of blocks are contiguous.
__device__ __forceinline__ int addr_of(int r, int c, int k) { return r * 2 * k + (c & 1) * k + (c >> 1); }
__device__ __forceinline__ int addr_sym(int r, int c, int k) { return r <= c ? addr_of(r, c, k) : addr_of(c, r, k); }
// Stored address of the element at positions (r, c) after the permutation.
__device__ __forceinline__ int addr_next(int r, int c, int k) { return addr_sym(dest_of(r, k), dest_of(c, k), k); }

// Rᵢᵀ·B·Rⱼ of one 2×2 block (R = [[c, s], [-s, c]]).
__device__ __forceinline__ void rotate_block(double2 ri, double2 rj, double a11, double a12, double a21, double a22,
                                             double& d11, double& d12, double& d21, double& d22) {
    const double b11 = ri.x * a11 - ri.y * a21, b12 = ri.x * a12 - ri.y * a22;
    const double b21 = ri.y * a11 + ri.x * a21, b22 = ri.y * a12 + ri.x * a22;
    d11 = rj.x * b11 - rj.y * b12;
    d12 = rj.y * b11 + rj.x * b12;
    d21 = rj.x * b21 - rj.y * b22;
    d22 = rj.y * b21 + rj.x * b22;
}

// rotation_or_identity without branches (both outcomes computed, then
// selected; the discarded one may be inf/NaN when apq = 0).
__device__ __forceinline__ double2 rotation_select(double a, double b, double g, double abs_floor) {
    const double theta = (b - a) * rcp_approx(2.0 * g);
    const double at = fabs(theta);
    const double u = fma(theta, theta, 1.0);
    const double t_small = copysign(rcp_approx(at + u * rsqrt_approx(u)), theta);
    const double t = at > 1e150 ? 0.5 * rcp_approx(theta) : t_small;
    const double w = fma(t, t, 1.0);
    double r = rsqrt_approx(w);
    r = r * fma(-0.5 * w, r * r, 1.5);
    r = r * fma(-0.5 * w, r * r, 1.5);
    const bool rotate = fabs(g) > abs_floor && g * g > 1e-30 * fabs(a * b);
    return rotate ? make_double2(r, t * r) : make_double2(1.0, 0.0);
}

__device__ __forceinline__ double2 rotation_or_identity(double app, double aqq, double apq, double abs_floor) {
    double c = 1.0, s = 0.0;
    if (fabs(apq) > abs_floor && apq * apq > 1e-30 * fabs(app * aqq)) rotation(app, aqq, apq, c, s);
    return make_double2(c, s);
}

// info[0] = rounds performed, info[1] = sweeps; diag_out[p] = A[p][p] at the end
// (position order), rot[round * k + i] = rotation of pair i in that round;
// prof (optional, TS_EIG_PROFILE) = {round-loop clocks, 0, 0, 0, rounds}; prof[7]
// on entry selects ablations.
//
// One barrier per round.  A round is issue-bound (every block costs the same
// few instructions), so the upper triangle's blocks are packed densely: worker
// warp w takes row pairs w and k-2-w (k blocks together, each row a contiguous
// lane segment) with every shared address precomputed.  The pivot warp's lane m
// updates diagonal block m and the off-diagonal block holding the entry that
// pairs the two players meeting in pair m NEXT round, then forms that next
// rotation — so round r+1's rotations are ready when round r's barrier opens and
// their latency hides behind the workers' updates of round r.
__global__ void __launch_bounds__(kValThreads, 1) jacobi_values_kernel(const double* __restrict__ Cin, int64_t ldc, int n,
                                                                    double2* __restrict__ rot,
                                                                    double* __restrict__ diag_out, int* __restrict__ info,
                                                                    unsigned long long* __restrict__ prof,
                                                                    int64_t strideC, int rel_only) {
    extern __shared__ __align__(16) double sm[];
    const int np = n + (n & 1);
    const int k = np / 2;
    // Batched launches (blockIdx.y = problem): per-problem operands and logs.
    Cin += blockIdx.y * strideC;
    rot += static_cast<int64_t>(blockIdx.y) * kMaxSweeps * (np - 1) * k;
    diag_out += static_cast<int64_t>(blockIdx.y) * np;
    info += 2 * blockIdx.y;
    if (blockIdx.y > 0) prof = nullptr;
    const int mat = np * np;
    // Layout: matrix buffers 0/1 (mat doubles each), rotations cs[2][kMaxNp/2],
    // then the rotation log ring (2·(np-1) rounds), flushed to global once per
    // sweep: a global store inside the round would stretch the round's barrier.
    const int ring = 2 * (np - 1);
    __shared__ int srcpos[kMaxNp];
    __shared__ unsigned xmask[kMaxNp / 2];
    __shared__ double red[2 * kValWarps];
    __shared__ double amax_s;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // Worker warps = enough for the round's off-diagonal blocks (launcher's choice,
    // ≤ kWorkWarps): fewer warps make every round's barriers cheaper at small n.
    const int nthreads = blockDim.x, nwork = nthreads / 32 - 1;
    for (int idx = tid; idx < np * np; idx += nthreads) {
        const int i = idx / np, j = idx % np;
        double v = 0.0;
        if (i < n && j < n && j >= i)
            v = 0.5 * (Cin[i + static_cast<int64_t>(j) * ldc] + Cin[j + static_cast<int64_t>(i) * ldc]);
        if (j >= i) sm[addr_of(i, j, k)] = v;
    }
    if (tid < np) srcpos[dest_of(tid, k)] = tid;
    if (tid < kMaxNp / 2) xmask[tid] = 0u;
    if (tid == 0) amax_s = 0.0;
    __syncthreads();
    {
        double mx = 0.0;
        for (int i = tid; i < n; i += nthreads) mx = fmax(mx, fabs(sm[addr_of(i, i, k)]));
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0 && mx > 0.0) atomicMax(reinterpret_cast<unsigned long long*>(&amax_s), __double_as_longlong(mx));
    }
    __syncthreads();
    // Entries below 1e-15·max|a_ii| sit under the Gram's rounding noise (the fast
    // path needs absolute accuracy only); rotating them only burns sweeps.
    // rel_only (block one-sided Jacobi, wide.cu): only the relative criterion
    // g² > 1e-30·|a·b| — tiny columns are orthogonalised too.
    const double abs_floor = rel_only ? 0.0 : 1e-15 * amax_s;

    const unsigned sbase = smem_u32(sm);
    const unsigned matb = static_cast<unsigned>(mat) * 8u;
    const unsigned csb = sbase + 2u * matb;  // cs buffer b at csb + 512·b
    const unsigned logb = csb + 1024u;       // ring slot s, pair m at logb + 16·(s·k + m)

    // Worker role: the t-th block (bi, bj), bj > bi, in row-major order among
    // those the pivot warp does not own (xmask[i] bit j: pivot-owned), so every
    // warp takes 32 consecutive blocks (one to three contiguous row segments).
    if (tid < k) {
        const int p = srcpos[2 * tid], q = srcpos[2 * tid + 1];
        atomicOr(&xmask[min(p, q) >> 1], 1u << (max(p, q) >> 1));
    }
    __syncthreads();
    bool work = false;
    unsigned la[4] = {0, 0, 0, 0}, sa[4] = {0, 0, 0, 0}, rio = 0, rjo = 0;
    if (warp < nwork) {
        const unsigned kmask = k == 32 ? 0xffffffffu : ((1u << k) - 1u);
        int t = tid, bi = -1, bj = -1;
        for (int i = 0; i < k - 1; ++i) {
            unsigned row = kmask & ~((2u << i) - 1u) & ~xmask[i];
            const int c = __popc(row);
            if (t < c) {
                for (int u = 0; u < t; ++u) row &= row - 1u;
                bi = i;
                bj = __ffs(row) - 1;
                break;
            }
            t -= c;
        }
        if (bi >= 0) {
            work = true;
            const int i2 = 2 * bi, j2 = 2 * bj;
            la[0] = 8u * addr_of(i2, j2, k);
            la[1] = 8u * addr_of(i2, j2 + 1, k);
            la[2] = 8u * addr_of(i2 + 1, j2, k);
            la[3] = 8u * addr_of(i2 + 1, j2 + 1, k);
            sa[0] = 8u * addr_next(i2, j2, k);
            sa[1] = 8u * addr_next(i2, j2 + 1, k);
            sa[2] = 8u * addr_next(i2 + 1, j2, k);
            sa[3] = 8u * addr_next(i2 + 1, j2 + 1, k);
            rio = 16u * bi;
            rjo = 16u * bj;
        }
    }
    // Pivot lane m: diagonal block m, the block (ea, eb) holding A[sp][sq] (sp/sq
    // the positions whose players form pair m next round; (ex, ey) within it), and
    // the diagonal blocks of sp and sq, whose rotated diagonal it recomputes
    // itself (same arithmetic as their owners) instead of exchanging it.  Lanes
    // ≥ k mirror lane k-1 and store nothing, so the warp stays converged.
    const bool pwarp = warp == nwork;
    const bool plane = pwarp && lane < k;
    unsigned dla[3] = {0, 0, 0}, dsa[3] = {0, 0, 0}, ela[4] = {0, 0, 0, 0}, esa[4] = {0, 0, 0, 0};
    unsigned pla[3] = {0, 0, 0}, qla[3] = {0, 0, 0};
    unsigned rmo = 0, rao = 0, rbo = 0, rpo = 0, rqo = 0;
    int ex = 0, ey = 0, sx = 0, sy = 0;
    if (pwarp) {
        const int m = min(lane, k - 1);
        const int sp = srcpos[2 * m], sq = srcpos[2 * m + 1];
        const int lo = min(sp, sq), hi = max(sp, sq);
        const int ea = lo >> 1, eb = hi >> 1;
        ex = lo & 1;
        ey = hi & 1;
        sx = sp & 1;
        sy = sq & 1;
        const int m2 = 2 * m, a2 = 2 * ea, b2 = 2 * eb, p2 = 2 * (sp >> 1), q2 = 2 * (sq >> 1);
        dla[0] = 8u * addr_of(m2, m2, k);
        dla[1] = 8u * addr_of(m2, m2 + 1, k);
        dla[2] = 8u * addr_of(m2 + 1, m2 + 1, k);
        dsa[0] = 8u * addr_next(m2, m2, k);
        dsa[1] = 8u * addr_next(m2, m2 + 1, k);
        dsa[2] = 8u * addr_next(m2 + 1, m2 + 1, k);
        ela[0] = 8u * addr_of(a2, b2, k);
        ela[1] = 8u * addr_of(a2, b2 + 1, k);
        ela[2] = 8u * addr_of(a2 + 1, b2, k);
        ela[3] = 8u * addr_of(a2 + 1, b2 + 1, k);
        esa[0] = 8u * addr_next(a2, b2, k);
        esa[1] = 8u * addr_next(a2, b2 + 1, k);
        esa[2] = 8u * addr_next(a2 + 1, b2, k);
        esa[3] = 8u * addr_next(a2 + 1, b2 + 1, k);
        pla[0] = 8u * addr_of(p2, p2, k);
        pla[1] = 8u * addr_of(p2, p2 + 1, k);
        pla[2] = 8u * addr_of(p2 + 1, p2 + 1, k);
        qla[0] = 8u * addr_of(q2, q2, k);
        qla[1] = 8u * addr_of(q2, q2 + 1, k);
        qla[2] = 8u * addr_of(q2 + 1, q2 + 1, k);
        rmo = 16u * m;
        rao = 16u * ea;
        rbo = 16u * eb;
        rpo = 16u * (sp >> 1);
        rqo = 16u * (sq >> 1);
        if (plane) {
            // Round 0's rotations from the input matrix.
            const double2 v = rotation_or_identity(lds64(sbase + dla[0]), lds64(sbase + dla[2]),
                                                   lds64(sbase + dla[1]), abs_floor);
            sts128(csb + rmo, v);
            sts128(logb + rmo, v);
        }
    }
    __syncthreads();

    unsigned cur = 0;  // byte offset of the current matrix buffer (0 or matb)
    int rounds = 0, sweeps_done = 0, wslot = 0;
    const long long tloop = clock64();
    // Timing ablations (TS_EIG_PROFILE=mode, tools/probe_jacobi.py): 4 = workers
    // skip their blocks, 8 = the pivot forms identity rotations.
    const int mode = prof != nullptr ? static_cast<int>(prof[7]) : 0;
    const bool skip_work = (mode & 4) != 0, skip_rot = (mode & 8) != 0;
    unsigned long long tail_clk = 0;
    double prev_off = 0.0;
    for (int sweep = 0; sweep < kMaxSweeps; ++sweep) {
        sweeps_done = sweep + 1;
        for (int r = 0; r < np - 1; ++r, ++rounds) {
            const unsigned A = sbase + cur, An = sbase + (matb - cur);
            const unsigned C = csb + (static_cast<unsigned>(rounds & 1) << 9);
            wslot = wslot + 1 == ring ? 0 : wslot + 1;
            if (!pwarp) {
                // Workers start their shared-memory traffic only once the pivot
                // warp's loads are queued ahead of it.
                asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
                if (work && !skip_work) {
                    const double2 ri = lds128(C + rio), rj = lds128(C + rjo);
                    double d11, d12, d21, d22;
                    rotate_block(ri, rj, lds64(A + la[0]), lds64(A + la[1]), lds64(A + la[2]), lds64(A + la[3]), d11,
                                 d12, d21, d22);
                    sts64(An + sa[0], d11);
                    sts64(An + sa[1], d12);
                    sts64(An + sa[2], d21);
                    sts64(An + sa[3], d22);
                }
            } else {
                // Loads in order of need: rotations, the entries that form the
                // next rotation, then this lane's two blocks.
                const double2 rp = lds128(C + rpo), rq = lds128(C + rqo), ra = lds128(C + rao), rb = lds128(C + rbo);
                const double2 rm = lds128(C + rmo);
                const double p11 = lds64(A + pla[0]), p12 = lds64(A + pla[1]), p22 = lds64(A + pla[2]);
                const double q11 = lds64(A + qla[0]), q12 = lds64(A + qla[1]), q22 = lds64(A + qla[2]);
                const double e11 = lds64(A + ela[0]), e12 = lds64(A + ela[1]), e21 = lds64(A + ela[2]),
                             e22 = lds64(A + ela[3]);
                const double a11 = lds64(A + dla[0]), a12 = lds64(A + dla[1]), a22 = lds64(A + dla[2]);
                asm volatile("bar.arrive 1, %0;" ::"r"(nthreads) : "memory");
                // Critical path first, branch-free so the block updates below can
                // fill the rotation's latency.  Rotated diagonal entry at sp / sq:
                // d11 of R_pᵀ·B·R_p, and d22 as d11 with (c, s) → (s, -c); the
                // pairing entry (ex, ey) of R_aᵀ·E·R_b.
                const double cp = sx ? rp.y : rp.x, spp = sx ? -rp.x : rp.y;
                const double cq = sy ? rq.y : rq.x, sqq = sy ? -rq.x : rq.y;
                const double app = cp * (cp * p11 - spp * p12) - spp * (cp * p12 - spp * p22);
                const double aqq = cq * (cq * q11 - sqq * q12) - sqq * (cq * q12 - sqq * q22);
                const double al = ex ? ra.y : ra.x, be = ex ? ra.x : -ra.y;
                const double ga = ey ? rb.y : rb.x, de = ey ? rb.x : -rb.y;
                const double e = ga * (al * e11 + be * e21) + de * (al * e12 + be * e22);
                const double2 v = skip_rot ? make_double2(1.0, 0.0) : rotation_select(app, aqq, e, abs_floor);
                double d11, d12, d21, d22;
                rotate_block(rm, rm, a11, a12, a12, a22, d11, d12, d21, d22);
                double f11, f12, f21, f22;
                rotate_block(ra, rb, e11, e12, e21, e22, f11, f12, f21, f22);
                if (plane) {
                    sts128(csb + (static_cast<unsigned>((rounds + 1) & 1) << 9) + rmo, v);
                    sts128(logb + 16u * static_cast<unsigned>(wslot * k) + rmo, v);
                    sts64(An + dsa[0], d11);
                    sts64(An + dsa[1], 0.5 * (d12 + d21));
                    sts64(An + dsa[2], d22);
                    sts64(An + esa[0], f11);
                    sts64(An + esa[1], f12);
                    sts64(An + esa[2], f21);
                    sts64(An + esa[3], f22);
                }
            }
            cur = matb - cur;
            __syncthreads();
        }
        const long long t_tail = clock64();
        {
            // This sweep's rounds sit in one contiguous half of the ring.
            const double2* logs = reinterpret_cast<const double2*>(sm + 2 * mat + 2 * kMaxNp) +
                                  static_cast<size_t>(sweep & 1) * (np - 1) * k;
            double2* dst = rot + static_cast<int64_t>(sweep) * (np - 1) * k;
            for (int e = tid; e < (np - 1) * k; e += nthreads) dst[e] = logs[e];
        }
        // off(A) and Σ diag² over the same block partition the rounds use (every
        // stored entry once; off-diagonal entries stand for both triangles).
        {
            const unsigned A = sbase + cur;
            double off = 0.0, dia = 0.0;
            if (work) {
                for (int u = 0; u < 4; ++u) {
                    const double x = lds64(A + la[u]);
                    off = fma(x, x, off);
                }
            } else if (plane) {
                const double a11 = lds64(A + dla[0]), a12 = lds64(A + dla[1]), a22 = lds64(A + dla[2]);
                dia = a11 * a11 + a22 * a22;
                off = a12 * a12;
                for (int u = 0; u < 4; ++u) {
                    const double x = lds64(A + ela[u]);
                    off = fma(x, x, off);
                }
            }
            off = warp_sum(off);
            dia = warp_sum(dia);
            if (lane == 0) {
                red[2 * warp] = off;
                red[2 * warp + 1] = dia;
            }
        }
        __syncthreads();
        // Stop at off(A) ≤ 1e-14·‖A‖_F, or once stalled on rounding noise ≤
        // 1e-12·‖A‖_F.  Every thread sums the per-warp partials in the same order,
        // so the decision is uniform; red[] is next written a whole sweep later.
        double o = 0.0, t = 0.0;
        for (int w = 0; w <= nwork; ++w) {
            o += red[2 * w];
            t += red[2 * w + 1];
        }
        o *= 2.0;
        t += o;
        const bool done = (o <= 1e-28 * t) || (o <= 1e-24 * t && o > 0.25 * prev_off);
        prev_off = o;
        if (prof != nullptr && tid == 0) tail_clk += clock64() + static_cast<long long>(done) - t_tail;
        if (done) break;
    }
    __syncthreads();  // the last flush and the final matrix are complete
    const double* A = sm + cur / 8;
    for (int p = tid; p < np; p += nthreads) diag_out[p] = A[addr_of(p, p, k)];
    if (tid == 0) {
        info[0] = rounds;
        info[1] = sweeps_done;
        if (prof) {
            prof[0] = static_cast<unsigned long long>(clock64() - tloop);
            prof[1] = prof[2] = 0;
            prof[3] = tail_clk;
            prof[4] = static_cast<unsigned long long>(rounds);
        }
    }
}


// One warp per row of V (row = original index 0..np-1): replay the rotation log
// on e_row with the same position permutation, then place each eigenvector
// column at its rank in descending eigenvalue order.  The padding player of an
// odd n never rotates (its row and column stay exactly zero); its final
// position is excluded from the ranking.
__global__ void __launch_bounds__(128) jacobi_vectors_kernel(int n, const double2* __restrict__ rot,
                                                             const double* __restrict__ diag_pos,
                                                             const int* __restrict__ info, double* __restrict__ lambda,
                                                             double* __restrict__ V, int64_t strideL, int64_t strideV) {
    const int np = n + (n & 1);
    const int k = np / 2;
    rot += static_cast<int64_t>(blockIdx.y) * kMaxSweeps * (np - 1) * k;
    diag_pos += static_cast<int64_t>(blockIdx.y) * np;
    info += 2 * blockIdx.y;
    lambda += blockIdx.y * strideL;
    V += blockIdx.y * strideV;
    const int lane = threadIdx.x & 31;
    const int row = blockIdx.x * 4 + (threadIdx.x >> 5);
    const int rounds = info[0];
    const bool vlane = lane < k;
    double f = (row == 2 * lane) ? 1.0 : 0.0;      // position 2·lane
    double g = (row == 2 * lane + 1) ? 1.0 : 0.0;  // position 2·lane + 1
    // The log streams through shared memory in chunks of kChunk rounds
    // (cp.async, double-buffered, shared by the CTA's four rows) so the
    // loop-carried chain never waits on L2.  Slots of lanes ≥ k hold the
    // identity, so the round loop has no branch.
    constexpr int kChunk = 32;
    __shared__ __align__(16) double2 logbuf[2][kChunk * 32];
    for (int e = threadIdx.x; e < 2 * kChunk * 32; e += blockDim.x)
        if ((e & 31) >= k) logbuf[e / (kChunk * 32)][e % (kChunk * 32)] = make_double2(1.0, 0.0);
    auto stage = [&](int chunk, int b) {
        const int r0 = chunk * kChunk;
        const int nr = min(kChunk, rounds - r0);
        for (int e = threadIdx.x; e < nr * k; e += blockDim.x)
            cp_async16(&logbuf[b][(e / k) * 32 + (e % k)], rot + static_cast<int64_t>(r0) * k + e, 16);
    };
    const int nchunks = (rounds + kChunk - 1) / kChunk;
    if (nchunks > 0) stage(0, 0);
    cp_async_commit();
    for (int ch = 0; ch < nchunks; ++ch) {
        if (ch + 1 < nchunks) stage(ch + 1, (ch + 1) & 1);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        const double2* cur = logbuf[ch & 1] + lane;
        const int nr = min(kChunk, rounds - ch * kChunk);
        // Lane l+1 ≥ 2 takes x of lane l, lane 1 takes y of lane 0 (the fixed
        // player's partner moves up); lane l < k-1 takes y of lane l+1 and lane
        // k-1 keeps its own x.  Two shuffles per round.
        double2 rr = cur[0];
        for (int ri = 0; ri < nr; ++ri) {
            const double2 rn = cur[min(ri + 1, kChunk - 1) * 32];
            const double x = rr.x * f - rr.y * g;
            const double y = rr.y * f + rr.x * g;
            const double up = __shfl_up_sync(0xffffffffu, lane == 0 ? y : x, 1);
            const double dn = __shfl_down_sync(0xffffffffu, y, 1);
            f = lane == 0 ? x : up;
            g = lane == k - 1 ? x : dn;
            rr = rn;
        }
        __syncthreads();
    }
    cp_async_wait<0>();
    if (!vlane || row >= n) return;
    int ppad = -1;
    if (np != n) {
        ppad = n;
        for (int r = 0; r < rounds; ++r) ppad = dest_of(ppad, k);
    }
    for (int h = 0; h < 2; ++h) {
        const int pos = 2 * lane + h;
        if (pos == ppad) continue;
        const double v = diag_pos[pos];
        int rank = 0;
        for (int i = 0; i < np; ++i) {
            if (i == ppad) continue;
            const double di = diag_pos[i];
            rank += (di > v) || (di == v && i < pos);
        }
        V[row + static_cast<int64_t>(rank) * n] = h == 0 ? f : g;
        if (row == 0) lambda[rank] = v;
    }
}

}  // namespace

unsigned long long* eig_probe_buffer() {
    static unsigned long long* const buf = [] {  // thread-safe one-time setup
        unsigned long long* p = nullptr;
        if (std::getenv("TS_EIG_PROFILE")) {
            TS_CUDA_CHECK(cudaMalloc(&p, 32 * sizeof(unsigned long long)));
            unsigned long long mode[32] = {};
            mode[7] = static_cast<unsigned long long>(std::atoi(std::getenv("TS_EIG_PROFILE")));
            TS_CUDA_CHECK(cudaMemcpy(p, mode, sizeof(mode), cudaMemcpyHostToDevice));
        }
        return p;
    }();
    return buf;
}

bool launch_sym_jacobi_pp(const double* C, int64_t ldc, int n, double* lambda, double* V, CallScratch& sc,
                          int* sweeps) {
    return launch_sym_jacobi_batched(C, ldc, n, lambda, V, sc, 1, 0, 0, 0, false, sweeps);
}

bool launch_sym_jacobi_batched(const double* C, int64_t ldc, int n, double* lambda, double* V, CallScratch& sc,
                               int count, int64_t strideC, int64_t strideL, int64_t strideV, bool rel_only,
                               int* sweeps) {
    const int np = n + (n & 1);
    if (np > kMaxNp || np < 4) return false;
    if (count < 1) return true;
    const int k = np / 2;
    const size_t smem = sizeof(double) * (2 * static_cast<size_t>(np) * np + 2 * kMaxNp + 4 * static_cast<size_t>(np - 1) * k + np);
    // Per-device, thread-safe smem attribute (runtime.hpp set_max_smem).
    set_max_smem(jacobi_values_kernel, 200 * 1024);
    auto* rot = sc.alloc_n<double2>(static_cast<size_t>(count) * kMaxSweeps * (np - 1) * k);
    double* dpos = sc.alloc_n<double>(static_cast<size_t>(count) * np);
    int* info = sc.alloc_n<int>(2 * static_cast<size_t>(count));
    // Upper bound on the off-diagonal blocks the workers own (all k(k-1)/2; the
    // pivot warp takes a few of them).  At n = 64 the 15-warp cap is exact.
    const int blocks = k * (k - 1) / 2;
    static const int force_warps = [] {
        const char* e = std::getenv("TS_EIG_WORK_WARPS");
        return e ? std::atoi(e) : 0;
    }();
    int work = std::min(kWorkWarps, std::max(1, (blocks + 31) / 32));
    if (force_warps > 0) work = std::max(work, std::min(force_warps, kWorkWarps));
    jacobi_values_kernel<<<dim3(1, static_cast<unsigned>(count)), 32 * (work + 1), smem, sc.stream()>>>(
        C, ldc, n, rot, dpos, info, eig_probe_buffer(), strideC, rel_only ? 1 : 0);
    TS_LAUNCH_CHECK();
    jacobi_vectors_kernel<<<dim3((np + 3) / 4, static_cast<unsigned>(count)), 128, 0, sc.stream()>>>(
        n, rot, dpos, info, lambda, V, strideL, strideV);
    TS_LAUNCH_CHECK();
    if (sweeps) TS_CUDA_CHECK(cudaMemcpyAsync(sweeps, info + 1, sizeof(int), cudaMemcpyDeviceToDevice, sc.stream()));
    sc.launches += 2;
    return true;
}

}  // namespace ts

// C ABI debug hook: per-phase clock totals of the last values-kernel run when
// TS_EIG_PROFILE is set (see jacobi_values_kernel), else zeros.
extern "C" void tsi_read_eig_profile(long long* out) {
    unsigned long long* p = ts::eig_probe_buffer();
    unsigned long long h[22] = {};
    if (p) TS_CUDA_CHECK(cudaMemcpy(h, p, sizeof(h), cudaMemcpyDeviceToHost));
    for (int i = 0; i < 22; ++i) out[i] = static_cast<long long>(h[i]);
}
