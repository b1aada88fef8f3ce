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

#include "kernels.cuh"

namespace ts {
namespace {

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;
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

// info[0] = rounds performed, info[1] = sweeps; diag_out[p] = A[p][p] at the end
// (position order), rot[round * k + i] = rotation of pair i in that round.
__global__ void __launch_bounds__(kThreads) jacobi_values_kernel(const double* __restrict__ Cin, int64_t ldc, int n,
                                                                 double2* __restrict__ rot, double* __restrict__ diag_out,
                                                                 int* __restrict__ info) {
    extern __shared__ __align__(16) double sm[];
    const int np = n + (n & 1);
    const int k = np / 2;
    const int ld = np + 2;    // even stride keeps column pairs 16-byte aligned
    const int mat = np * ld;  // buffer c at sm + c·mat (arithmetic selection stays in shared space)
    double2* cs = reinterpret_cast<double2*>(sm + 2 * mat);
    __shared__ int stop;
    __shared__ double red[2 * kWarps];
    __shared__ double prev_off, amax_s;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int idx = tid; idx < np * ld; idx += kThreads) {
        const int i = idx / ld, j = idx % ld;
        double v = 0.0;
        if (i < n && j < n && j >= i)
            v = 0.5 * (Cin[i + static_cast<int64_t>(j) * ldc] + Cin[j + static_cast<int64_t>(i) * ldc]);
        sm[idx] = v;
        sm[mat + idx] = 0.0;
    }
    if (tid == 0) {
        amax_s = 0.0;
        prev_off = 0.0;
        stop = 0;
    }
    __syncthreads();
    {
        double mx = 0.0;
        for (int i = tid; i < n; i += kThreads) mx = fmax(mx, fabs(sm[i * ld + i]));
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0 && mx > 0.0) atomicMax(reinterpret_cast<unsigned long long*>(&amax_s), __double_as_longlong(mx));
    }
    __syncthreads();
    // Entries below 1e-15·max|a_ii| sit under the Gram's rounding noise (the fast
    // path needs absolute accuracy only); rotating them only burns sweeps.
    const double abs_floor = 1e-15 * amax_s;

    // Fixed roles: warp i → row pair (2i, 2i+1), lane j → column pair (2j, 2j+1), j ≥ i.
    const bool active = warp < k && lane < k && lane >= warp;
    const bool dblk = lane == warp;
    const int i2 = 2 * warp, j2 = 2 * lane;
    int dst[4] = {0, 0, 0, 0};
    if (active) {
        const int ra[2] = {i2, i2 + 1}, cb[2] = {j2, j2 + 1};
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
            for (int y = 0; y < 2; ++y) {
                const int da = dest_of(ra[x], k), db = dest_of(cb[y], k);
                dst[2 * x + y] = min(da, db) * ld + max(da, db);
            }
    }

    int cur = 0, rounds = 0, sweeps_done = 0;
    for (int sweep = 0; sweep < kMaxSweeps; ++sweep) {
        sweeps_done = sweep + 1;
        for (int r = 0; r < np - 1; ++r, ++rounds) {
            const double* A = sm + cur * mat;
            double* An = sm + (cur ^ 1) * mat;
            if (tid < k) {
                const int p = 2 * tid, q = p + 1;
                const double app = A[p * ld + p], aqq = A[q * ld + q], apq = A[p * ld + q];
                double c = 1.0, s = 0.0;
                if (fabs(apq) > abs_floor && apq * apq > 1e-30 * fabs(app * aqq)) rotation(app, aqq, apq, c, s);
                const double2 v = make_double2(c, s);
                cs[tid] = v;
                rot[static_cast<int64_t>(rounds) * k + tid] = v;
            }
            __syncthreads();
            if (active) {
                const double2 ri = cs[warp], rj = cs[lane];
                const double2 top = *reinterpret_cast<const double2*>(A + i2 * ld + j2);        // (2i, 2j), (2i, 2j+1)
                const double2 bot = *reinterpret_cast<const double2*>(A + (i2 + 1) * ld + j2);  // (2i+1, 2j), (2i+1, 2j+1)
                const double a11 = top.x, a12 = top.y, a22 = bot.y;
                const double a21 = dblk ? top.y : bot.x;  // diagonal block: the lower entry mirrors a12
                // rows: Rᵀ·B with R = [[c, s], [-s, c]], then columns: ·R
                const double b11 = ri.x * a11 - ri.y * a21, b12 = ri.x * a12 - ri.y * a22;
                const double b21 = ri.y * a11 + ri.x * a21, b22 = ri.y * a12 + ri.x * a22;
                const double d11 = rj.x * b11 - rj.y * b12, d12 = rj.y * b11 + rj.x * b12;
                const double d21 = rj.x * b21 - rj.y * b22, d22 = rj.y * b21 + rj.x * b22;
                An[dst[0]] = d11;
                An[dst[3]] = d22;
                if (dblk) {
                    An[dst[1]] = 0.5 * (d12 + d21);
                } else {
                    An[dst[1]] = d12;
                    An[dst[2]] = d21;
                }
            }
            cur ^= 1;
            __syncthreads();
        }
        // Stop at off(A) ≤ 1e-14·‖A‖_F, or once stalled on rounding noise ≤ 1e-12·‖A‖_F.
        const double* A = sm + cur * mat;
        double off = 0.0, tot = 0.0;
        for (int idx = tid; idx < np * np; idx += kThreads) {
            const int i = idx / np, j = idx % np;
            if (j < i) continue;
            const double a = A[i * ld + j];
            const double w2 = (i == j) ? 1.0 : 2.0;
            tot = fma(w2 * a, a, tot);
            if (i != j) off = fma(w2 * a, a, off);
        }
        off = warp_sum(off);
        tot = warp_sum(tot);
        if (lane == 0) {
            red[2 * warp] = off;
            red[2 * warp + 1] = tot;
        }
        __syncthreads();
        if (tid == 0) {
            double o = 0.0, t = 0.0;
            for (int w = 0; w < kWarps; ++w) {
                o += red[2 * w];
                t += red[2 * w + 1];
            }
            stop = (o <= 1e-28 * t) || (o <= 1e-24 * t && o > 0.25 * prev_off);
            prev_off = o;
        }
        __syncthreads();
        if (stop) break;
    }
    const double* A = sm + cur * mat;
    for (int p = tid; p < np; p += kThreads) diag_out[p] = A[p * ld + p];
    if (tid == 0) {
        info[0] = rounds;
        info[1] = sweeps_done;
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
                                                             double* __restrict__ V) {
    const int np = n + (n & 1);
    const int k = np / 2;
    const int lane = threadIdx.x & 31;
    const int row = blockIdx.x * 4 + (threadIdx.x >> 5);
    const int rounds = info[0];
    const bool vlane = lane < k;
    double f = (row == 2 * lane) ? 1.0 : 0.0;      // position 2·lane
    double g = (row == 2 * lane + 1) ? 1.0 : 0.0;  // position 2·lane + 1
    // The log streams through shared memory in chunks of kChunk rounds
    // (cp.async, double-buffered, shared by the CTA's four rows) so the
    // loop-carried chain never waits on L2.
    constexpr int kChunk = 32;
    __shared__ __align__(16) double2 logbuf[2][kChunk * 32];
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
        const double2* cur = logbuf[ch & 1];
        const int nr = min(kChunk, rounds - ch * kChunk);
        for (int ri = 0; ri < nr; ++ri) {
            const double2 rr = vlane ? cur[ri * 32 + lane] : make_double2(1.0, 0.0);
            const double x = rr.x * f - rr.y * g;
            const double y = rr.y * f + rr.x * g;
            const double x_up = __shfl_up_sync(0xffffffffu, x, 1);
            const double y_dn = __shfl_down_sync(0xffffffffu, y, 1);
            const double y0 = __shfl_sync(0xffffffffu, y, 0);
            const double xk = __shfl_sync(0xffffffffu, x, k - 1);
            f = lane == 0 ? x : (lane == 1 ? y0 : x_up);
            g = lane == k - 1 ? xk : y_dn;
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

bool launch_sym_jacobi_pp(const double* C, int64_t ldc, int n, double* lambda, double* V, CallScratch& sc,
                          int* sweeps) {
    const int np = n + (n & 1);
    if (np > kMaxNp || np < 4) return false;
    const int k = np / 2;
    const size_t smem = sizeof(double) * (2 * static_cast<size_t>(np) * (np + 2) + 2 * k) + 16;
    static bool configured = false;
    if (!configured) {
        TS_CUDA_CHECK(cudaFuncSetAttribute(jacobi_values_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        configured = true;
    }
    auto* rot = sc.alloc_n<double2>(static_cast<size_t>(kMaxSweeps) * (np - 1) * k);
    double* dpos = sc.alloc_n<double>(static_cast<size_t>(np));
    int* info = sc.alloc_n<int>(2);
    jacobi_values_kernel<<<1, kThreads, smem, sc.stream()>>>(C, ldc, n, rot, dpos, info);
    TS_LAUNCH_CHECK();
    jacobi_vectors_kernel<<<(np + 3) / 4, 128, 0, sc.stream()>>>(n, rot, dpos, info, lambda, V);
    TS_LAUNCH_CHECK();
    if (sweeps) TS_CUDA_CHECK(cudaMemcpyAsync(sweeps, info + 1, sizeof(int), cudaMemcpyDeviceToDevice, sc.stream()));
    sc.launches += 2;
    return true;
}

}  // namespace ts

// Kept for the C ABI debug hook; the two-kernel solver has no phase probe.
extern "C" void tsi_read_eig_profile(long long* out) {
    for (int i = 0; i < 4; ++i) out[i] = 0;
}
