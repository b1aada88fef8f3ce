// kernels.cu — stage B (core × implicit Khatri-Rao), stage D (TSQR), stage G
// (one-sided Jacobi SVD, unfolding) kernels for sm_100a.
#include <algorithm>
#include <cfloat>
#include <cmath>

#include "kernels.cuh"

namespace ts {
namespace {

constexpr int kKrpThreads = 128;
constexpr int kKrpCT = 32;  // sketch columns per CTA (one per lane)
constexpr int kKrpJC = 32;  // complement-index chunk

// grid = (atoms, order, ceil(s / CT)).  Thread (ag = warp, c = lane) owns rows
// a ≡ ag (mod 4) of the RT-row output tile for sketch column c.
template <int RT>
__global__ void __launch_bounds__(kKrpThreads) krp_contract_kernel(KrpArgs args) {
    constexpr int RPT = RT / 4;
    const Atom& at = args.atoms[blockIdx.x];
    const int n = blockIdx.y;
    const int c0 = blockIdx.z * kKrpCT;
    const int order = args.order, s = args.s;
    const int tid = threadIdx.x, lane = tid & 31, ag = tid >> 5;

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

    extern __shared__ __align__(16) double sm[];
    int moff[kMaxOrder];
    int msum = 0;
    for (int j = 0; j < order; ++j) {
        moff[j] = msum;
        if (j != n) msum += shape[j] * kKrpCT;
    }
    double* Ms = sm;                                  // Σ_{j≠n} r_j × CT
    double* Ks = Ms + msum;                           // JC × CT
    double* Gs = Ks + kKrpJC * kKrpCT;                // RT × JC
    int64_t* Goff = reinterpret_cast<int64_t*>(Gs + RT * kKrpJC);  // JC
    int* Idx = reinterpret_cast<int*>(Goff + kKrpJC);              // JC × order

    for (int j = 0; j < order; ++j) {
        if (j == n) continue;
        const double* Z = args.Z[j];
        for (int idx = tid; idx < shape[j] * kKrpCT; idx += kKrpThreads) {
            const int a = idx / kKrpCT, c = idx % kKrpCT;
            const int cg = c0 + c;
            Ms[moff[j] + idx] = cg < s ? Z[cg + static_cast<int64_t>(col[j] + a) * s] : 0.0;
        }
    }
    const double w = args.weights[at.summand];
    const double* core = args.cores + at.core_off;
    double* Wn = args.W[n];
    const int64_t Rn = args.R[n];
    __syncthreads();

    for (int a0 = 0; a0 < rn; a0 += RT) {
        double acc[RPT];
#pragma unroll
        for (int i = 0; i < RPT; ++i) acc[i] = 0.0;
        for (int64_t J0 = 0; J0 < jtot; J0 += kKrpJC) {
            if (tid < kKrpJC) {
                const int64_t J = J0 + tid;
                int64_t off = -1;
                if (J < jtot) {
                    int64_t rem = J;
                    off = 0;
                    for (int j = 0; j < order; ++j) {
                        if (j == n) continue;
                        const int aj = static_cast<int>(rem % shape[j]);
                        rem /= shape[j];
                        off += aj * gstride[j];
                        Idx[tid * kMaxOrder + j] = aj;
                    }
                }
                Goff[tid] = off;
            }
            __syncthreads();
            for (int idx = tid; idx < kKrpJC * kKrpCT; idx += kKrpThreads) {
                const int jj = idx / kKrpCT, c = idx % kKrpCT;
                double v = 0.0;
                if (Goff[jj] >= 0) {
                    v = 1.0;
                    for (int j = 0; j < order; ++j) {
                        if (j == n) continue;
                        v *= Ms[moff[j] + Idx[jj * kMaxOrder + j] * kKrpCT + c];
                    }
                }
                Ks[idx] = v;
            }
            for (int idx = tid; idx < RT * kKrpJC; idx += kKrpThreads) {
                const int a = idx / kKrpJC, jj = idx % kKrpJC;
                const int64_t off = Goff[jj];
                Gs[idx] = (off >= 0 && a0 + a < rn) ? core[off + (a0 + a) * gstride[n]] : 0.0;
            }
            __syncthreads();
#pragma unroll 8
            for (int jj = 0; jj < kKrpJC; ++jj) {
                const double k = Ks[jj * kKrpCT + lane];
#pragma unroll
                for (int i = 0; i < RPT; ++i) acc[i] = fma(Gs[(ag + 4 * i) * kKrpJC + jj], k, acc[i]);
            }
            __syncthreads();
        }
        const int cg = c0 + lane;
        if (cg < s) {
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const int a = a0 + ag + 4 * i;
                if (a < rn) Wn[(col[n] + a) + static_cast<int64_t>(cg) * Rn] = w * acc[i];
            }
        }
    }
}

// ------------------------------------------------------------------ TSQR
constexpr int kQrThreads = 256;
constexpr int kQrWarps = kQrThreads / 32;

// Householder QR of one rows × cols block held column-major in shared memory.
// Reflector convention of Eigen's makeHouseholder (see oracle/tucksum_oracle.cpp).
__global__ void __launch_bounds__(kQrThreads) tsqr_factor_kernel(const QrTask* __restrict__ tasks) {
    const QrTask tk = tasks[blockIdx.x];
    const int rows = tk.rows, cols = tk.cols, kk = min(rows, cols);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    extern __shared__ __align__(16) double As[];
    __shared__ double sh_beta, sh_tau, sh_inv;
    for (int idx = tid; idx < rows * cols; idx += kQrThreads) {
        const int i = idx % rows, c = idx / rows;
        As[idx] = tk.A[i + c * tk.lda];
    }
    __syncthreads();
    for (int k = 0; k < kk; ++k) {
        double* x = As + k * rows;
        if (warp == 0) {
            double tail = 0.0;
            for (int i = k + 1 + lane; i < rows; i += 32) tail += x[i] * x[i];
            tail = warp_sum(tail);
            if (lane == 0) {
                const double c0 = x[k];
                if (tail <= DBL_MIN) {
                    sh_tau = 0.0;
                    sh_beta = c0;
                    sh_inv = 0.0;
                } else {
                    double beta = sqrt(c0 * c0 + tail);
                    if (c0 >= 0.0) beta = -beta;
                    sh_beta = beta;
                    sh_inv = 1.0 / (c0 - beta);
                    sh_tau = (beta - c0) / beta;
                }
            }
        }
        __syncthreads();
        const double tau = sh_tau, inv = sh_inv;
        for (int i = k + 1 + tid; i < rows; i += kQrThreads) x[i] = tau == 0.0 ? 0.0 : x[i] * inv;
        __syncthreads();
        if (tid == 0) {
            x[k] = sh_beta;
            tk.tau[k] = tau;
        }
        if (tau != 0.0) {
            for (int j = k + 1 + warp; j < cols; j += kQrWarps) {
                double* y = As + j * rows;
                double wsum = 0.0;
                for (int i = k + 1 + lane; i < rows; i += 32) wsum += x[i] * y[i];
                wsum = (warp_sum(wsum) + y[k]) * tau;
                for (int i = k + 1 + lane; i < rows; i += 32) y[i] -= wsum * x[i];
                __syncwarp();
                if (lane == 0) y[k] -= wsum;
            }
        }
        __syncthreads();
    }
    for (int idx = tid; idx < rows * cols; idx += kQrThreads) {
        const int i = idx % rows, c = idx / rows;
        tk.A[i + c * tk.lda] = As[idx];
    }
    for (int idx = tid; idx < kk * cols; idx += kQrThreads) {
        const int i = idx % kk, c = idx / kk;
        tk.R[i + c * tk.ldr] = i <= c ? As[i + c * rows] : 0.0;
    }
}

// Q formation for one block: Q = H_0 ⋯ H_{kk-1} · [Qin; 0], optional column signs.
__global__ void __launch_bounds__(kQrThreads) tsqr_apply_kernel(const QrApplyTask* __restrict__ tasks) {
    const QrApplyTask tk = tasks[blockIdx.x];
    const int rows = tk.rows, kk = tk.kk, q = tk.q;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    extern __shared__ __align__(16) double Qs[];
    double* v = Qs + rows * q;
    for (int idx = tid; idx < rows * q; idx += kQrThreads) {
        const int i = idx % rows, c = idx / rows;
        double val = 0.0;
        if (i < kk) val = tk.Qin ? tk.Qin[i + c * tk.ldqin] : (i == c ? 1.0 : 0.0);
        Qs[idx] = val;
    }
    __syncthreads();
    for (int k = kk - 1; k >= 0; --k) {
        const double tau = tk.tau[k];
        if (tau == 0.0) continue;
        for (int i = k + 1 + tid; i < rows; i += kQrThreads) v[i] = tk.V[i + k * tk.ldv];
        __syncthreads();
        for (int c = warp; c < q; c += kQrWarps) {
            double* y = Qs + c * rows;
            double wsum = 0.0;
            for (int i = k + 1 + lane; i < rows; i += 32) wsum += v[i] * y[i];
            wsum = (warp_sum(wsum) + y[k]) * tau;
            for (int i = k + 1 + lane; i < rows; i += 32) y[i] -= wsum * v[i];
            __syncwarp();
            if (lane == 0) y[k] -= wsum;
        }
        __syncthreads();
    }
    for (int idx = tid; idx < rows * q; idx += kQrThreads) {
        const int i = idx % rows, c = idx / rows;
        double val = Qs[idx];
        if (tk.Rsign && tk.Rsign[c + c * tk.ldrs] < 0.0) val = -val;
        tk.Q[i + c * tk.ldq] = val;
    }
}

// ------------------------------------------------------------------ Jacobi SVD
constexpr int kJacThreads = 256;
constexpr int kJacWarps = kJacThreads / 32;

__global__ void __launch_bounds__(kJacThreads) jacobi_svd_kernel(const double* __restrict__ R, int64_t ldr, int m,
                                                                 int nc, double* __restrict__ sigma,
                                                                 double* __restrict__ U) {
    extern __shared__ __align__(16) double sm[];
    double* W = sm;           // m × nc (ld m)
    double* J = W + m * nc;   // nc × nc (ld nc)
    double* nrm = J + nc * nc;  // nc
    __shared__ int rotated;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int idx = tid; idx < m * nc; idx += kJacThreads) {
        const int i = idx % m, c = idx / m;
        W[idx] = R[i + c * ldr];
    }
    for (int idx = tid; idx < nc * nc; idx += kJacThreads) J[idx] = (idx % nc == idx / nc) ? 1.0 : 0.0;
    const int np = nc + (nc & 1);  // players (one dummy when odd)
    const double tol = 1e-15;
    for (int sweep = 0; sweep < 80; ++sweep) {
        if (tid == 0) rotated = 0;
        __syncthreads();
        for (int r = 0; r < np - 1; ++r) {
            for (int pi = warp; pi < np / 2; pi += kJacWarps) {
                int p, q;
                if (pi == 0) {
                    p = np - 1;
                    q = r;
                } else {
                    p = (r + pi) % (np - 1);
                    q = (r - pi + (np - 1)) % (np - 1);
                }
                if (p >= nc || q >= nc) continue;
                if (p > q) {
                    const int tmp = p;
                    p = q;
                    q = tmp;
                }
                double* wp = W + p * m;
                double* wq = W + q * m;
                double al = 0.0, be = 0.0, ga = 0.0;
                for (int i = lane; i < m; i += 32) {
                    const double x = wp[i], y = wq[i];
                    al += x * x;
                    be += y * y;
                    ga += x * y;
                }
                al = warp_sum(al);
                be = warp_sum(be);
                ga = warp_sum(ga);
                if (ga == 0.0 || fabs(ga) <= tol * sqrt(al * be)) continue;
                const double zeta = (be - al) / (2.0 * ga);
                const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
                for (int i = lane; i < m; i += 32) {
                    const double x = wp[i], y = wq[i];
                    wp[i] = c * x - s * y;
                    wq[i] = s * x + c * y;
                }
                double* jp = J + p * nc;
                double* jq = J + q * nc;
                for (int i = lane; i < nc; i += 32) {
                    const double x = jp[i], y = jq[i];
                    jp[i] = c * x - s * y;
                    jq[i] = s * x + c * y;
                }
                if (lane == 0) rotated = 1;
            }
            __syncthreads();
        }
        if (!rotated) break;
        __syncthreads();
    }
    for (int c = warp; c < nc; c += kJacWarps) {
        double a = 0.0;
        for (int i = lane; i < m; i += 32) a += W[i + c * m] * W[i + c * m];
        a = warp_sum(a);
        if (lane == 0) nrm[c] = sqrt(a);
    }
    __syncthreads();
    // Stable descending order: rank = #{i : n_i > n_c or (n_i == n_c and i < c)}.
    for (int c = tid; c < nc; c += kJacThreads) {
        const double v = nrm[c];
        int rank = 0;
        for (int i = 0; i < nc; ++i) rank += (nrm[i] > v) || (nrm[i] == v && i < c);
        sigma[rank] = v;
        for (int i = 0; i < nc; ++i) U[i + static_cast<int64_t>(rank) * nc] = J[i + c * nc];
    }
}

// ------------------------------------------------------------------ misc
struct UnfoldArgs {
    int64_t shape[kMaxOrder];
    int order, mode;
};

__global__ void unfold_t_kernel(const double* __restrict__ g, UnfoldArgs a, double* __restrict__ X, int64_t total) {
    int64_t left = 1, right = 1;
    for (int j = 0; j < a.order; ++j) {
        if (j < a.mode) left *= a.shape[j];
        else if (j > a.mode) right *= a.shape[j];
    }
    const int64_t qk = a.shape[a.mode], rest = left * right;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t l = e % left;
        const int64_t i = (e / left) % qk;
        const int64_t r = e / (left * qk);
        X[(l + left * r) + i * rest] = g[e];
    }
}

__global__ void sumsq_kernel(const double* __restrict__ x, int64_t n, double* out) {
    __shared__ double part[32];
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += x[i] * x[i];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < blockDim.x / 32 ? part[threadIdx.x] : 0.0;
        v = warp_sum(v);
        if (threadIdx.x == 0) out[0] = v;
    }
}

__global__ void scale_columns_kernel(const double* __restrict__ F, int64_t n, int64_t R, const double* __restrict__ sc,
                                     double* __restrict__ out, bool transpose) {
    const int64_t total = n * R;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e % n, c = e / n;
        const double v = F[e] * sc[c];
        if (transpose) out[c + i * R] = v;
        else out[e] = v;
    }
}

int tsqr_block_rows(int64_t cols) {
    const int64_t cap = 20480 / std::max<int64_t>(cols, 1);  // 160 KB of fp64 per block
    return static_cast<int>(std::max<int64_t>(2 * cols, std::min<int64_t>(256, cap)));
}

}  // namespace

int max_tsqr_cols() { return 96; }

void launch_krp_contract(const KrpArgs& args, int max_shape, CallScratch& sc) {
    if (args.natoms == 0) return;
    int msum_max = 0;  // Σ_{j≠n} r_j ≤ Σ_j max r
    msum_max = max_shape * args.order;
    const int RT = max_shape <= 16 ? 16 : (max_shape <= 32 ? 32 : 64);
    const size_t smem = sizeof(double) * (static_cast<size_t>(msum_max) * kKrpCT + kKrpJC * kKrpCT + RT * kKrpJC) +
                        sizeof(int64_t) * kKrpJC + sizeof(int) * kKrpJC * kMaxOrder;
    dim3 grid(static_cast<unsigned>(args.natoms), static_cast<unsigned>(args.order),
              static_cast<unsigned>((args.s + kKrpCT - 1) / kKrpCT));
    auto go = [&](auto kern) {
        TS_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        kern<<<grid, kKrpThreads, smem, sc.stream()>>>(args);
        TS_LAUNCH_CHECK();
    };
    if (RT == 16) go(krp_contract_kernel<16>);
    else if (RT == 32) go(krp_contract_kernel<32>);
    else go(krp_contract_kernel<64>);
    sc.launches += 1;
}

TsqrPlan plan_tsqr(double* A, int64_t lda, int64_t rows, int64_t cols, double* Q, int64_t ldq, CallScratch& sc) {
    TsqrPlan plan;
    const int br = tsqr_block_rows(cols);
    double* cur = A;
    int64_t cur_ld = lda, cur_rows = rows;
    struct LevelInfo {
        double* A;
        int64_t ld, rows;
        std::vector<int64_t> row0, brows, roff;
        double* taus;
    };
    std::vector<LevelInfo> info;
    while (true) {
        LevelInfo li;
        li.A = cur;
        li.ld = cur_ld;
        li.rows = cur_rows;
        const int64_t nblk = cur_rows <= br ? 1 : (cur_rows + br - 1) / br;
        int64_t next_rows = 0;
        for (int64_t b = 0; b < nblk; ++b) {
            const int64_t r0 = b * br, rb = std::min<int64_t>(br, cur_rows - r0);
            li.row0.push_back(r0);
            li.brows.push_back(rb);
            li.roff.push_back(next_rows);
            next_rows += std::min<int64_t>(rb, cols);
        }
        li.taus = sc.alloc_n<double>(static_cast<size_t>(nblk * cols));
        double* Rbuf = sc.alloc_n<double>(static_cast<size_t>(std::max<int64_t>(next_rows, 1) * cols));
        std::vector<QrTask> tasks;
        for (int64_t b = 0; b < nblk; ++b) {
            QrTask t{};
            t.A = cur + li.row0[static_cast<size_t>(b)];
            t.lda = cur_ld;
            t.rows = static_cast<int>(li.brows[static_cast<size_t>(b)]);
            t.cols = static_cast<int>(cols);
            t.tau = li.taus + b * cols;
            t.R = Rbuf + li.roff[static_cast<size_t>(b)];
            t.ldr = next_rows;
            tasks.push_back(t);
        }
        plan.levels.push_back(std::move(tasks));
        info.push_back(li);
        if (nblk == 1) {
            plan.Rtop = Rbuf;
            plan.kk = next_rows;
            break;
        }
        cur = Rbuf;
        cur_ld = next_rows;
        cur_rows = next_rows;
    }
    if (Q != nullptr) {
        const int64_t q = std::min(rows, cols);
        // Top-down: level L's Q buffer (rows_L × q); level 0 writes into Q.
        std::vector<double*> qbuf(info.size());
        std::vector<int64_t> qld(info.size());
        for (size_t L = 0; L < info.size(); ++L) {
            if (L == 0) {
                qbuf[L] = Q;
                qld[L] = ldq;
            } else {
                qbuf[L] = sc.alloc_n<double>(static_cast<size_t>(info[L].rows * q));
                qld[L] = info[L].rows;
            }
        }
        for (size_t Li = info.size(); Li-- > 0;) {
            const LevelInfo& li = info[Li];
            std::vector<QrApplyTask> tasks;
            for (size_t b = 0; b < li.row0.size(); ++b) {
                QrApplyTask t{};
                t.V = li.A + li.row0[b];
                t.ldv = li.ld;
                t.tau = li.taus + static_cast<int64_t>(b) * cols;
                t.rows = static_cast<int>(li.brows[b]);
                t.kk = static_cast<int>(std::min<int64_t>(li.brows[b], cols));
                t.q = static_cast<int>(q);
                if (Li + 1 == info.size()) {
                    t.Qin = nullptr;
                    t.Rsign = plan.Rtop;
                    t.ldrs = plan.kk;
                } else {
                    t.Qin = qbuf[Li + 1] + li.roff[b];
                    t.ldqin = qld[Li + 1];
                    t.Rsign = nullptr;
                }
                t.Q = qbuf[Li] + li.row0[b];
                t.ldq = qld[Li];
                tasks.push_back(t);
            }
            plan.applies.push_back(std::move(tasks));
        }
    }
    return plan;
}

void run_tsqr(const std::vector<TsqrPlan*>& plans, CallScratch& sc, bool form_q) {
    size_t nlev = 0, napp = 0;
    for (auto* p : plans) {
        nlev = std::max(nlev, p->levels.size());
        napp = std::max(napp, p->applies.size());
    }
    static bool configured = false;
    if (!configured) {
        TS_CUDA_CHECK(cudaFuncSetAttribute(tsqr_factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        TS_CUDA_CHECK(cudaFuncSetAttribute(tsqr_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        configured = true;
    }
    for (size_t L = 0; L < nlev; ++L) {
        std::vector<QrTask> tasks;
        size_t smem = 0;
        for (auto* p : plans)
            if (L < p->levels.size())
                for (const QrTask& t : p->levels[L]) {
                    tasks.push_back(t);
                    smem = std::max(smem, sizeof(double) * static_cast<size_t>(t.rows) * t.cols);
                }
        if (tasks.empty()) continue;
        auto* d = static_cast<const QrTask*>(sc.upload(tasks.data(), tasks.size() * sizeof(QrTask)));
        tsqr_factor_kernel<<<static_cast<unsigned>(tasks.size()), kQrThreads, smem, sc.stream()>>>(d);
        TS_LAUNCH_CHECK();
        sc.launches += 1;
    }
    if (!form_q) return;
    // Apply levels are stored top-down per plan; align plans at their top level.
    for (size_t A = 0; A < napp; ++A) {
        std::vector<QrApplyTask> tasks;
        size_t smem = 0;
        for (auto* p : plans) {
            const size_t off = napp - p->applies.size();  // plans with fewer levels start later
            if (A < off) continue;
            for (const QrApplyTask& t : p->applies[A - off]) {
                tasks.push_back(t);
                smem = std::max(smem, sizeof(double) * static_cast<size_t>(t.rows) * (t.q + 1));
            }
        }
        if (tasks.empty()) continue;
        auto* d = static_cast<const QrApplyTask*>(sc.upload(tasks.data(), tasks.size() * sizeof(QrApplyTask)));
        tsqr_apply_kernel<<<static_cast<unsigned>(tasks.size()), kQrThreads, smem, sc.stream()>>>(d);
        TS_LAUNCH_CHECK();
        sc.launches += 1;
    }
}

void launch_jacobi_svd(const double* R, int64_t ldr, int m, int nc, double* sigma, double* U, CallScratch& sc) {
    const size_t smem = sizeof(double) * (static_cast<size_t>(m) * nc + static_cast<size_t>(nc) * nc + nc);
    static bool configured = false;
    if (!configured) {
        TS_CUDA_CHECK(cudaFuncSetAttribute(jacobi_svd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        configured = true;
    }
    jacobi_svd_kernel<<<1, kJacThreads, smem, sc.stream()>>>(R, ldr, m, nc, sigma, U);
    TS_LAUNCH_CHECK();
    sc.launches += 1;
}

void launch_unfold_t(const double* g, int order, const int64_t* shape, int mode, double* X, CallScratch& sc) {
    UnfoldArgs a{};
    int64_t total = 1;
    for (int j = 0; j < order; ++j) {
        a.shape[j] = shape[j];
        total *= shape[j];
    }
    a.order = order;
    a.mode = mode;
    const int threads = 256;
    const int64_t blocks = std::min<int64_t>((total + threads - 1) / threads, 2048);
    unfold_t_kernel<<<static_cast<unsigned>(std::max<int64_t>(blocks, 1)), threads, 0, sc.stream()>>>(g, a, X, total);
    TS_LAUNCH_CHECK();
    sc.launches += 1;
}

void launch_scale_columns(const double* F, int64_t n, int64_t R, const double* scale, double* out, bool transpose,
                          CallScratch& sc) {
    const int threads = 256;
    const int64_t blocks = std::min<int64_t>((n * R + threads - 1) / threads, 4096);
    scale_columns_kernel<<<static_cast<unsigned>(std::max<int64_t>(blocks, 1)), threads, 0, sc.stream()>>>(F, n, R, scale,
                                                                                                         out, transpose);
    TS_LAUNCH_CHECK();
    sc.launches += 1;
}

void launch_sumsq(const double* x, int64_t n, double* out, CallScratch& sc) {
    sumsq_kernel<<<1, 1024, 0, sc.stream()>>>(x, n, out);
    TS_LAUNCH_CHECK();
    sc.launches += 1;
}

}  // namespace ts
