// tucksum_oracle.cpp — TEST INFRASTRUCTURE ONLY.
//
// Eigen-free CPU restatement of the reference's KRP sketched Tucker summation
// (arXiv 2603.13532, `krp_sum` → `sketched_sum(krp=true)`), used as the parity
// checker for the CUDA path and as the CPU baseline in bench.py.  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
// may load this library; the product path (paper_2603_13532_b200) never does.
//
// The reference itself needs Eigen >= 3.4, which is absent from this image
// (SURVEY.md F4), so it cannot be compiled as oracle/_ref.  Every function below
// cites the reference file:line it restates (paths relative to
// /root/reference/proj).  Third-party arithmetic restated here:
//   * Eigen HouseholderQR (src/kernels.cpp:50-63) → unblocked Householder with
//     Eigen's makeHouseholder convention and the R_ii >= 0 sign fix.
//   * Eigen BDCSVD (src/kernels.cpp:65-68) → QR-preconditioned one-sided Jacobi.
//   * Eigen SelfAdjointEigenSolver (src/kernels.cpp:70-86) → cyclic Jacobi.
//   * libstdc++ <random> mt19937_64 + normal_distribution (src/kernels.cpp:88-101)
//     → the SAME libstdc++ implementation, so Ω is bit-identical.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace oracle {

using Index = std::int64_t;

// ---------------------------------------------------------------- storage
// Column-major matrix (reference include/tucksum/types.hpp:10).
struct Mat {
    Index r = 0, c = 0;
    std::vector<double> a;
    Mat() = default;
    Mat(Index rows, Index cols) : r(rows), c(cols), a(static_cast<size_t>(rows * cols), 0.0) {}
    double& operator()(Index i, Index j) { return a[static_cast<size_t>(i + j * r)]; }
    double operator()(Index i, Index j) const { return a[static_cast<size_t>(i + j * r)]; }
    double* col(Index j) { return a.data() + j * r; }
    const double* col(Index j) const { return a.data() + j * r; }
};

// Column-major N-d tensor, first index fastest (include/tucksum/dense_tensor.hpp:11-13).
struct Tensor {
    std::vector<Index> shape;
    std::vector<double> a;
    Tensor() = default;
    explicit Tensor(std::vector<Index> s) : shape(std::move(s)) {
        Index n = 1;
        for (Index d : shape) {
            if (d < 1) throw std::invalid_argument("DenseTensor: every dimension must be >= 1");
            n *= d;
        }
        if (shape.empty()) throw std::invalid_argument("DenseTensor: shape must have order >= 1");
        a.assign(static_cast<size_t>(n), 0.0);
    }
    Index order() const { return static_cast<Index>(shape.size()); }
    Index size() const { return static_cast<Index>(a.size()); }
    Index dim(Index k) const { return shape[static_cast<size_t>(k)]; }
};

struct Block {
    std::vector<Index> off;
    Tensor data;
};

// TuckerTensor with super-diagonal block core (include/tucksum/tucker.hpp:13-48).
struct Tucker {
    std::vector<Index> dims, ranks;
    std::vector<Mat> factors;
    std::vector<Block> blocks;
    Index order() const { return static_cast<Index>(ranks.size()); }
};

// src/tucker.cpp:16-55 validate_structure.
void validate_structure(const Tucker& x) {
    const size_t order = x.ranks.size();
    if (order == 0) throw std::invalid_argument("TuckerTensor: order must be >= 1");
    if (x.factors.size() != order || x.dims.size() != order)
        throw std::invalid_argument("TuckerTensor: one factor matrix per mode required");
    for (size_t k = 0; k < order; ++k) {
        if (x.factors[k].r != x.dims[k] || x.factors[k].c != x.ranks[k])
            throw std::invalid_argument("TuckerTensor: factor shape must be dims[k] x ranks[k]");
        if (x.dims[k] < 1 || x.ranks[k] < 1)
            throw std::invalid_argument("TuckerTensor: dims and ranks must be positive");
    }
    if (x.blocks.empty()) throw std::invalid_argument("TuckerTensor: core needs at least one block");
    std::vector<Index> cursor(order, 0);
    for (const auto& b : x.blocks) {
        if (b.off.size() != order || b.data.shape.size() != order)
            throw std::invalid_argument("TuckerTensor: block order mismatch");
        for (size_t k = 0; k < order; ++k) {
            if (b.off[k] != cursor[k])
                throw std::invalid_argument("TuckerTensor: blocks must tile the super-diagonal");
            cursor[k] += b.data.shape[k];
        }
    }
    for (size_t k = 0; k < order; ++k)
        if (cursor[k] != x.ranks[k])
            throw std::invalid_argument("TuckerTensor: blocks must span the full rank box");
}

Tucker make_dense_tucker(Tensor core, std::vector<Mat> factors) {
    Tucker t;
    for (auto& f : factors) t.dims.push_back(f.r);
    t.ranks = core.shape;
    t.factors = std::move(factors);
    Block b;
    b.off.assign(t.ranks.size(), 0);
    b.data = std::move(core);
    t.blocks.push_back(std::move(b));
    validate_structure(t);
    return t;
}

// ---------------------------------------------------------------- RNG
// src/kernels.cpp:14-19.
std::uint64_t splitmix64(std::uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

struct Seed {
    std::uint64_t seed = 0, stream = 0;
    // src/kernels.cpp:23-25.
    Seed substream(std::uint64_t salt) const { return Seed{seed, splitmix64(stream ^ splitmix64(salt))}; }
};

// src/kernels.cpp:88-101: mt19937_64 seeded from splitmix64 of (seed, stream),
// libstdc++ polar normal, filled column by column.
Mat gaussian_matrix(Index rows, Index cols, Seed s) {
    if (rows < 0 || cols < 0) throw std::invalid_argument("gaussian_matrix: negative extent");
    std::mt19937_64 engine(splitmix64(s.seed) ^ splitmix64(splitmix64(s.stream) + 0x6a09e667f3bcc909ULL));
    std::normal_distribution<double> normal(0.0, 1.0);
    Mat out(rows, cols);
    for (Index j = 0; j < cols; ++j)
        for (Index i = 0; i < rows; ++i) out(i, j) = normal(engine);
    return out;
}

// ---------------------------------------------------------------- dense kernels
// C(m×n) (+)= alpha · op(A) · op(B). Plain blocked loops; the reference uses Eigen GEMM.
void gemm(bool ta, bool tb, Index m, Index n, Index k, double alpha, const double* A, Index lda,
          const double* B, Index ldb, double beta, double* C, Index ldc) {
    for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < m; ++i) C[i + j * ldc] = beta == 0.0 ? 0.0 : beta * C[i + j * ldc];
    if (m == 0 || n == 0 || k == 0) return;
    if (!ta) {
        // C(:,j) += alpha * A(:,p) * op(B)(p,j); contiguous in A and C.
        const Index KB = 256;
        for (Index p0 = 0; p0 < k; p0 += KB) {
            const Index p1 = std::min(k, p0 + KB);
            for (Index j = 0; j < n; ++j) {
                double* c = C + j * ldc;
                for (Index p = p0; p < p1; ++p) {
                    const double b = alpha * (tb ? B[j + p * ldb] : B[p + j * ldb]);
                    const double* a = A + p * lda;
                    for (Index i = 0; i < m; ++i) c[i] += a[i] * b;
                }
            }
        }
    } else if (!tb) {
        // C(i,j) = alpha * dot(A(:,i), B(:,j)); 4x4 register blocks of dot products.
        Index i = 0;
        for (; i + 4 <= m; i += 4) {
            const double* a0 = A + (i + 0) * lda; const double* a1 = A + (i + 1) * lda;
            const double* a2 = A + (i + 2) * lda; const double* a3 = A + (i + 3) * lda;
            Index j = 0;
            for (; j + 4 <= n; j += 4) {
                const double* b0 = B + (j + 0) * ldb; const double* b1 = B + (j + 1) * ldb;
                const double* b2 = B + (j + 2) * ldb; const double* b3 = B + (j + 3) * ldb;
                double s[16] = {0};
                for (Index p = 0; p < k; ++p) {
                    const double x0 = a0[p], x1 = a1[p], x2 = a2[p], x3 = a3[p];
                    const double y0 = b0[p], y1 = b1[p], y2 = b2[p], y3 = b3[p];
                    s[0] += x0 * y0; s[1] += x1 * y0; s[2] += x2 * y0; s[3] += x3 * y0;
                    s[4] += x0 * y1; s[5] += x1 * y1; s[6] += x2 * y1; s[7] += x3 * y1;
                    s[8] += x0 * y2; s[9] += x1 * y2; s[10] += x2 * y2; s[11] += x3 * y2;
                    s[12] += x0 * y3; s[13] += x1 * y3; s[14] += x2 * y3; s[15] += x3 * y3;
                }
                for (int q = 0; q < 4; ++q)
                    for (int pp = 0; pp < 4; ++pp) C[(i + pp) + (j + q) * ldc] += alpha * s[q * 4 + pp];
            }
            for (; j < n; ++j) {
                const double* b0 = B + j * ldb;
                double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
                for (Index p = 0; p < k; ++p) {
                    s0 += a0[p] * b0[p]; s1 += a1[p] * b0[p]; s2 += a2[p] * b0[p]; s3 += a3[p] * b0[p];
                }
                C[i + j * ldc] += alpha * s0; C[i + 1 + j * ldc] += alpha * s1;
                C[i + 2 + j * ldc] += alpha * s2; C[i + 3 + j * ldc] += alpha * s3;
            }
        }
        for (; i < m; ++i) {
            const double* a0 = A + i * lda;
            for (Index j = 0; j < n; ++j) {
                const double* b0 = B + j * ldb;
                double s0 = 0;
                for (Index p = 0; p < k; ++p) s0 += a0[p] * b0[p];
                C[i + j * ldc] += alpha * s0;
            }
        }
    } else {
        for (Index j = 0; j < n; ++j)
            for (Index i = 0; i < m; ++i) {
                double s0 = 0;
                for (Index p = 0; p < k; ++p) s0 += A[p + i * lda] * B[j + p * ldb];
                C[i + j * ldc] += alpha * s0;
            }
    }
}

Mat matmul(const Mat& A, bool ta, const Mat& B, bool tb) {
    const Index m = ta ? A.c : A.r, k = ta ? A.r : A.c;
    const Index k2 = tb ? B.c : B.r, n = tb ? B.r : B.c;
    if (k != k2) throw std::invalid_argument("matmul: inner dimensions differ");
    Mat C(m, n);
    gemm(ta, tb, m, n, k, 1.0, A.a.data(), std::max<Index>(A.r, 1), B.a.data(), std::max<Index>(B.r, 1), 0.0,
         C.a.data(), std::max<Index>(m, 1));
    return C;
}

Mat middle_cols(const Mat& A, Index c0, Index nc) {
    Mat out(A.r, nc);
    std::memcpy(out.a.data(), A.a.data() + c0 * A.r, sizeof(double) * static_cast<size_t>(A.r * nc));
    return out;
}

Mat middle_rows(const Mat& A, Index r0, Index nr) {
    Mat out(nr, A.c);
    for (Index j = 0; j < A.c; ++j)
        for (Index i = 0; i < nr; ++i) out(i, j) = A(r0 + i, j);
    return out;
}

Mat transpose(const Mat& A) {
    Mat t(A.c, A.r);
    for (Index j = 0; j < A.c; ++j)
        for (Index i = 0; i < A.r; ++i) t(j, i) = A(i, j);
    return t;
}

// src/kernels.cpp:27-35.
Mat kron(const Mat& a, const Mat& b) {
    Mat out(a.r * b.r, a.c * b.c);
    for (Index j = 0; j < a.c; ++j)
        for (Index i = 0; i < a.r; ++i)
            for (Index l = 0; l < b.c; ++l)
                for (Index k = 0; k < b.r; ++k) out(i * b.r + k, j * b.c + l) = a(i, j) * b(k, l);
    return out;
}

// src/kernels.cpp:37-48: column c = kron(a(:,c), b(:,c)), b's rows fastest.
Mat khatri_rao(const Mat& a, const Mat& b) {
    if (a.c != b.c) throw std::invalid_argument("khatri_rao: operands must have equal column counts");
    Mat out(a.r * b.r, a.c);
    for (Index c = 0; c < a.c; ++c)
        for (Index i = 0; i < a.r; ++i)
            for (Index k = 0; k < b.r; ++k) out(i * b.r + k, c) = a(i, c) * b(k, c);
    return out;
}

// src/dense_tensor.cpp:125-134.
void split_extents(const std::vector<Index>& shape, Index mode, Index& left, Index& right) {
    left = 1;
    right = 1;
    for (Index k = 0; k < static_cast<Index>(shape.size()); ++k) {
        if (k < mode) left *= shape[static_cast<size_t>(k)];
        else if (k > mode) right *= shape[static_cast<size_t>(k)];
    }
}

// src/dense_tensor.cpp:145-164: column j = l + left*r holds t[l + i*left + r*left*nk].
Mat unfold(const Tensor& t, Index mode) {
    if (mode < 0 || mode >= t.order()) throw std::invalid_argument("unfold: mode out of range");
    const Index nk = t.dim(mode);
    Index left, right;
    split_extents(t.shape, mode, left, right);
    Mat out(nk, left * right);
    for (Index r = 0; r < right; ++r)
        for (Index i = 0; i < nk; ++i) {
            const double* blk = t.a.data() + (i + r * nk) * left;
            for (Index l = 0; l < left; ++l) out(i, l + left * r) = blk[l];
        }
    return out;
}

// src/dense_tensor.cpp:166-190.
Tensor fold(const Mat& m, Index mode, std::vector<Index> shape) {
    if (mode < 0 || mode >= static_cast<Index>(shape.size())) throw std::invalid_argument("fold: mode out of range");
    Index count = 1;
    for (Index n : shape) count *= n;
    const Index nk = shape[static_cast<size_t>(mode)];
    if (m.r != nk || m.r * m.c != count)
        throw std::invalid_argument("fold: matrix shape does not match target tensor shape");
    Index left, right;
    split_extents(shape, mode, left, right);
    Tensor t(std::move(shape));
    for (Index r = 0; r < right; ++r)
        for (Index i = 0; i < nk; ++i) {
            double* blk = t.a.data() + (i + r * nk) * left;
            for (Index l = 0; l < left; ++l) blk[l] = m(i, l + left * r);
        }
    return t;
}

// src/dense_tensor.cpp:192-210: mode-k unfolding of the result is a * unfold(t, k).
Tensor ttm(const Tensor& t, const Mat& a, Index mode) {
    if (mode < 0 || mode >= t.order()) throw std::invalid_argument("ttm: mode out of range");
    if (a.c != t.dim(mode))
        throw std::invalid_argument("ttm: matrix columns must match the contracted mode dimension");
    std::vector<Index> out_shape = t.shape;
    out_shape[static_cast<size_t>(mode)] = a.r;
    if (mode == 0) {
        Index left, right;
        split_extents(t.shape, 0, left, right);
        Tensor out(out_shape);
        gemm(false, false, a.r, right, t.dim(0), 1.0, a.a.data(), std::max<Index>(a.r, 1), t.a.data(), t.dim(0), 0.0,
             out.a.data(), a.r);
        return out;
    }
    Mat u = unfold(t, mode);
    return fold(matmul(a, false, u, false), mode, std::move(out_shape));
}

// ---------------------------------------------------------------- factorizations
struct Qr {
    Mat q, r;
};

// src/kernels.cpp:50-63 (Eigen HouseholderQR + explicit thin Q + R_ii >= 0 flip).
// Householder vectors follow Eigen's makeHouseholder: beta = -sign(c0)·‖x‖,
// tau = (beta - c0)/beta, v = [1; x_tail/(c0 - beta)]; tau = 0 when the tail
// is below the smallest normal double.
Qr qr_econ(const Mat& a_in) {
    Mat a = a_in;
    const Index m = a.r, n = a.c, kk = std::min(m, n);
    std::vector<double> tau(static_cast<size_t>(kk), 0.0);
    for (Index k = 0; k < kk; ++k) {
        double* x = a.col(k) + k;
        const Index len = m - k;
        const double c0 = x[0];
        double tail = 0.0;
        for (Index i = 1; i < len; ++i) tail += x[i] * x[i];
        double beta, t;
        if (tail <= std::numeric_limits<double>::min()) {
            t = 0.0;
            beta = c0;
            for (Index i = 1; i < len; ++i) x[i] = 0.0;
        } else {
            beta = std::sqrt(c0 * c0 + tail);
            if (c0 >= 0.0) beta = -beta;
            const double inv = 1.0 / (c0 - beta);
            for (Index i = 1; i < len; ++i) x[i] *= inv;
            t = (beta - c0) / beta;
        }
        x[0] = beta;
        tau[static_cast<size_t>(k)] = t;
        if (t == 0.0) continue;
        for (Index j = k + 1; j < n; ++j) {
            double* y = a.col(j) + k;
            double w = y[0];
            for (Index i = 1; i < len; ++i) w += x[i] * y[i];
            w *= t;
            y[0] -= w;
            for (Index i = 1; i < len; ++i) y[i] -= w * x[i];
        }
    }
    Qr out;
    out.r = Mat(kk, n);
    for (Index j = 0; j < n; ++j)
        for (Index i = 0; i <= std::min(j, kk - 1); ++i) out.r(i, j) = a(i, j);
    out.q = Mat(m, kk);
    for (Index j = 0; j < kk; ++j) out.q(j, j) = 1.0;
    for (Index k = kk - 1; k >= 0; --k) {
        const double t = tau[static_cast<size_t>(k)];
        if (t == 0.0) continue;
        const double* x = a.col(k) + k;
        const Index len = m - k;
        for (Index j = k; j < kk; ++j) {
            double* y = out.q.col(j) + k;
            double w = y[0];
            for (Index i = 1; i < len; ++i) w += x[i] * y[i];
            w *= t;
            y[0] -= w;
            for (Index i = 1; i < len; ++i) y[i] -= w * x[i];
        }
    }
    for (Index i = 0; i < kk; ++i) {
        if (out.r(i, i) < 0.0) {
            for (Index j = 0; j < n; ++j) out.r(i, j) = -out.r(i, j);
            for (Index p = 0; p < m; ++p) out.q(p, i) = -out.q(p, i);
        }
    }
    return out;
}

// One-sided (Hestenes) Jacobi on the columns of W (rows × n); accumulates the
// rotations into J (n × n). Columns of W end mutually orthogonal.
void one_sided_jacobi(Mat& W, Mat& J) {
    const Index n = W.c, rows = W.r;
    J = Mat(n, n);
    for (Index i = 0; i < n; ++i) J(i, i) = 1.0;
    const double tol = 1e-15;
    for (int sweep = 0; sweep < 80; ++sweep) {
        bool rotated = false;
        for (Index p = 0; p < n - 1; ++p)
            for (Index q = p + 1; q < n; ++q) {
                double alpha = 0, beta = 0, gamma = 0;
                const double* wp = W.col(p);
                const double* wq = W.col(q);
                for (Index i = 0; i < rows; ++i) {
                    alpha += wp[i] * wp[i];
                    beta += wq[i] * wq[i];
                    gamma += wp[i] * wq[i];
                }
                if (gamma == 0.0 || std::fabs(gamma) <= tol * std::sqrt(alpha * beta)) continue;
                rotated = true;
                const double zeta = (beta - alpha) / (2.0 * gamma);
                const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
                double* xp = W.col(p);
                double* xq = W.col(q);
                for (Index i = 0; i < rows; ++i) {
                    const double u = xp[i], v = xq[i];
                    xp[i] = c * u - s * v;
                    xq[i] = s * u + c * v;
                }
                double* jp = J.col(p);
                double* jq = J.col(q);
                for (Index i = 0; i < n; ++i) {
                    const double u = jp[i], v = jq[i];
                    jp[i] = c * u - s * v;
                    jq[i] = s * u + c * v;
                }
            }
        if (!rotated) break;
    }
}

struct Svd {
    Mat u;
    std::vector<double> s;  // descending
    Mat v;
};

// Completes columns [from, k) of U (m × k) to an orthonormal set (Gram–Schmidt on
// unit vectors), for singular vectors whose singular value is zero.
void complete_orthonormal(Mat& U, const std::vector<bool>& bad) {
    const Index m = U.r, k = U.c;
    Index probe = 0;
    for (Index j = 0; j < k; ++j) {
        if (!bad[static_cast<size_t>(j)]) continue;
        for (; probe < m; ++probe) {
            std::vector<double> v(static_cast<size_t>(m), 0.0);
            v[static_cast<size_t>(probe)] = 1.0;
            for (int pass = 0; pass < 2; ++pass)
                for (Index c = 0; c < k; ++c) {
                    if (c == j || (bad[static_cast<size_t>(c)] && c > j)) continue;
                    double d = 0;
                    for (Index i = 0; i < m; ++i) d += U(i, c) * v[static_cast<size_t>(i)];
                    for (Index i = 0; i < m; ++i) v[static_cast<size_t>(i)] -= d * U(i, c);
                }
            double nrm = 0;
            for (double x : v) nrm += x * x;
            nrm = std::sqrt(nrm);
            if (nrm > 0.5) {
                for (Index i = 0; i < m; ++i) U(i, j) = v[static_cast<size_t>(i)] / nrm;
                ++probe;
                break;
            }
        }
    }
}

// src/kernels.cpp:65-68 (thin SVD, any accurate method): a = u·diag(s)·vᵀ.
Svd svd_econ(const Mat& a) {
    const Index m = a.r, n = a.c;
    if (m < n) {
        Svd t = svd_econ(transpose(a));
        return Svd{std::move(t.v), std::move(t.s), std::move(t.u)};
    }
    // m >= n: a = Q R, R·J = W (orthogonal columns), a = (Q·W·Σ⁻¹)·Σ·Jᵀ.
    Qr qr = qr_econ(a);
    Mat W = qr.r;  // n × n
    Mat J;
    one_sided_jacobi(W, J);
    std::vector<double> sig(static_cast<size_t>(n));
    for (Index j = 0; j < n; ++j) {
        double s2 = 0;
        for (Index i = 0; i < n; ++i) s2 += W(i, j) * W(i, j);
        sig[static_cast<size_t>(j)] = std::sqrt(s2);
    }
    std::vector<Index> perm(static_cast<size_t>(n));
    std::iota(perm.begin(), perm.end(), Index(0));
    std::stable_sort(perm.begin(), perm.end(), [&](Index x, Index y) { return sig[static_cast<size_t>(x)] > sig[static_cast<size_t>(y)]; });
    Svd out;
    out.s.resize(static_cast<size_t>(n));
    Mat Ur(n, n);
    out.v = Mat(n, n);
    std::vector<bool> bad(static_cast<size_t>(n), false);
    const double smax = n > 0 ? sig[static_cast<size_t>(perm[0])] : 0.0;
    for (Index j = 0; j < n; ++j) {
        const Index p = perm[static_cast<size_t>(j)];
        const double sv = sig[static_cast<size_t>(p)];
        out.s[static_cast<size_t>(j)] = sv;
        for (Index i = 0; i < n; ++i) out.v(i, j) = J(i, p);
        if (sv > 0.0 && sv > 1e-300 && !(smax > 0 && sv < smax * 1e-300)) {
            for (Index i = 0; i < n; ++i) Ur(i, j) = W(i, p) / sv;
        } else {
            bad[static_cast<size_t>(j)] = true;
        }
    }
    complete_orthonormal(Ur, bad);
    out.u = matmul(qr.q, false, Ur, false);
    return out;
}

struct SymEig {
    std::vector<double> values;  // descending
    Mat vectors;
};

// src/kernels.cpp:70-86 (symmetrize, eigendecompose, descending): cyclic Jacobi.
SymEig sym_eig(const Mat& a_in) {
    if (a_in.r != a_in.c) throw std::invalid_argument("sym_eig: matrix must be square");
    const Index n = a_in.r;
    Mat a(n, n);
    for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < n; ++i) a(i, j) = 0.5 * (a_in(i, j) + a_in(j, i));
    Mat v(n, n);
    for (Index i = 0; i < n; ++i) v(i, i) = 1.0;
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0, diag = 0;
        for (Index j = 0; j < n; ++j)
            for (Index i = 0; i < n; ++i) (i == j ? diag : off) += a(i, j) * a(i, j);
        if (off <= 1e-32 * std::max(diag, std::numeric_limits<double>::min())) break;
        for (Index p = 0; p < n - 1; ++p)
            for (Index q = p + 1; q < n; ++q) {
                const double apq = a(p, q);
                if (apq == 0.0) continue;
                const double app = a(p, p), aqq = a(q, q);
                const double theta = (aqq - app) / (2.0 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(1.0 + theta * theta));
                const double c = 1.0 / std::sqrt(1.0 + t * t), s = t * c;
                for (Index k = 0; k < n; ++k) {  // columns p, q
                    const double akp = a(k, p), akq = a(k, q);
                    a(k, p) = c * akp - s * akq;
                    a(k, q) = s * akp + c * akq;
                }
                for (Index k = 0; k < n; ++k) {  // rows p, q
                    const double apk = a(p, k), aqk = a(q, k);
                    a(p, k) = c * apk - s * aqk;
                    a(q, k) = s * apk + c * aqk;
                }
                for (Index k = 0; k < n; ++k) {
                    const double vkp = v(k, p), vkq = v(k, q);
                    v(k, p) = c * vkp - s * vkq;
                    v(k, q) = s * vkp + c * vkq;
                }
            }
    }
    std::vector<Index> perm(static_cast<size_t>(n));
    std::iota(perm.begin(), perm.end(), Index(0));
    std::stable_sort(perm.begin(), perm.end(), [&](Index x, Index y) { return a(x, x) > a(y, y); });
    SymEig out;
    out.values.resize(static_cast<size_t>(n));
    out.vectors = Mat(n, n);
    for (Index j = 0; j < n; ++j) {
        const Index p = perm[static_cast<size_t>(j)];
        out.values[static_cast<size_t>(j)] = a(p, p);
        for (Index i = 0; i < n; ++i) out.vectors(i, j) = v(i, p);
    }
    return out;
}

// ---------------------------------------------------------------- Tucker algebra
// src/tucker.cpp:102-119.
Tensor reconstruct(const Tucker& x, Index max_elems = Index(1) << 27) {
    Index count = 1;
    for (Index n : x.dims) count *= n;
    if (count > max_elems) throw std::runtime_error("reconstruct: dense size exceeds the cap");
    Tensor acc(x.dims);
    for (const auto& b : x.blocks) {
        Tensor tmp = b.data;
        for (Index k = 0; k < x.order(); ++k)
            tmp = ttm(tmp, middle_cols(x.factors[static_cast<size_t>(k)], b.off[static_cast<size_t>(k)], b.data.dim(k)), k);
        for (size_t i = 0; i < acc.a.size(); ++i) acc.a[i] += tmp.a[i];
    }
    return acc;
}

struct Orthogonalized {
    std::vector<Mat> q;
    Tensor core;
};

// src/tucker.cpp:132-155.
Orthogonalized orthogonalize(const Tucker& x) {
    const Index order = x.order();
    Orthogonalized out;
    out.q.resize(static_cast<size_t>(order));
    std::vector<Mat> r(static_cast<size_t>(order));
    std::vector<Index> qshape(static_cast<size_t>(order));
    for (Index k = 0; k < order; ++k) {
        Qr f = qr_econ(x.factors[static_cast<size_t>(k)]);
        out.q[static_cast<size_t>(k)] = std::move(f.q);
        r[static_cast<size_t>(k)] = std::move(f.r);
        qshape[static_cast<size_t>(k)] = r[static_cast<size_t>(k)].r;
    }
    out.core = Tensor(qshape);
    for (const auto& b : x.blocks) {
        Tensor tmp = b.data;
        for (Index k = 0; k < order; ++k)
            tmp = ttm(tmp, middle_cols(r[static_cast<size_t>(k)], b.off[static_cast<size_t>(k)], b.data.dim(k)), k);
        for (size_t i = 0; i < out.core.a.size(); ++i) out.core.a[i] += tmp.a[i];
    }
    return out;
}

double norm2(const std::vector<double>& v) {
    double s = 0;
    for (double x : v) s += x * x;
    return std::sqrt(s);
}

// src/tucker.cpp:159.
double tucker_norm(const Tucker& x) { return norm2(orthogonalize(x).core.a); }

// src/tucker.cpp:161-181.
double tucker_inner(const Tucker& x, const Tucker& y) {
    if (x.dims != y.dims) throw std::invalid_argument("tucker_inner: operands must share dims");
    const Index order = x.order();
    double acc = 0.0;
    for (const auto& bx : x.blocks)
        for (const auto& by : y.blocks) {
            Tensor tmp = by.data;
            for (Index k = 0; k < order; ++k) {
                const size_t ku = static_cast<size_t>(k);
                Mat w = matmul(middle_cols(x.factors[ku], bx.off[ku], bx.data.dim(k)), true,
                               middle_cols(y.factors[ku], by.off[ku], by.data.dim(k)), false);
                tmp = ttm(tmp, w, k);
            }
            double d = 0;
            for (size_t i = 0; i < tmp.a.size(); ++i) d += bx.data.a[i] * tmp.a[i];
            acc += d;
        }
    return acc;
}

// src/tucker.cpp:183-226.
Tucker formal_sum(const std::vector<const Tucker*>& xs, const std::vector<double>& weights) {
    if (xs.empty() || xs.size() != weights.size())
        throw std::invalid_argument("formal_sum: need matching, nonempty summands and weights");
    for (const Tucker* x : xs)
        if (x == nullptr) throw std::invalid_argument("formal_sum: null summand");
    const Index order = xs.front()->order();
    const auto& dims = xs.front()->dims;
    for (const Tucker* x : xs)
        if (x->dims != dims) throw std::invalid_argument("formal_sum: all summands must share dims");
    const size_t ou = static_cast<size_t>(order);
    Tucker out;
    out.dims = dims;
    out.ranks.assign(ou, 0);
    for (const Tucker* x : xs)
        for (size_t k = 0; k < ou; ++k) out.ranks[k] += x->ranks[k];
    out.factors.resize(ou);
    for (size_t k = 0; k < ou; ++k) {
        out.factors[k] = Mat(dims[k], out.ranks[k]);
        Index col = 0;
        for (const Tucker* x : xs) {
            std::memcpy(out.factors[k].col(col), x->factors[k].a.data(), sizeof(double) * x->factors[k].a.size());
            col += x->ranks[k];
        }
    }
    std::vector<Index> shift(ou, 0);
    for (size_t i = 0; i < xs.size(); ++i) {
        for (const auto& b : xs[i]->blocks) {
            Block nb;
            nb.off.resize(ou);
            for (size_t k = 0; k < ou; ++k) nb.off[k] = shift[k] + b.off[k];
            nb.data = b.data;
            for (double& v : nb.data.a) v *= weights[i];
            out.blocks.push_back(std::move(nb));
        }
        for (size_t k = 0; k < ou; ++k) shift[k] += xs[i]->ranks[k];
    }
    validate_structure(out);
    return out;
}

// src/tucker.cpp:298-303.
double tucker_rel_error(const Tucker& x, const Tucker& ref) {
    const double denom = tucker_norm(ref);
    const double diff = tucker_norm(formal_sum({&x, &ref}, {1.0, -1.0}));
    if (denom == 0.0) return diff;
    return diff / denom;
}

struct StHosvd {
    Tensor core;
    std::vector<Mat> factors;
};

// src/tucker.cpp:239-283, plus the optional per-mode rank cap of SURVEY.md §8(d)
// (rank = min(rank_rule, cap[k]) when cap is given; cap == nullptr ≡ reference).
StHosvd st_hosvd(Tensor g, double tau, const Index* cap) {
    if (tau < 0.0) throw std::invalid_argument("st_hosvd: tolerance must be nonnegative");
    const Index order = g.order();
    double sq = 0;
    for (double v : g.a) sq += v * v;
    const double theta = tau * tau * sq / static_cast<double>(order);
    std::vector<Index> mode_order(static_cast<size_t>(order));
    std::iota(mode_order.begin(), mode_order.end(), Index(0));
    std::stable_sort(mode_order.begin(), mode_order.end(), [&](Index a, Index b) { return g.dim(a) < g.dim(b); });
    StHosvd out;
    out.factors.resize(static_cast<size_t>(order));
    for (Index k : mode_order) {
        Svd svd = svd_econ(unfold(g, k));
        const std::vector<double>& s = svd.s;
        const Index count = static_cast<Index>(s.size());
        Index rank = 1;
        if (tau == 0.0) {
            const double floor = 1e-14 * s[0];
            rank = count;
            while (rank > 1 && s[static_cast<size_t>(rank - 1)] <= floor) --rank;
        } else {
            std::vector<double> suffix(static_cast<size_t>(count) + 1, 0.0);
            for (Index j = count - 1; j >= 0; --j)
                suffix[static_cast<size_t>(j)] = suffix[static_cast<size_t>(j) + 1] + s[static_cast<size_t>(j)] * s[static_cast<size_t>(j)];
            rank = count;
            for (Index r = 1; r <= count; ++r)
                if (suffix[static_cast<size_t>(r)] <= theta) {
                    rank = r;
                    break;
                }
        }
        if (cap != nullptr && cap[k] > 0) rank = std::min(rank, cap[k]);
        Mat p = middle_cols(svd.u, 0, rank);
        g = ttm(g, transpose(p), k);
        out.factors[static_cast<size_t>(k)] = std::move(p);
    }
    out.core = std::move(g);
    return out;
}

// src/tucker.cpp:285-296 (Lazy rounding), plus the optional rank cap.
Tucker tucker_rounding(const Tucker& x, double tau, const Index* cap) {
    if (tau < 0.0) throw std::invalid_argument("tucker_rounding: tolerance must be nonnegative");
    Orthogonalized o = orthogonalize(x);
    StHosvd st = st_hosvd(std::move(o.core), tau, cap);
    std::vector<Mat> factors(static_cast<size_t>(x.order()));
    for (size_t k = 0; k < factors.size(); ++k) factors[k] = matmul(o.q[k], false, st.factors[k], false);
    return make_dense_tucker(std::move(st.core), std::move(factors));
}

void validate_request(const std::vector<const Tucker*>& xs, const std::vector<double>& ws) {
    // src/sketch.cpp:16-30.
    if (xs.empty() || xs.size() != ws.size())
        throw std::invalid_argument("sum request needs matching, nonempty summands and weights");
    for (const Tucker* x : xs)
        if (x == nullptr) throw std::invalid_argument("sum request holds a null summand");
    const auto& dims = xs.front()->dims;
    for (const Tucker* x : xs)
        if (x->dims != dims) throw std::invalid_argument("sum request summands must share dims");
}

struct SumIntermediates {
    std::vector<Mat> omega, y, uhat;
    Tensor h;
};

// Partial range-finder accumulation over summands [i0, i1): src/sketch.cpp:103-143.
// krp: one Khatri-Rao contraction per (block, mode); otherwise (Kron) the block
// is multiplied by m[j] = Ω_jᵀU_j in every mode j ≠ n (:132-140) and its mode-n
// unfolding has Π_{j≠n} s_j columns.
void accumulate_sketch(const std::vector<const Tucker*>& xs, const std::vector<double>& ws, size_t i0, size_t i1,
                       const std::vector<Mat>& omega, std::vector<Mat>& y, bool krp = true) {
    for (size_t i = i0; i < i1; ++i) {
        const Tucker& x = *xs[i];
        const double w = ws[i];
        const Index order = x.order();
        const size_t ou = static_cast<size_t>(order);
        std::vector<Mat> m(ou);
        for (size_t j = 0; j < ou; ++j)  // :108-112
            m[j] = krp ? matmul(x.factors[j], true, omega[j], false) : matmul(omega[j], true, x.factors[j], false);
        for (Index n = 0; n < order; ++n) {
            const size_t nu = static_cast<size_t>(n);
            for (const Block& b : x.blocks) {
                Mat v;
                if (krp) {
                    Mat k;
                    bool first = true;
                    for (Index j = order - 1; j >= 0; --j) {  // :117-129, highest mode outermost
                        if (j == n) continue;
                        const size_t ju = static_cast<size_t>(j);
                        Mat slice = middle_rows(m[ju], b.off[ju], b.data.dim(j));
                        k = first ? std::move(slice) : khatri_rao(k, slice);
                        first = false;
                    }
                    v = matmul(unfold(b.data, n), false, k, false);  // :130
                } else {
                    Tensor t = b.data;  // :133-139
                    for (Index j = 0; j < order; ++j) {
                        if (j == n) continue;
                        const size_t ju = static_cast<size_t>(j);
                        t = ttm(t, middle_cols(m[ju], b.off[ju], b.data.dim(j)), j);
                    }
                    v = unfold(t, n);
                }
                Mat fs = middle_cols(x.factors[nu], b.off[nu], b.data.dim(n));
                // :131 / :140 y[n] += w * (factor_slice * v)
                gemm(false, false, fs.r, v.c, fs.c, w, fs.a.data(), fs.r, v.a.data(), v.r, 1.0, y[nu].a.data(), y[nu].r);
            }
        }
    }
}

// Partial core projection over summands [i0, i1): src/sketch.cpp:152-169.
void accumulate_core(const std::vector<const Tucker*>& xs, const std::vector<double>& ws, size_t i0, size_t i1,
                     const std::vector<Mat>& uhat, Tensor& h) {
    for (size_t i = i0; i < i1; ++i) {
        const Tucker& x = *xs[i];
        const size_t ou = x.ranks.size();
        std::vector<Mat> proj(ou);
        for (size_t n = 0; n < ou; ++n) proj[n] = matmul(uhat[n], true, x.factors[n], false);
        for (const Block& b : x.blocks) {
            Tensor v = b.data;
            for (size_t n = 0; n < ou; ++n)
                v = ttm(v, middle_cols(proj[n], b.off[n], b.data.dim(static_cast<Index>(n))), static_cast<Index>(n));
            for (size_t e = 0; e < h.a.size(); ++e) h.a[e] += ws[i] * v.a[e];
        }
    }
}

// Runs fn(i0, i1, slot) over `parts` contiguous summand ranges, then the caller
// reduces slots in index order (SPEC.md:313-314 index-ordered parallel reduction).
template <class F>
void for_ranges(size_t count, int parts, F fn) {
#pragma omp parallel for schedule(static, 1) num_threads(parts) if (parts > 1)
    for (int p = 0; p < parts; ++p) {
        const size_t i0 = count * static_cast<size_t>(p) / static_cast<size_t>(parts);
        const size_t i1 = count * static_cast<size_t>(p + 1) / static_cast<size_t>(parts);
        fn(i0, i1, p);
    }
}

// Π_{j≠skip} v_j, saturating (src/sketch.cpp complement_product).
Index complement_product(const std::vector<Index>& v, size_t skip) {
    const Index cap = Index(1) << 50;
    Index prod = 1;
    for (size_t j = 0; j < v.size(); ++j) {
        if (j == skip) continue;
        const Index f = std::max<Index>(v[j], 1);
        if (prod > cap / f) return cap;
        prod *= f;
    }
    return prod;
}

// src/sketch.cpp:66-181 with the plan passed in (mode_sketch_dims = widths);
// krp = true: uniform width s = max widths; krp = false (Kron): Ω_n is
// n_n × widths[n] and Y_n has Π_{j≠n} widths[j] columns.  `cap` is the optional
// rank cap (nullptr ≡ reference semantics).
Tucker sketched_sum(const std::vector<const Tucker*>& xs, const std::vector<double>& ws, const std::vector<Index>& widths,
                    Seed seed, double eps, const Index* cap, int threads, SumIntermediates* inter, bool krp) {
    validate_request(xs, ws);
    if (eps < 0.0) throw std::invalid_argument("tolerance must be nonnegative");
    const Index order = xs.front()->order();
    if (order < 2) throw std::invalid_argument("sketched summation needs order >= 2");
    const auto& dims = xs.front()->dims;
    const size_t ou = static_cast<size_t>(order);
    if (widths.size() != ou) throw std::invalid_argument("plan order does not match summand order");
    for (Index s : widths)
        if (s < 1) throw std::invalid_argument("plan sketch widths must be positive");
    const Index s = *std::max_element(widths.begin(), widths.end());
    std::vector<Mat> omega(ou);
    for (size_t n = 0; n < ou; ++n)  // :91-95
        omega[n] = gaussian_matrix(dims[n], krp ? s : widths[n], seed.substream(n));

    const int parts = std::max(1, std::min<int>(threads, static_cast<int>(xs.size())));
    std::vector<std::vector<Mat>> ys(static_cast<size_t>(parts));
    for (auto& yp : ys) {
        yp.resize(ou);
        for (size_t n = 0; n < ou; ++n) yp[n] = Mat(dims[n], krp ? s : complement_product(widths, n));  // :97-101
    }
    for_ranges(xs.size(), parts, [&](size_t i0, size_t i1, int p) {
        accumulate_sketch(xs, ws, i0, i1, omega, ys[static_cast<size_t>(p)], krp);
    });
    std::vector<Mat> y = std::move(ys[0]);
    for (int p = 1; p < parts; ++p)
        for (size_t n = 0; n < ou; ++n)
            for (size_t e = 0; e < y[n].a.size(); ++e) y[n].a[e] += ys[static_cast<size_t>(p)][n].a[e];

    std::vector<Mat> uhat(ou);
    std::vector<Index> qdims(ou);
    for (size_t n = 0; n < ou; ++n) {  // :145-150
        uhat[n] = qr_econ(y[n]).q;
        qdims[n] = uhat[n].c;
    }
    std::vector<Tensor> hs(static_cast<size_t>(parts));
    for (auto& hp : hs) hp = Tensor(qdims);
    for_ranges(xs.size(), parts, [&](size_t i0, size_t i1, int p) { accumulate_core(xs, ws, i0, i1, uhat, hs[static_cast<size_t>(p)]); });
    Tensor h = std::move(hs[0]);
    for (int p = 1; p < parts; ++p)
        for (size_t e = 0; e < h.a.size(); ++e) h.a[e] += hs[static_cast<size_t>(p)].a[e];
    if (inter != nullptr) {
        inter->omega = omega;
        inter->y = y;
        inter->uhat = uhat;
        inter->h = h;
    }
    StHosvd fin = st_hosvd(std::move(h), eps, cap);  // :171
    std::vector<Mat> out_factors(ou);
    for (size_t n = 0; n < ou; ++n) out_factors[n] = matmul(uhat[n], false, fin.factors[n], false);  // :172-175
    return make_dense_tucker(std::move(fin.core), std::move(out_factors));
}

Tucker krp_sum(const std::vector<const Tucker*>& xs, const std::vector<double>& ws, const std::vector<Index>& widths,
               Seed seed, double eps, const Index* cap, int threads, SumIntermediates* inter) {
    return sketched_sum(xs, ws, widths, seed, eps, cap, threads, inter, true);
}

// src/sketch.cpp:222-270: balanced Kron widths, then the deterministic repair.
std::vector<Index> kron_sketch_dims(const std::vector<Index>& targets, const std::vector<Index>& dims) {
    const size_t n = targets.size();
    if (n < 2 || n != dims.size())
        throw std::invalid_argument("kron_sketch_dims: need order >= 2 and matching dims");
    for (size_t i = 0; i < n; ++i) {
        if (targets[i] < 1 || dims[i] < 1)
            throw std::invalid_argument("kron_sketch_dims: targets and dims must be positive");
        if (targets[i] > complement_product(dims, i))
            throw std::invalid_argument("kron_sketch_dims: target exceeds attainable mode rank");
    }
    long double logp = 0.0L;
    for (Index t : targets) logp += std::log(static_cast<long double>(t));
    const long double root = std::exp(logp / static_cast<long double>(n - 1));
    std::vector<Index> s(n);
    for (size_t i = 0; i < n; ++i) {
        long double q = root / static_cast<long double>(targets[i]);
        const long double snapped = std::round(q);
        if (snapped >= 1.0L && std::fabs(q - snapped) < 1e-9L) q = snapped;
        const auto si = static_cast<Index>(std::ceil(static_cast<double>(q)));
        s[i] = std::clamp<Index>(si, 1, dims[i]);
    }
    bool changed = true;
    while (changed) {
        changed = false;
        for (size_t m = 0; m < n; ++m) {
            while (complement_product(s, m) < targets[m]) {
                size_t pick = n;
                for (size_t j = 0; j < n; ++j) {
                    if (j == m || s[j] >= dims[j]) continue;
                    if (pick == n || s[j] < s[pick]) pick = j;
                }
                if (pick == n) throw std::logic_error("kron_sketch_dims: infeasible despite capped targets");
                ++s[pick];
                changed = true;
            }
        }
    }
    return s;
}

// src/sketch.cpp:272-349 (krp widths: uniform max target; kron: kron_sketch_dims).
std::vector<Index> effective_subrank(const std::vector<const Tucker*>& xs, const std::vector<double>& ws, double eps,
                                     const std::vector<Index>& oversampling, std::vector<Index>* eff_out,
                                     std::vector<Index>* targets_out, bool krp = true) {
    validate_request(xs, ws);
    if (eps < 0.0) throw std::invalid_argument("tolerance must be nonnegative");
    const Index order = xs.front()->order();
    const auto& dims = xs.front()->dims;
    const size_t ou = static_cast<size_t>(order);
    if (oversampling.size() != ou) throw std::invalid_argument("oversampling vector must have one entry per mode");
    for (Index p : oversampling)
        if (p < 0) throw std::invalid_argument("oversampling must be nonnegative");
    std::vector<double> energy(xs.size());
    for (size_t i = 0; i < xs.size(); ++i) {
        double sq = 0;
        for (const auto& b : xs[i]->blocks)
            for (double v : b.data.a) sq += v * v;
        energy[i] = std::fabs(ws[i]) * std::sqrt(sq);
    }
    std::vector<Index> eff(ou), targets(ou);
    for (size_t n = 0; n < ou; ++n) {
        Index total = 0;
        for (const Tucker* x : xs) total += x->ranks[n];
        Mat v(dims[n], total);
        Index col = 0;
        for (size_t i = 0; i < xs.size(); ++i) {
            const Mat& f = xs[i]->factors[n];
            for (size_t e = 0; e < f.a.size(); ++e) v.a[static_cast<size_t>(col * dims[n]) + e] = energy[i] * f.a[e];
            col += xs[i]->ranks[n];
        }
        SymEig eig = sym_eig(matmul(v, true, v, false));
        std::vector<double> lam = eig.values;
        for (double& l : lam) l = std::max(l, 0.0);
        const double lmax = lam.empty() ? 0.0 : lam[0];
        const double floor = static_cast<double>(total) * std::numeric_limits<double>::epsilon() * lmax;
        for (double& l : lam)
            if (l < floor) l = 0.0;
        const Index count = static_cast<Index>(lam.size());
        std::vector<double> suffix(static_cast<size_t>(count) + 1, 0.0);
        for (Index j = count - 1; j >= 0; --j) suffix[static_cast<size_t>(j)] = suffix[static_cast<size_t>(j) + 1] + lam[static_cast<size_t>(j)];
        const double thresh = eps * eps / static_cast<double>(order) * suffix[0];
        Index keep = count;
        for (Index r = 1; r <= count; ++r)
            if (suffix[static_cast<size_t>(r)] <= thresh) {
                keep = r;
                break;
            }
        eff[n] = keep;
        Index target = keep + oversampling[n];
        target = std::min({target, dims[n], complement_product(dims, n)});
        targets[n] = std::max<Index>(target, 1);
    }
    if (eff_out) *eff_out = eff;
    if (targets_out) *targets_out = targets;
    if (!krp) return kron_sketch_dims(targets, dims);  // :340-341
    const Index smax = *std::max_element(targets.begin(), targets.end());
    return std::vector<Index>(ou, smax);
}

}  // namespace oracle

// ====================================================================== C ABI
// Flat, ctypes-friendly entry points for tests/ and bench.py.
namespace {

thread_local std::string g_err;

struct OrTuckerView {
    std::int64_t order;
    const std::int64_t* dims;          // [order]
    const std::int64_t* ranks;         // [order]
    const double* const* factors;      // [order], column-major dims[k] × ranks[k]
    std::int64_t num_blocks;
    const std::int64_t* block_offsets; // [num_blocks * order]
    const std::int64_t* block_shapes;  // [num_blocks * order]
    const double* const* block_data;   // [num_blocks], column-major
};

oracle::Tucker from_view(const OrTuckerView& v) {
    oracle::Tucker t;
    const size_t o = static_cast<size_t>(v.order);
    if (v.order < 1 || v.order > 32) throw std::invalid_argument("TuckerTensor: order must be >= 1");
    t.dims.assign(v.dims, v.dims + o);
    t.ranks.assign(v.ranks, v.ranks + o);
    for (size_t k = 0; k < o; ++k) {
        oracle::Mat f(t.dims[k], t.ranks[k]);
        if (!f.a.empty()) std::memcpy(f.a.data(), v.factors[k], sizeof(double) * f.a.size());
        t.factors.push_back(std::move(f));
    }
    for (std::int64_t b = 0; b < v.num_blocks; ++b) {
        oracle::Block blk;
        blk.off.assign(v.block_offsets + b * v.order, v.block_offsets + (b + 1) * v.order);
        blk.data = oracle::Tensor(std::vector<std::int64_t>(v.block_shapes + b * v.order, v.block_shapes + (b + 1) * v.order));
        std::memcpy(blk.data.a.data(), v.block_data[b], sizeof(double) * blk.data.a.size());
        t.blocks.push_back(std::move(blk));
    }
    oracle::validate_structure(t);
    return t;
}

struct OrResult {
    oracle::Tucker t;
    oracle::SumIntermediates inter;
    std::vector<std::int64_t> widths, eff, targets;
};

template <class F>
int guarded(F fn) {
    try {
        fn();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

std::vector<oracle::Tucker> views_to_tuckers(const OrTuckerView* views, std::int64_t count) {
    std::vector<oracle::Tucker> xs;
    xs.reserve(static_cast<size_t>(std::max<std::int64_t>(count, 0)));
    for (std::int64_t i = 0; i < count; ++i) xs.push_back(from_view(views[i]));
    return xs;
}

}  // namespace

extern "C" {

const char* or_last_error() { return g_err.c_str(); }

void or_substream(std::uint64_t seed, std::uint64_t stream, std::uint64_t salt, std::uint64_t* out_seed,
                  std::uint64_t* out_stream) {
    const oracle::Seed s = oracle::Seed{seed, stream}.substream(salt);
    *out_seed = s.seed;
    *out_stream = s.stream;
}

int or_gaussian_matrix(std::int64_t rows, std::int64_t cols, std::uint64_t seed, std::uint64_t stream, double* out) {
    return guarded([&] {
        oracle::Mat m = oracle::gaussian_matrix(rows, cols, oracle::Seed{seed, stream});
        std::memcpy(out, m.a.data(), sizeof(double) * m.a.size());
    });
}

int or_unfold(std::int64_t order, const std::int64_t* shape, const double* data, std::int64_t mode, double* out) {
    return guarded([&] {
        oracle::Tensor t(std::vector<std::int64_t>(shape, shape + order));
        std::memcpy(t.a.data(), data, sizeof(double) * t.a.size());
        oracle::Mat m = oracle::unfold(t, mode);
        std::memcpy(out, m.a.data(), sizeof(double) * m.a.size());
    });
}

int or_fold(std::int64_t order, const std::int64_t* shape, const double* mat, std::int64_t mode, double* out) {
    return guarded([&] {
        std::vector<std::int64_t> sh(shape, shape + order);
        std::int64_t count = 1;
        for (auto v : sh) count *= v;
        oracle::Mat m(sh[static_cast<size_t>(mode)], count / sh[static_cast<size_t>(mode)]);
        std::memcpy(m.a.data(), mat, sizeof(double) * m.a.size());
        oracle::Tensor t = oracle::fold(m, mode, sh);
        std::memcpy(out, t.a.data(), sizeof(double) * t.a.size());
    });
}

int or_ttm(std::int64_t order, const std::int64_t* shape, const double* data, const double* a, std::int64_t a_rows,
           std::int64_t a_cols, std::int64_t mode, double* out) {
    return guarded([&] {
        oracle::Tensor t(std::vector<std::int64_t>(shape, shape + order));
        std::memcpy(t.a.data(), data, sizeof(double) * t.a.size());
        oracle::Mat m(a_rows, a_cols);
        std::memcpy(m.a.data(), a, sizeof(double) * m.a.size());
        oracle::Tensor r = oracle::ttm(t, m, mode);
        std::memcpy(out, r.a.data(), sizeof(double) * r.a.size());
    });
}

int or_kron(std::int64_t ar, std::int64_t ac, const double* a, std::int64_t br, std::int64_t bc, const double* b,
            double* out) {
    return guarded([&] {
        oracle::Mat A(ar, ac), B(br, bc);
        std::memcpy(A.a.data(), a, sizeof(double) * A.a.size());
        std::memcpy(B.a.data(), b, sizeof(double) * B.a.size());
        oracle::Mat K = oracle::kron(A, B);
        std::memcpy(out, K.a.data(), sizeof(double) * K.a.size());
    });
}

int or_khatri_rao(std::int64_t ar, std::int64_t ac, const double* a, std::int64_t br, std::int64_t bc, const double* b,
                  double* out) {
    return guarded([&] {
        oracle::Mat A(ar, ac), B(br, bc);
        std::memcpy(A.a.data(), a, sizeof(double) * A.a.size());
        std::memcpy(B.a.data(), b, sizeof(double) * B.a.size());
        oracle::Mat K = oracle::khatri_rao(A, B);
        std::memcpy(out, K.a.data(), sizeof(double) * K.a.size());
    });
}

// q: rows × min(rows, cols); r: min × cols.
int or_qr_econ(std::int64_t rows, std::int64_t cols, const double* a, double* q, double* r) {
    return guarded([&] {
        oracle::Mat A(rows, cols);
        std::memcpy(A.a.data(), a, sizeof(double) * A.a.size());
        oracle::Qr f = oracle::qr_econ(A);
        std::memcpy(q, f.q.a.data(), sizeof(double) * f.q.a.size());
        std::memcpy(r, f.r.a.data(), sizeof(double) * f.r.a.size());
    });
}

// u: rows × k, s: k, v: cols × k with k = min(rows, cols).
int or_svd_econ(std::int64_t rows, std::int64_t cols, const double* a, double* u, double* s, double* v) {
    return guarded([&] {
        oracle::Mat A(rows, cols);
        std::memcpy(A.a.data(), a, sizeof(double) * A.a.size());
        oracle::Svd f = oracle::svd_econ(A);
        std::memcpy(u, f.u.a.data(), sizeof(double) * f.u.a.size());
        std::memcpy(s, f.s.data(), sizeof(double) * f.s.size());
        std::memcpy(v, f.v.a.data(), sizeof(double) * f.v.a.size());
    });
}

int or_sym_eig(std::int64_t n, const double* a, double* values, double* vectors) {
    return guarded([&] {
        oracle::Mat A(n, n);
        std::memcpy(A.a.data(), a, sizeof(double) * A.a.size());
        oracle::SymEig e = oracle::sym_eig(A);
        std::memcpy(values, e.values.data(), sizeof(double) * e.values.size());
        std::memcpy(vectors, e.vectors.a.data(), sizeof(double) * e.vectors.a.size());
    });
}

// Runs krp_sum on K summand views. widths == nullptr → the plan is built by
// effective_subrank (src/sketch.cpp:75-79) with the given oversampling.
// krp != 0: krp_sum (src/sketch.cpp:360-362); krp == 0: kron_sum (:364-366).
int or_sketched_sum(const OrTuckerView* views, std::int64_t count, const double* weights, const std::int64_t* widths,
                    std::int64_t oversampling, std::uint64_t seed, std::uint64_t stream, double eps,
                    const std::int64_t* cap, int threads, int keep_intermediates, int krp, void** out) {
    return guarded([&] {
        std::vector<oracle::Tucker> xs = views_to_tuckers(views, count);
        std::vector<const oracle::Tucker*> ptrs;
        for (auto& x : xs) ptrs.push_back(&x);
        std::vector<double> ws(weights, weights + std::max<std::int64_t>(count, 0));
        auto res = std::make_unique<OrResult>();
        if (ptrs.empty()) throw std::invalid_argument("sum request needs matching, nonempty summands and weights");
        const size_t order = ptrs.front()->ranks.size();
        if (widths != nullptr) {
            res->widths.assign(widths, widths + order);
        } else {
            if (order < 2) throw std::invalid_argument("sketched summation needs order >= 2");
            res->widths = oracle::effective_subrank(ptrs, ws, eps, std::vector<std::int64_t>(order, oversampling),
                                                    &res->eff, &res->targets, krp != 0);
        }
        res->t = oracle::sketched_sum(ptrs, ws, res->widths, oracle::Seed{seed, stream}, eps, cap, threads,
                                      keep_intermediates ? &res->inter : nullptr, krp != 0);
        *out = res.release();
    });
}

int or_krp_sum(const OrTuckerView* views, std::int64_t count, const double* weights, const std::int64_t* widths,
               std::int64_t oversampling, std::uint64_t seed, std::uint64_t stream, double eps,
               const std::int64_t* cap, int threads, int keep_intermediates, void** out) {
    return or_sketched_sum(views, count, weights, widths, oversampling, seed, stream, eps, cap, threads,
                           keep_intermediates, 1, out);
}

// lazy_sum (src/sketch.cpp:48-50): tucker_rounding(formal_sum(summands, weights), eps).
int or_lazy_sum(const OrTuckerView* views, std::int64_t count, const double* weights, double eps,
                const std::int64_t* cap, void** out) {
    return guarded([&] {
        std::vector<oracle::Tucker> xs = views_to_tuckers(views, count);
        std::vector<const oracle::Tucker*> ptrs;
        for (auto& x : xs) ptrs.push_back(&x);
        std::vector<double> ws(weights, weights + std::max<std::int64_t>(count, 0));
        auto res = std::make_unique<OrResult>();
        res->t = oracle::tucker_rounding(oracle::formal_sum(ptrs, ws), eps, cap);
        res->widths.assign(res->t.ranks.size(), 0);
        *out = res.release();
    });
}

int or_kron_sketch_dims(std::int64_t order, const std::int64_t* targets, const std::int64_t* dims, std::int64_t* out) {
    return guarded([&] {
        const size_t o = static_cast<size_t>(std::max<std::int64_t>(order, 0));
        std::vector<std::int64_t> s =
            oracle::kron_sketch_dims(std::vector<std::int64_t>(targets, targets + o), std::vector<std::int64_t>(dims, dims + o));
        std::copy(s.begin(), s.end(), out);
    });
}

int or_effective_subrank(const OrTuckerView* views, std::int64_t count, const double* weights, double eps,
                         const std::int64_t* oversampling, int krp, std::int64_t* eff, std::int64_t* targets,
                         std::int64_t* widths) {
    return guarded([&] {
        std::vector<oracle::Tucker> xs = views_to_tuckers(views, count);
        std::vector<const oracle::Tucker*> ptrs;
        for (auto& x : xs) ptrs.push_back(&x);
        if (ptrs.empty()) throw std::invalid_argument("sum request needs matching, nonempty summands and weights");
        std::vector<double> ws(weights, weights + count);
        const size_t order = ptrs.front()->ranks.size();
        std::vector<std::int64_t> e, t;
        std::vector<std::int64_t> w =
            oracle::effective_subrank(ptrs, ws, eps, std::vector<std::int64_t>(oversampling, oversampling + order), &e, &t,
                                      krp != 0);
        std::copy(e.begin(), e.end(), eff);
        std::copy(t.begin(), t.end(), targets);
        std::copy(w.begin(), w.end(), widths);
    });
}

// Sharded building blocks (the two data-parallel loops of src/sketch.cpp:103-143
// and :155-169 over a subset of summands).  y_out: concatenated Y_n (dims[n] × s).
int or_partial_sketch(const OrTuckerView* views, std::int64_t count, const double* weights, std::int64_t s,
                      std::uint64_t seed, std::uint64_t stream, double* y_out) {
    return guarded([&] {
        std::vector<oracle::Tucker> xs = views_to_tuckers(views, count);
        std::vector<const oracle::Tucker*> ptrs;
        for (auto& x : xs) ptrs.push_back(&x);
        std::vector<double> ws(weights, weights + count);
        const size_t ou = ptrs.front()->ranks.size();
        std::vector<oracle::Mat> omega(ou), y(ou);
        for (size_t n = 0; n < ou; ++n) {
            omega[n] = oracle::gaussian_matrix(ptrs.front()->dims[n], s, oracle::Seed{seed, stream}.substream(n));
            y[n] = oracle::Mat(ptrs.front()->dims[n], s);
        }
        oracle::accumulate_sketch(ptrs, ws, 0, ptrs.size(), omega, y);
        size_t off = 0;
        for (size_t n = 0; n < ou; ++n) {
            std::memcpy(y_out + off, y[n].a.data(), sizeof(double) * y[n].a.size());
            off += y[n].a.size();
        }
    });
}

// As or_partial_sketch with per-mode plan widths; krp = 0 is the Kron sketch
// (Ω_n is dims[n] × widths[n], Y_n has Π_{j≠n} widths[j] columns).
int or_partial_sketch_ex(const OrTuckerView* views, std::int64_t count, const double* weights,
                         const std::int64_t* widths, int krp, std::uint64_t seed, std::uint64_t stream, double* y_out) {
    return guarded([&] {
        std::vector<oracle::Tucker> xs = views_to_tuckers(views, count);
        std::vector<const oracle::Tucker*> ptrs;
        for (auto& x : xs) ptrs.push_back(&x);
        std::vector<double> ws(weights, weights + count);
        const size_t ou = ptrs.front()->ranks.size();
        std::vector<std::int64_t> wv(widths, widths + ou);
        const std::int64_t smax = *std::max_element(wv.begin(), wv.end());
        std::vector<oracle::Mat> omega(ou), y(ou);
        for (size_t n = 0; n < ou; ++n) {
            omega[n] = oracle::gaussian_matrix(ptrs.front()->dims[n], krp ? smax : wv[n],
                                               oracle::Seed{seed, stream}.substream(n));
            y[n] = oracle::Mat(ptrs.front()->dims[n], krp ? smax : oracle::complement_product(wv, n));
        }
        oracle::accumulate_sketch(ptrs, ws, 0, ptrs.size(), omega, y, krp != 0);
        size_t off = 0;
        for (size_t n = 0; n < ou; ++n) {
            std::memcpy(y_out + off, y[n].a.data(), sizeof(double) * y[n].a.size());
            off += y[n].a.size();
        }
    });
}

// h_out (prod qdims) = Σ_i w_i G_i ×_n (Û_nᵀ U_n^(i)) over the given summands.
int or_partial_core(const OrTuckerView* views, std::int64_t count, const double* weights,
                    const double* const* uhat, const std::int64_t* qdims, double* h_out) {
    return guarded([&] {
        std::vector<oracle::Tucker> xs = views_to_tuckers(views, count);
        std::vector<const oracle::Tucker*> ptrs;
        for (auto& x : xs) ptrs.push_back(&x);
        std::vector<double> ws(weights, weights + count);
        const size_t ou = ptrs.front()->ranks.size();
        std::vector<oracle::Mat> u(ou);
        std::vector<std::int64_t> q(qdims, qdims + ou);
        for (size_t n = 0; n < ou; ++n) {
            u[n] = oracle::Mat(ptrs.front()->dims[n], q[n]);
            std::memcpy(u[n].a.data(), uhat[n], sizeof(double) * u[n].a.size());
        }
        oracle::Tensor h(q);
        oracle::accumulate_core(ptrs, ws, 0, ptrs.size(), u, h);
        std::memcpy(h_out, h.a.data(), sizeof(double) * h.a.size());
    });
}

// Result accessors (a dense-core Tucker tensor).
std::int64_t or_result_order(void* h) { return static_cast<OrResult*>(h)->t.order(); }
void or_result_dims(void* h, std::int64_t* dims) {
    auto* r = static_cast<OrResult*>(h);
    std::copy(r->t.dims.begin(), r->t.dims.end(), dims);
}
void or_result_ranks(void* h, std::int64_t* ranks) {
    auto* r = static_cast<OrResult*>(h);
    std::copy(r->t.ranks.begin(), r->t.ranks.end(), ranks);
}
void or_result_widths(void* h, std::int64_t* widths) {
    auto* r = static_cast<OrResult*>(h);
    std::copy(r->widths.begin(), r->widths.end(), widths);
}
void or_result_factor(void* h, std::int64_t mode, double* out) {
    auto* r = static_cast<OrResult*>(h);
    const auto& f = r->t.factors[static_cast<size_t>(mode)];
    std::memcpy(out, f.a.data(), sizeof(double) * f.a.size());
}
void or_result_core(void* h, double* out) {
    auto* r = static_cast<OrResult*>(h);
    const auto& c = r->t.blocks[0].data;
    std::memcpy(out, c.a.data(), sizeof(double) * c.a.size());
}
// Intermediates (when keep_intermediates): which = 0 Ω_n, 1 Y_n, 2 Û_n (cols via *cols), 3 h (mode ignored).
std::int64_t or_result_inter(void* h, int which, std::int64_t mode, double* out, std::int64_t* rows, std::int64_t* cols) {
    auto* r = static_cast<OrResult*>(h);
    const oracle::Mat* m = nullptr;
    if (which == 0) m = &r->inter.omega[static_cast<size_t>(mode)];
    if (which == 1) m = &r->inter.y[static_cast<size_t>(mode)];
    if (which == 2) m = &r->inter.uhat[static_cast<size_t>(mode)];
    if (which == 3) {
        if (out) std::memcpy(out, r->inter.h.a.data(), sizeof(double) * r->inter.h.a.size());
        if (rows) *rows = r->inter.h.size();
        if (cols) *cols = 1;
        return r->inter.h.size();
    }
    if (m == nullptr) return -1;
    if (out) std::memcpy(out, m->a.data(), sizeof(double) * m->a.size());
    if (rows) *rows = m->r;
    if (cols) *cols = m->c;
    return static_cast<std::int64_t>(m->a.size());
}
void or_result_free(void* h) { delete static_cast<OrResult*>(h); }

// Error metrics on Tucker views (src/tucker.cpp:159-181,298-303).
int or_tucker_norm(const OrTuckerView* x, double* out) {
    return guarded([&] { *out = oracle::tucker_norm(from_view(*x)); });
}
int or_tucker_inner(const OrTuckerView* x, const OrTuckerView* y, double* out) {
    return guarded([&] { *out = oracle::tucker_inner(from_view(*x), from_view(*y)); });
}
// rel error of x against formal_sum(summands, weights) (src/tucker.cpp:298-303 + 183-233).
int or_rel_error_to_sum(const OrTuckerView* x, const OrTuckerView* views, std::int64_t count, const double* weights,
                        double* out) {
    return guarded([&] {
        oracle::Tucker xt = from_view(*x);
        std::vector<oracle::Tucker> xs = views_to_tuckers(views, count);
        std::vector<const oracle::Tucker*> ptrs;
        for (auto& v : xs) ptrs.push_back(&v);
        oracle::Tucker ref = oracle::formal_sum(ptrs, std::vector<double>(weights, weights + count));
        *out = oracle::tucker_rel_error(xt, ref);
    });
}
// Gram-based relative error ‖x − Σ w_k X_k‖/‖Σ w_k X_k‖ through pairwise inner products
// (SURVEY.md §8(d) error metric for configs whose formal-sum core cannot be densified).
int or_rel_error_gram(const OrTuckerView* x, const OrTuckerView* views, std::int64_t count, const double* weights,
                      int threads, double* out) {
    return guarded([&] {
        oracle::Tucker xt = from_view(*x);
        std::vector<oracle::Tucker> xs = views_to_tuckers(views, count);
        const std::int64_t K = count;
        std::vector<double> rows(static_cast<size_t>(K), 0.0), cross(static_cast<size_t>(K), 0.0);
#pragma omp parallel for schedule(dynamic) num_threads(std::max(1, threads))
        for (std::int64_t i = 0; i < K; ++i) {
            double acc = 0.0;
            for (std::int64_t j = 0; j < K; ++j) acc += weights[j] * oracle::tucker_inner(xs[static_cast<size_t>(i)], xs[static_cast<size_t>(j)]);
            rows[static_cast<size_t>(i)] = weights[i] * acc;
            cross[static_cast<size_t>(i)] = weights[i] * oracle::tucker_inner(xs[static_cast<size_t>(i)], xt);
        }
        double ss = 0, sx = 0;
        for (std::int64_t i = 0; i < K; ++i) {
            ss += rows[static_cast<size_t>(i)];
            sx += cross[static_cast<size_t>(i)];
        }
        const double xx = oracle::tucker_inner(xt, xt);
        const double diff2 = std::max(0.0, ss - 2.0 * sx + xx);
        *out = ss > 0 ? std::sqrt(diff2 / ss) : std::sqrt(diff2);
    });
}

// Dense reconstruction (src/tucker.cpp:102-119); out has prod(dims) entries.
int or_reconstruct(const OrTuckerView* x, double* out) {
    return guarded([&] {
        oracle::Tensor t = oracle::reconstruct(from_view(*x));
        std::memcpy(out, t.a.data(), sizeof(double) * t.a.size());
    });
}

int or_num_threads() {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

}  // extern "C"
