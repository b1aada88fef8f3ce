// capi_host.cpp — a C++ caller of the drop-in C ABI (include/tucksum_cuda.h),
// the way the reference's adapter would use it, with no Python in the loop.
//
// Builds K orthonormal-factor Tucker summands on the host, uploads them,
// runs ts_krp_sum twice (the second call reuses the device batch and the cached
// Ω), and checks: status codes, the reference's error behaviour on malformed
// requests (TS_INVALID_ARGUMENT ↔ std::invalid_argument), output ranks, factor
// orthonormality, bitwise determinism, and that the result reproduces a summand
// set whose exact sum has rank below the cap (annihilation / pass-through
// semantics of proj/tests/test_sketch_sum.cpp).  Exit code 0 = pass.
//
// Built by __graft_entry__.build() (tests/cpp/build.sh); run by
// tests/test_gpu_parity.py::test_cpp_host_caller.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "tucksum_cuda.h"

namespace {

int failures = 0;
#define CHECK(cond, ...)                                  \
    do {                                                  \
        if (!(cond)) {                                    \
            std::fprintf(stderr, "FAIL %s:%d: ", __FILE__, __LINE__); \
            std::fprintf(stderr, __VA_ARGS__);            \
            std::fprintf(stderr, "\n");                   \
            ++failures;                                   \
        }                                                 \
    } while (0)

// Column-major n × r matrix with orthonormal columns (modified Gram-Schmidt of a
// Gaussian matrix).
std::vector<double> orthonormal(int64_t n, int64_t r, std::mt19937_64& gen) {
    std::normal_distribution<double> N01;
    std::vector<double> a(static_cast<size_t>(n * r));
    for (double& x : a) x = N01(gen);
    for (int64_t j = 0; j < r; ++j) {
        double* cj = a.data() + j * n;
        for (int64_t i = 0; i < j; ++i) {
            const double* ci = a.data() + i * n;
            double d = 0.0;
            for (int64_t t = 0; t < n; ++t) d += ci[t] * cj[t];
            for (int64_t t = 0; t < n; ++t) cj[t] -= d * ci[t];
        }
        double nn = 0.0;
        for (int64_t t = 0; t < n; ++t) nn += cj[t] * cj[t];
        nn = std::sqrt(nn);
        for (int64_t t = 0; t < n; ++t) cj[t] /= nn;
    }
    return a;
}

struct Summand {
    std::vector<int64_t> dims, ranks, offsets;
    std::vector<std::vector<double>> factors;
    std::vector<double> core;
    std::vector<const double*> fptr;
    const double* cptr = nullptr;
    ts_tucker_view view() {
        fptr.clear();
        for (auto& f : factors) fptr.push_back(f.data());
        cptr = core.data();
        ts_tucker_view v{};
        v.order = static_cast<int64_t>(dims.size());
        v.dims = dims.data();
        v.ranks = ranks.data();
        v.factors = fptr.data();
        v.num_blocks = 1;
        v.block_offsets = offsets.data();
        v.block_shapes = ranks.data();
        v.block_data = &cptr;
        return v;
    }
};

struct Result {
    std::vector<int64_t> ranks;
    std::vector<std::vector<double>> factors;
    std::vector<double> core;
};

Result fetch(ts_result* r, int order, const std::vector<int64_t>& dims) {
    Result out;
    out.ranks.resize(static_cast<size_t>(order));
    ts_result_ranks(r, out.ranks.data());
    int64_t csize = 1;
    for (int k = 0; k < order; ++k) {
        out.factors.emplace_back(static_cast<size_t>(dims[static_cast<size_t>(k)] * out.ranks[static_cast<size_t>(k)]));
        CHECK(ts_result_factor(r, k, out.factors.back().data()) == TS_OK, "ts_result_factor: %s", ts_last_error());
        csize *= out.ranks[static_cast<size_t>(k)];
    }
    out.core.resize(static_cast<size_t>(csize));
    CHECK(ts_result_core(r, out.core.data()) == TS_OK, "ts_result_core: %s", ts_last_error());
    return out;
}

}  // namespace

int main() {
    const int order = 3;
    const int64_t n = 64, r = 6, K = 4, s = 20;
    std::mt19937_64 gen(2603);
    std::normal_distribution<double> N01;

    // Summands 2 and 3 repeat the factors of 0 and 1, so the exact sum has
    // multilinear rank ≤ 12 < cap = 16 … but with 4 distinct cores.
    std::vector<Summand> xs(static_cast<size_t>(K));
    for (int64_t k = 0; k < K; ++k) {
        Summand& x = xs[static_cast<size_t>(k)];
        x.dims.assign(order, n);
        x.ranks.assign(order, r);
        x.offsets.assign(order, 0);
        for (int j = 0; j < order; ++j) {
            if (k < 2) x.factors.push_back(orthonormal(n, r, gen));
            else x.factors.push_back(xs[static_cast<size_t>(k - 2)].factors[static_cast<size_t>(j)]);
        }
        x.core.resize(static_cast<size_t>(r * r * r));
        for (double& c : x.core) c = N01(gen);
    }
    std::vector<ts_tucker_view> views;
    for (auto& x : xs) views.push_back(x.view());
    const std::vector<double> w = {1.0, 0.5, -0.25, 2.0};
    const std::vector<int64_t> widths(order, s), cap(order, 16), dims(order, n);

    ts_ctx* ctx = nullptr;
    if (ts_ctx_create(0, &ctx) != TS_OK) {
        std::fprintf(stderr, "FAIL ts_ctx_create: %s\n", ts_last_error());
        return 2;
    }
    ts_batch* batch = nullptr;
    CHECK(ts_batch_upload(ctx, views.data(), K, &batch) == TS_OK, "upload: %s", ts_last_error());
    CHECK(ts_batch_count(batch) == K, "batch count");

    // Malformed requests keep the reference's exception class.
    ts_result* bad = nullptr;
    CHECK(ts_krp_sum(ctx, batch, w.data(), widths.data(), 7, 1, -1.0, nullptr, &bad) == TS_INVALID_ARGUMENT,
          "negative eps must be TS_INVALID_ARGUMENT");
    const std::vector<int64_t> zero(order, 0);
    CHECK(ts_krp_sum(ctx, batch, w.data(), zero.data(), 7, 1, 0.0, nullptr, &bad) == TS_INVALID_ARGUMENT,
          "zero width must be TS_INVALID_ARGUMENT");
    CHECK(ts_krp_sum(ctx, batch, nullptr, widths.data(), 7, 1, 0.0, nullptr, &bad) == TS_INVALID_ARGUMENT,
          "null weights must be TS_INVALID_ARGUMENT");

    Result out[2];
    for (int rep = 0; rep < 2; ++rep) {
        ts_result* res = nullptr;
        CHECK(ts_krp_sum(ctx, batch, w.data(), widths.data(), 7, 1, 1e-12, cap.data(), &res) == TS_OK, "krp_sum: %s",
              ts_last_error());
        if (!res) return 1;
        CHECK(ts_result_order(res) == order, "order");
        out[rep] = fetch(res, order, dims);
        ts_result_free(res);
    }
    // Exact rank 12 per mode (two distinct factor sets of rank 6) is recovered.
    for (int k = 0; k < order; ++k) CHECK(out[0].ranks[static_cast<size_t>(k)] == 12, "rank[%d] = %lld, want 12", k,
                                          static_cast<long long>(out[0].ranks[static_cast<size_t>(k)]));
    // Orthonormal output factors.
    for (int k = 0; k < order; ++k) {
        const int64_t rk = out[0].ranks[static_cast<size_t>(k)];
        const double* U = out[0].factors[static_cast<size_t>(k)].data();
        double worst = 0.0;
        for (int64_t a = 0; a < rk; ++a)
            for (int64_t b = 0; b < rk; ++b) {
                double d = 0.0;
                for (int64_t t = 0; t < n; ++t) d += U[t + a * n] * U[t + b * n];
                worst = std::fmax(worst, std::fabs(d - (a == b ? 1.0 : 0.0)));
            }
        CHECK(worst < 1e-12, "factor %d not orthonormal (%.3e)", k, worst);
    }
    // Bitwise determinism across calls (device batch and Ω reused).
    for (int k = 0; k < order; ++k)
        CHECK(out[0].factors[static_cast<size_t>(k)] == out[1].factors[static_cast<size_t>(k)], "factor %d differs", k);
    CHECK(out[0].core == out[1].core, "core differs between identical calls");

    // The sum is exactly representable at rank 12: compare ‖X̃‖² with ‖Σ w_k X_k‖²
    // through the core Grams (factors orthonormal, shared factor sets).
    double out_norm2 = 0.0;
    for (double c : out[0].core) out_norm2 += c * c;
    // Exact: summands 0/2 share factors, 1/3 share factors → combined cores.
    double exact_norm2 = 0.0;
    {
        std::vector<double> c02(static_cast<size_t>(r * r * r)), c13(c02.size());
        for (size_t i = 0; i < c02.size(); ++i) {
            c02[i] = w[0] * xs[0].core[i] + w[2] * xs[2].core[i];
            c13[i] = w[1] * xs[1].core[i] + w[3] * xs[3].core[i];
        }
        double n02 = 0.0, n13 = 0.0;
        for (size_t i = 0; i < c02.size(); ++i) {
            n02 += c02[i] * c02[i];
            n13 += c13[i] * c13[i];
        }
        // Cross term ⟨X02, X13⟩ = ⟨c02 ×_j (U0ᵀU1), c13⟩.
        std::vector<double> M[3];
        for (int j = 0; j < order; ++j) {
            M[j].assign(static_cast<size_t>(r * r), 0.0);
            const double* A = xs[0].factors[static_cast<size_t>(j)].data();
            const double* B = xs[1].factors[static_cast<size_t>(j)].data();
            for (int64_t a = 0; a < r; ++a)
                for (int64_t b = 0; b < r; ++b) {
                    double d = 0.0;
                    for (int64_t t = 0; t < n; ++t) d += A[t + a * n] * B[t + b * n];
                    M[j][static_cast<size_t>(a + b * r)] = d;
                }
        }
        double cross = 0.0;
        for (int64_t a0 = 0; a0 < r; ++a0)
            for (int64_t a1 = 0; a1 < r; ++a1)
                for (int64_t a2 = 0; a2 < r; ++a2) {
                    const double x = c02[static_cast<size_t>(a0 + r * (a1 + r * a2))];
                    for (int64_t b0 = 0; b0 < r; ++b0)
                        for (int64_t b1 = 0; b1 < r; ++b1)
                            for (int64_t b2 = 0; b2 < r; ++b2)
                                cross += x * M[0][static_cast<size_t>(a0 + b0 * r)] * M[1][static_cast<size_t>(a1 + b1 * r)] *
                                         M[2][static_cast<size_t>(a2 + b2 * r)] *
                                         c13[static_cast<size_t>(b0 + r * (b1 + r * b2))];
                }
        exact_norm2 = n02 + n13 + 2.0 * cross;
    }
    CHECK(std::fabs(out_norm2 - exact_norm2) <= 1e-10 * exact_norm2, "‖X̃‖² = %.15e vs exact %.15e", out_norm2,
          exact_norm2);

    // The same sum through the other device strategies and the device norms:
    // Lazy rounding (stacked rank 4·6 = 24) and the Kron sketch recover rank 12,
    // the orthogonalized norm of the formal sum equals the exact norm, and the
    // device error of the KRP result to the exact sum is ~0 (exact rank).
    {
        double snorm = 0.0;
        CHECK(ts_tucker_norm(ctx, batch, w.data(), &snorm) == TS_OK, "tucker_norm: %s", ts_last_error());
        CHECK(std::fabs(snorm * snorm - exact_norm2) <= 1e-10 * exact_norm2, "tucker_norm² %.15e vs %.15e",
              snorm * snorm, exact_norm2);
        double ss = 0.0;
        CHECK(ts_tucker_inner(ctx, batch, w.data(), batch, w.data(), &ss) == TS_OK, "tucker_inner: %s", ts_last_error());
        CHECK(std::fabs(ss - exact_norm2) <= 1e-10 * exact_norm2, "tucker_inner %.15e vs %.15e", ss, exact_norm2);
        ts_result* lz = nullptr;
        CHECK(ts_lazy_sum(ctx, batch, w.data(), 1e-12, nullptr, &lz) == TS_OK, "lazy_sum: %s", ts_last_error());
        if (lz) {
            std::vector<int64_t> rk(static_cast<size_t>(order));
            ts_result_ranks(lz, rk.data());
            for (int k = 0; k < order; ++k) CHECK(rk[static_cast<size_t>(k)] == 12, "lazy rank[%d] = %lld", k,
                                                  static_cast<long long>(rk[static_cast<size_t>(k)]));
            double err = 1.0;
            CHECK(ts_rel_error_to_sum(ctx, lz, batch, w.data(), &err) == TS_OK, "rel_error: %s", ts_last_error());
            CHECK(err < 1e-6, "lazy error to the exact sum %.3e", err);
            ts_result_free(lz);
        }
        std::vector<int64_t> kw(static_cast<size_t>(order)), tg(static_cast<size_t>(order), 16);
        CHECK(ts_kron_sketch_dims(order, tg.data(), dims.data(), kw.data()) == TS_OK, "kron dims: %s", ts_last_error());
        ts_result* kr = nullptr;
        CHECK(ts_kron_sum(ctx, batch, w.data(), kw.data(), 7, 2, 1e-12, nullptr, &kr) == TS_OK, "kron_sum: %s",
              ts_last_error());
        if (kr) {
            std::vector<int64_t> rk(static_cast<size_t>(order));
            ts_result_ranks(kr, rk.data());
            for (int k = 0; k < order; ++k) CHECK(rk[static_cast<size_t>(k)] == 12, "kron rank[%d] = %lld", k,
                                                  static_cast<long long>(rk[static_cast<size_t>(k)]));
            ts_result_free(kr);
        }
    }

    CHECK(ts_batch_free(batch) == TS_OK, "batch free");
    CHECK(ts_ctx_destroy(ctx) == TS_OK, "ctx destroy");
    if (failures == 0) std::printf("capi_host ok: ranks 12/12/12, |X|^2 = %.12e (exact %.12e)\n", out_norm2, exact_norm2);
    return failures == 0 ? 0 : 1;
}
