// tucksum_cuda_adapter.hpp — reference-side C++ binding of the B200 C ABI.
//
// Header-only adapter a maintainer of the reference (/root/reference/proj) adds to
// route `tucksum::krp_sum` / `kron_sum` / `round_sum` (every strategy) and the
// tucker_norm / tucker_inner / tucker_rel_error / tucker_rounding helpers to
// libtucksum_cuda.so with the exact reference signatures
// (include/tucksum/sketch.hpp:85-94, include/tucksum/tucker.hpp).  It needs the
// reference headers and therefore Eigen >= 3.4 (include/tucksum/types.hpp:4); it is
// compiled (syntax only, -Werror) against the real reference headers with a minimal Eigen
// shim by tests/test_capi_cpu.py — see INTEGRATION.md.
#pragma once

#include <cstdlib>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "tucksum/sketch.hpp"
#include "tucksum_cuda.h"

namespace tucksum::cuda {

namespace detail {

[[noreturn]] inline void rethrow(int rc) {
    const std::string msg = ts_last_error();
    if (rc == TS_INVALID_ARGUMENT) throw std::invalid_argument(msg);  // src/sketch.cpp:16-30 contract
    throw std::runtime_error(msg);
}
inline void check(int rc) {
    if (rc != TS_OK) rethrow(rc);
}

// Borrowed ts_tucker_view of a reference TuckerTensor (no copies on the host).
struct View {
    std::vector<int64_t> dims, ranks, offsets, shapes;
    std::vector<const double*> factors, blocks;
    ts_tucker_view v{};
    explicit View(const TuckerTensor& x) {
        const auto d = static_cast<size_t>(x.order());
        for (size_t k = 0; k < d; ++k) {
            dims.push_back(x.dims()[k]);
            ranks.push_back(x.ranks()[k]);
            factors.push_back(x.factors()[k].data());  // column-major, ld = dims[k]
        }
        for (const CoreBlock& b : x.blocks()) {
            for (size_t k = 0; k < d; ++k) {
                offsets.push_back(b.offsets[k]);
                shapes.push_back(b.data.shape()[k]);
            }
            blocks.push_back(b.data.data());  // column-major, first index fastest
        }
        v = ts_tucker_view{static_cast<int64_t>(d), dims.data(), ranks.data(), factors.data(),
                           static_cast<int64_t>(blocks.size()), offsets.data(), shapes.data(), blocks.data()};
    }
};

inline ts_ctx* context() {  // one context per process (device from TUCKSUM_DEVICE, default 0)
    static std::unique_ptr<ts_ctx, int (*)(ts_ctx*)> ctx = [] {
        ts_ctx* c = nullptr;
        const char* env = std::getenv("TUCKSUM_DEVICE");
        check(ts_ctx_create(env ? std::atoi(env) : 0, &c));
        return std::unique_ptr<ts_ctx, int (*)(ts_ctx*)>(c, ts_ctx_destroy);
    }();
    return ctx.get();
}

}  // namespace detail

namespace detail {

using BatchPtr = std::unique_ptr<ts_batch, int (*)(ts_batch*)>;
using ResultPtr = std::unique_ptr<ts_result, int (*)(ts_result*)>;

// Device copy of tensors in the stacked formal-sum layout (ts_batch_upload).
inline BatchPtr upload(const std::vector<const TuckerTensor*>& xs) {
    std::vector<View> views;
    views.reserve(xs.size());
    for (const TuckerTensor* x : xs) {
        if (x == nullptr) throw std::invalid_argument("sum request holds a null summand");
        views.emplace_back(*x);
    }
    std::vector<ts_tucker_view> vs;
    for (auto& v : views) vs.push_back(v.v);
    ts_batch* batch = nullptr;
    check(ts_batch_upload(context(), vs.data(), static_cast<int64_t>(vs.size()), &batch));
    return BatchPtr(batch, ts_batch_free);
}

inline TuckerTensor to_tucker(ts_result* res) {
    ResultPtr guard(res, ts_result_free);
    const auto d = static_cast<size_t>(ts_result_order(res));
    std::vector<int64_t> dims(d), ranks(d);
    ts_result_dims(res, dims.data());
    ts_result_ranks(res, ranks.data());
    std::vector<Matrix> factors(d);
    for (size_t n = 0; n < d; ++n) {
        factors[n].resize(dims[n], ranks[n]);
        check(ts_result_factor(res, static_cast<int64_t>(n), factors[n].data()));
    }
    DenseTensor core(std::vector<Index>(ranks.begin(), ranks.end()));
    check(ts_result_core(res, core.data()));
    return TuckerTensor(std::move(core), std::move(factors));
}

// sketched_sum (src/sketch.cpp:66-181) for krp = true (ts_krp_sum) / false (ts_kron_sum).
inline TuckerTensor sketched(const SumRequest& req, const SketchPlan* plan, SumStats* stats, bool krp) {
    if (req.summands.empty() || req.summands.size() != req.weights.size())
        throw std::invalid_argument("sum request needs matching, nonempty summands and weights");
    ts_ctx* ctx = context();
    BatchPtr bguard = upload(req.summands);
    ts_batch* batch = bguard.get();
    const auto d = static_cast<size_t>(req.summands.front()->order());
    SketchPlan p;
    if (plan != nullptr) {
        p = *plan;
    } else {  // plan stage on the device (src/sketch.cpp:75-79 → effective_subrank)
        p.strategy = krp ? Strategy::Krp : Strategy::Kron;
        p.eps = req.eps;
        p.seed = req.seed;
        p.oversampling.assign(d, req.oversampling);
        p.effective_ranks.resize(d);
        p.targets.resize(d);
        p.mode_sketch_dims.resize(d);
        std::vector<int64_t> ov(p.oversampling.begin(), p.oversampling.end()), e(d), t(d), w(d);
        check((krp ? ts_effective_subrank : ts_effective_subrank_kron)(ctx, batch, req.weights.data(), req.eps,
                                                                       ov.data(), e.data(), t.data(), w.data()));
        for (size_t n = 0; n < d; ++n) {
            p.effective_ranks[n] = e[n];
            p.targets[n] = t[n];
            p.mode_sketch_dims[n] = w[n];
        }
    }
    if (p.mode_sketch_dims.size() != d) throw std::invalid_argument("plan order does not match summand order");
    std::vector<int64_t> widths(p.mode_sketch_dims.begin(), p.mode_sketch_dims.end());
    ts_result* res = nullptr;
    check((krp ? ts_krp_sum : ts_kron_sum)(ctx, batch, req.weights.data(), widths.data(), req.seed.seed,
                                           req.seed.stream, req.eps, nullptr, &res));
    TuckerTensor out = to_tucker(res);
    if (stats != nullptr) {
        stats->plan = p;
        stats->has_plan = true;
    }
    return out;
}

}  // namespace detail

// Drop-in for tucksum::krp_sum (src/sketch.cpp:360-362 → sketched_sum(krp=true)).
inline TuckerTensor krp_sum(const SumRequest& req, const SketchPlan* plan = nullptr, SumStats* stats = nullptr) {
    return detail::sketched(req, plan, stats, true);
}

// Drop-in for tucksum::kron_sum (src/sketch.cpp:364-366 → sketched_sum(krp=false)).
inline TuckerTensor kron_sum(const SumRequest& req, const SketchPlan* plan = nullptr, SumStats* stats = nullptr) {
    return detail::sketched(req, plan, stats, false);
}

// Drop-in for tucksum::tucker_rounding (src/tucker.cpp:285-296), stacked ranks ≤ 96.
inline TuckerTensor tucker_rounding(const TuckerTensor& x, double tau) {
    if (tau < 0.0) throw std::invalid_argument("tucker_rounding: tolerance must be nonnegative");
    detail::BatchPtr b = detail::upload({&x});
    const double one = 1.0;
    ts_result* res = nullptr;
    detail::check(ts_lazy_sum(detail::context(), b.get(), &one, tau, nullptr, &res));
    return detail::to_tucker(res);
}

// Drop-in for tucksum::tucker_norm / tucker_inner / tucker_rel_error (src/tucker.cpp:159-181,298-303).
inline double tucker_norm(const TuckerTensor& x) {
    detail::BatchPtr b = detail::upload({&x});
    const double one = 1.0;
    double out = 0.0;
    detail::check(ts_tucker_norm(detail::context(), b.get(), &one, &out));
    return out;
}
inline double tucker_inner(const TuckerTensor& x, const TuckerTensor& y) {
    if (x.dims() != y.dims()) throw std::invalid_argument("tucker_inner: operands must share dims");
    detail::BatchPtr bx = detail::upload({&x}), by = detail::upload({&y});
    const double one = 1.0;
    double out = 0.0;
    detail::check(ts_tucker_inner(detail::context(), bx.get(), &one, by.get(), &one, &out));
    return out;
}
inline double tucker_rel_error(const TuckerTensor& x, const TuckerTensor& ref) {
    detail::BatchPtr bd = detail::upload({&x, &ref});
    const double w[2] = {1.0, -1.0};
    double diff = 0.0;
    detail::check(ts_tucker_norm(detail::context(), bd.get(), w, &diff));
    const double denom = cuda::tucker_norm(ref);  // qualified: ADL also finds tucksum::tucker_norm
    return denom == 0.0 ? diff : diff / denom;
}

// Drop-in dispatcher (src/sketch.cpp:368-376): every strategy on the B200.
// Lazy = one device rounding of the formal sum; Eager = the reference's left
// fold with one device rounding per summand (src/sketch.cpp:52-64).
inline TuckerTensor round_sum(const SumRequest& req, const SketchPlan* plan = nullptr, SumStats* stats = nullptr) {
    switch (req.strategy) {
        case Strategy::Krp: return cuda::krp_sum(req, plan, stats);
        case Strategy::Kron: return cuda::kron_sum(req, plan, stats);
        case Strategy::Lazy: {
            detail::BatchPtr b = detail::upload(req.summands);
            ts_result* res = nullptr;
            detail::check(ts_lazy_sum(detail::context(), b.get(), req.weights.data(), req.eps, nullptr, &res));
            return detail::to_tucker(res);
        }
        case Strategy::Eager: {
            if (req.summands.empty() || req.summands.size() != req.weights.size())
                throw std::invalid_argument("sum request needs matching, nonempty summands and weights");
            if (stats != nullptr) stats->eager_rank_trace.clear();
            TuckerTensor acc = formal_sum(std::vector<const TuckerTensor*>{req.summands.front()}, {req.weights.front()});
            for (std::size_t i = 1; i < req.summands.size(); ++i) {
                acc = cuda::tucker_rounding(tucker_axby(1.0, acc, req.weights[i], *req.summands[i]), req.eps);
                if (stats != nullptr) stats->eager_rank_trace.push_back(acc.ranks());
            }
            return acc;
        }
    }
    throw std::invalid_argument("unknown strategy");
}

}  // namespace tucksum::cuda
