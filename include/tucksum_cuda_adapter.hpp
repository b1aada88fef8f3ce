// tucksum_cuda_adapter.hpp — reference-side C++ binding of the B200 C ABI.
//
// Header-only adapter a maintainer of the reference (/root/reference/proj) adds to
// route `tucksum::krp_sum` / `round_sum(Strategy::Krp)` to libtucksum_cuda.so with
// the exact reference signatures (include/tucksum/sketch.hpp:85-94).  It needs the
// reference headers and therefore Eigen >= 3.4 (include/tucksum/types.hpp:4); it is
// not compiled in this image (no Eigen) — see INTEGRATION.md.
#pragma once

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

// Drop-in for tucksum::krp_sum (src/sketch.cpp:360-362 → sketched_sum(krp=true)).
inline TuckerTensor krp_sum(const SumRequest& req, const SketchPlan* plan = nullptr, SumStats* stats = nullptr) {
    if (req.summands.empty() || req.summands.size() != req.weights.size())
        throw std::invalid_argument("sum request needs matching, nonempty summands and weights");
    std::vector<detail::View> views;
    views.reserve(req.summands.size());
    for (const TuckerTensor* x : req.summands) {
        if (x == nullptr) throw std::invalid_argument("sum request holds a null summand");
        views.emplace_back(*x);
    }
    std::vector<ts_tucker_view> vs;
    for (auto& v : views) vs.push_back(v.v);
    ts_ctx* ctx = detail::context();
    ts_batch* batch = nullptr;
    detail::check(ts_batch_upload(ctx, vs.data(), static_cast<int64_t>(vs.size()), &batch));
    std::unique_ptr<ts_batch, int (*)(ts_batch*)> bguard(batch, ts_batch_free);
    const auto d = static_cast<size_t>(req.summands.front()->order());
    SketchPlan p;
    if (plan != nullptr) {
        p = *plan;
    } else {  // plan stage on the device (src/sketch.cpp:75-79 → effective_subrank)
        p.strategy = Strategy::Krp;
        p.eps = req.eps;
        p.seed = req.seed;
        p.oversampling.assign(d, req.oversampling);
        p.effective_ranks.resize(d);
        p.targets.resize(d);
        p.mode_sketch_dims.resize(d);
        std::vector<int64_t> ov(p.oversampling.begin(), p.oversampling.end()), e(d), t(d), w(d);
        detail::check(ts_effective_subrank(ctx, batch, req.weights.data(), req.eps, ov.data(), e.data(), t.data(),
                                           w.data()));
        for (size_t n = 0; n < d; ++n) {
            p.effective_ranks[n] = e[n];
            p.targets[n] = t[n];
            p.mode_sketch_dims[n] = w[n];
        }
    }
    if (p.mode_sketch_dims.size() != d) throw std::invalid_argument("plan order does not match summand order");
    std::vector<int64_t> widths(p.mode_sketch_dims.begin(), p.mode_sketch_dims.end());
    ts_result* res = nullptr;
    detail::check(ts_krp_sum(ctx, batch, req.weights.data(), widths.data(), req.seed.seed, req.seed.stream, req.eps,
                             nullptr, &res));
    std::unique_ptr<ts_result, int (*)(ts_result*)> rguard(res, ts_result_free);
    std::vector<int64_t> dims(d), ranks(d);
    ts_result_dims(res, dims.data());
    ts_result_ranks(res, ranks.data());
    std::vector<Matrix> factors(d);
    for (size_t n = 0; n < d; ++n) {
        factors[n].resize(dims[n], ranks[n]);
        detail::check(ts_result_factor(res, static_cast<int64_t>(n), factors[n].data()));
    }
    DenseTensor core(std::vector<Index>(ranks.begin(), ranks.end()));
    detail::check(ts_result_core(res, core.data()));
    if (stats != nullptr) {
        stats->plan = p;
        stats->has_plan = true;
    }
    return TuckerTensor(std::move(core), std::move(factors));
}

// Drop-in dispatcher: Strategy::Krp goes to the B200; the others stay on the CPU.
inline TuckerTensor round_sum(const SumRequest& req, const SketchPlan* plan = nullptr, SumStats* stats = nullptr) {
    if (req.strategy == Strategy::Krp) return krp_sum(req, plan, stats);
    return tucksum::round_sum(req, plan, stats);
}

}  // namespace tucksum::cuda
