// Minimal stand-in for the reference's public types (include/tucksum/*.hpp),
// shaped like their Eigen-based originals, so tests can compile
// include/tucksum_cuda_adapter.hpp in an image without Eigen.  Test-only.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <vector>

namespace tucksum {
using Index = std::int64_t;
struct Matrix {
    Index r = 0, c = 0;
    std::vector<double> a;
    void resize(Index rows, Index cols) { r = rows; c = cols; a.assign(static_cast<size_t>(rows * cols), 0.0); }
    double* data() { return a.data(); }
    const double* data() const { return a.data(); }
};
struct DenseTensor {
    std::vector<Index> s;
    std::vector<double> a;
    DenseTensor() = default;
    explicit DenseTensor(std::vector<Index> shape) : s(std::move(shape)) {
        Index n = 1;
        for (Index x : s) n *= x;
        a.assign(static_cast<size_t>(n), 0.0);
    }
    const std::vector<Index>& shape() const { return s; }
    double* data() { return a.data(); }
    const double* data() const { return a.data(); }
};
struct CoreBlock {
    std::vector<Index> offsets;
    DenseTensor data;
};
struct RngSeed {
    std::uint64_t seed = 0, stream = 0;
};
class TuckerTensor {
public:
    TuckerTensor(DenseTensor core, std::vector<Matrix> factors) : f_(std::move(factors)) {
        for (auto& m : f_) { d_.push_back(m.r); r_.push_back(m.c); }
        b_.push_back(CoreBlock{std::vector<Index>(f_.size(), 0), std::move(core)});
    }
    Index order() const { return static_cast<Index>(f_.size()); }
    const std::vector<Index>& dims() const { return d_; }
    const std::vector<Index>& ranks() const { return r_; }
    const std::vector<Matrix>& factors() const { return f_; }
    const std::vector<CoreBlock>& blocks() const { return b_; }
private:
    std::vector<Index> d_, r_;
    std::vector<Matrix> f_;
    std::vector<CoreBlock> b_;
};
enum class Strategy { Lazy, Eager, Krp, Kron };
struct SumRequest {
    std::vector<const TuckerTensor*> summands;
    std::vector<double> weights;
    double eps = 1e-8;
    Index oversampling = 5;
    Strategy strategy = Strategy::Lazy;
    RngSeed seed{};
};
struct SketchPlan {
    Strategy strategy = Strategy::Krp;
    std::vector<Index> effective_ranks, oversampling, targets, mode_sketch_dims;
    double eps = 0.0;
    RngSeed seed{};
};
struct SumStats {
    std::vector<std::vector<Index>> eager_rank_trace;
    SketchPlan plan;
    bool has_plan = false;
};
// Declarations only (the adapter calls them in its Eager fold).
TuckerTensor formal_sum(const std::vector<const TuckerTensor*>& xs, const std::vector<double>& weights);
TuckerTensor tucker_axby(double alpha, const TuckerTensor& x, double beta, const TuckerTensor& y);
}  // namespace tucksum
