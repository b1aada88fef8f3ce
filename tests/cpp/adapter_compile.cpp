// Compile check of include/tucksum_cuda_adapter.hpp against tests/cpp/stub (the
// reference's public types without Eigen).  Instantiates every adapter entry point.
#include "tucksum_cuda_adapter.hpp"

namespace tucksum {
TuckerTensor formal_sum(const std::vector<const TuckerTensor*>& xs, const std::vector<double>&) { return *xs[0]; }
TuckerTensor tucker_axby(double, const TuckerTensor& x, double, const TuckerTensor&) { return x; }
}  // namespace tucksum

using namespace tucksum;

int adapter_entry_points(const SumRequest& req, const TuckerTensor& x) {
    SumStats stats;
    TuckerTensor a = cuda::krp_sum(req, nullptr, &stats);
    TuckerTensor b = cuda::kron_sum(req, &stats.plan, nullptr);
    TuckerTensor c = cuda::round_sum(req, nullptr, &stats);
    TuckerTensor r = cuda::tucker_rounding(x, 1e-8);
    const double v = cuda::tucker_norm(a) + cuda::tucker_inner(b, c) + cuda::tucker_rel_error(r, x);
    return v > 0.0 ? 0 : 1;
}
