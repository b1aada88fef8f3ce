// Compile check of include/tucksum_cuda_adapter.hpp against the REAL reference
// headers (/root/reference/proj/include, -I first) with the Eigen shim in
// tests/cpp/eigen_shim: every adapter entry point is instantiated with the
// reference's own SumRequest / SketchPlan / SumStats / TuckerTensor types, so a
// signature drift between the adapter and include/tucksum/sketch.hpp:85-94 or
// tucker.hpp fails to compile (-Werror).  Syntax only: nothing is linked.
#include "tucksum_cuda_adapter.hpp"

using namespace tucksum;

int adapter_entry_points(const SumRequest& req, const TuckerTensor& x) {
    SumStats stats;
    TuckerTensor a = cuda::krp_sum(req, nullptr, &stats);
    TuckerTensor b = cuda::kron_sum(req, &stats.plan, nullptr);
    TuckerTensor c = cuda::round_sum(req, nullptr, &stats);
    TuckerTensor r = cuda::tucker_rounding(x, 1e-8);
    const double v = cuda::tucker_norm(a) + cuda::tucker_inner(b, c) + cuda::tucker_rel_error(r, x);
    // The drop-ins must be interchangeable with the reference's own entry points.
    TuckerTensor (*ref_krp)(const SumRequest&, const SketchPlan*, SumStats*) = &tucksum::krp_sum;
    TuckerTensor (*dev_krp)(const SumRequest&, const SketchPlan*, SumStats*) = &cuda::krp_sum;
    TuckerTensor (*ref_round)(const SumRequest&, const SketchPlan*, SumStats*) = &tucksum::round_sum;
    TuckerTensor (*dev_round)(const SumRequest&, const SketchPlan*, SumStats*) = &cuda::round_sum;
    double (*ref_norm)(const TuckerTensor&) = &tucksum::tucker_norm;
    double (*dev_norm)(const TuckerTensor&) = &cuda::tucker_norm;
    (void)ref_krp, (void)dev_krp, (void)ref_round, (void)dev_round, (void)ref_norm, (void)dev_norm;
    return v > 0.0 ? 0 : 1;
}
