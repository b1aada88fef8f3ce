// capi.cu — C ABI (include/tucksum_cuda.h) and the host-side orchestration of
// the KRP sketched Tucker summation on one B200 (plus NCCL all-reduce across GPUs).
//
// Pipeline of ts_krp_sum (reference src/sketch.cpp:66-181, krp = true), with the
// summands stored once in the stacked formal-sum layout F_j = [U_j^(1) … U_j^(K)]:
//   A  Z_j = Ω_jᵀ F_j                       grouped TN DMMA GEMM      (sketch.cpp:108-112)
//   B  W_n[b] = w_b · G_b,(n) · ⊙_{j≠n} M_j  KRP generated in smem      (sketch.cpp:117-130)
//   C  Y_n = F_n W_n                         grouped NT DMMA GEMM (W stored transposed) (sketch.cpp:131)
//      all-reduce Y over GPUs (NCCL)
//   D  Û_n = thin Q(Y_n), R_ii >= 0          Householder TSQR          (sketch.cpp:145-150)
//   E  P_n = Û_nᵀ F_n                        grouped TN DMMA GEMM      (sketch.cpp:157-160)
//   F1 T_b = w_b · G_b ×_0 P_0,b ⋯ ×_{d-2}    grouped batched GEMMs     (sketch.cpp:161-166)
//   F2 h = [T_b]_b · P_{d-1}ᵀ                 NT DMMA GEMM (sum over b) (sketch.cpp:167)
//      all-reduce h over GPUs (NCCL)
//   G  st_hosvd(h, eps [, cap])              TSQR(R) + Jacobi SVD + TTM (tucker.cpp:239-283)
//   H  Ũ_n = Û_n P_n                          grouped NN DMMA GEMM      (sketch.cpp:172-175)
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <array>
#include <atomic>
#include <set>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <tuple>
#include <mutex>
#include <thread>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/tucksum_cuda.h"
#include "gemm.cuh"
#include "kernels.cuh"

namespace ts {
void substream(std::uint64_t seed, std::uint64_t stream, std::uint64_t salt, std::uint64_t* out_seed,
               std::uint64_t* out_stream);
void gaussian_fill(std::int64_t rows, std::int64_t cols, std::uint64_t seed, std::uint64_t stream, double* out);
}  // namespace ts

namespace {

thread_local std::string g_err;

// NCCL entry points resolved at run time (libnccl.so.2 — the copy torch already
// loaded when present), so the library has no link-time NCCL dependency.
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string error;
};

NcclApi& nccl_api() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.error = dlerror() ? dlerror() : "dlopen libnccl.so.2 failed";
            return;
        }
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
        api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(h, "ncclAllReduce"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
        api.CommCount = reinterpret_cast<decltype(api.CommCount)>(dlsym(h, "ncclCommCount"));
        api.CommUserRank = reinterpret_cast<decltype(api.CommUserRank)>(dlsym(h, "ncclCommUserRank"));
        if (!api.GetUniqueId || !api.CommInitRank || !api.AllReduce) api.error = "libnccl.so.2 lacks required symbols";
    });
    if (!api.error.empty()) throw ts::Error(TS_NCCL, "NCCL unavailable: " + api.error);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        const char* m = nccl_api().GetErrorString ? nccl_api().GetErrorString(r) : "?";
        throw ts::Error(TS_NCCL, std::string(what) + ": " + m);
    }
}

[[noreturn]] void invalid(const std::string& m) { throw ts::Error(TS_INVALID_ARGUMENT, m); }

template <class F>
int guarded(F fn) {
    try {
        fn();
        return TS_OK;
    } catch (const ts::Error& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return TS_OOM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return TS_RUNTIME;
    }
}

struct OmegaKey {
    std::uint64_t seed, stream;
    std::vector<std::int64_t> widths;  // per mode (uniform for the KRP sketch)
    std::vector<std::int64_t> dims;
    bool operator<(const OmegaKey& o) const {
        return std::tie(seed, stream, widths, dims) < std::tie(o.seed, o.stream, o.widths, o.dims);
    }
};

constexpr int kNumStages = 11;  // + two hook pairs: stage A's and stage C's GEMM kernel alone (before any reduce)

// One captured call (CUDA graph) of the speculative ε = 0 path: everything from
// stage A to the acceptance flags' download is replayed by one cudaGraphLaunch.
// The graph owns its descriptor staging (pinned, never reset after capture), a
// device weight buffer refreshed before each replay, and its output buffers,
// copied into fresh result buffers after each replay.
struct GraphKey {
    std::uint64_t batch;
    int method;
    std::vector<std::int64_t> widths, cap;
    std::uint64_t seed, stream;
    double eps;
    std::vector<double> weights;  // some launches take a weight as a host scalar (GEMM alpha)
    bool operator<(const GraphKey& o) const {
        return std::tie(batch, method, widths, cap, seed, stream, eps, weights) <
               std::tie(o.batch, o.method, o.widths, o.cap, o.seed, o.stream, o.eps, o.weights);
    }
};
struct GraphEntry {
    ts::HostStage stage;
    cudaGraphExec_t exec = nullptr;
    double* d_w = nullptr;   // device weights (count)
    double* h_w = nullptr;   // pinned staging of the weights
    std::int64_t count = 0;
    double* out_f[TS_MAX_ORDER] = {};
    double* out_core = nullptr;
    std::int64_t dims[TS_MAX_ORDER] = {}, ranks[TS_MAX_ORDER] = {};
    int order = 0;
    int* h_flags = nullptr;  // pinned: [0, 2d) stage-D / stage-G acceptance flags
    std::int64_t launches = 0;
    std::uint64_t last_use = 0;
    ~GraphEntry() {
        if (exec) cudaGraphExecDestroy(exec);
        if (d_w) cudaFree(d_w);
        if (h_w) cudaFreeHost(h_w);
        for (auto* f : out_f)
            if (f) cudaFree(f);
        if (out_core) cudaFree(out_core);
        if (h_flags) cudaFreeHost(h_flags);
    }
};

}  // namespace

struct OmegaEntry {
    double* ptr = nullptr;
    std::int64_t bytes = 0;
    std::uint64_t last_use = 0;
};

struct ts_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    // Side stream + fork/join events: stage D's CholeskyQR2 factor R runs on
    // `side` while stage E's GEMM runs on `stream` (see sketched_sum_impl).
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    int num_sms = 148;
    ts::HostStage stage;
    // Device Ω cache (shared with the lanes), bounded: least recently used
    // entries beyond kOmegaMaxEntries / kOmegaMaxBytes are freed (together with
    // the captured graphs that read them).
    std::map<OmegaKey, OmegaEntry> omega;
    // Ω_j pre-sliced for the int8 stage-A engine (ozaki.cu), keyed by the Ω_j
    // device pointer; released with its Ω entry.
    std::map<const double*, ts::OzOperand> oz_cache;
    std::int64_t omega_bytes = 0;
    std::uint64_t omega_clock = 0;
    std::uint64_t omega_pin = ~std::uint64_t(0);  // entries used at clock >= pin are never evicted
    ncclComm_t comm = nullptr;
    // Alternative exchange: a host all-reduce callback (e.g. gloo) — the same
    // sharded orchestration without NCCL, for CPU-interconnect or testing setups.
    ts_host_allreduce_fn host_ar = nullptr;
    void* host_ar_user = nullptr;
    int nranks = 1, rank = 0;
    bool debug = false, timing = false;
    std::vector<double> stage_ms;
    std::int64_t launches = 0;
    std::vector<cudaEvent_t> events;
    int last_qr_fallbacks = 0, last_svd_fallbacks = 0;  // accurate-path uses in the last call
    unsigned last_int8_stages = 0;  // bit 0/1/2/3: stage A/C/E/F2 of the last call ran on the int8 engine (ozaki.cu)
    bool f2_int8 = false;           // set by project_core when F2 took the int8 engine
    int last_eig_fallbacks = 0;  // tridiagonal-eigensolver rejections (Jacobi recomputes) in the last call
    // ST-HOSVD modes that needed the accurate path in the last synchronous call
    // with these sketch dims: the next such call goes there directly (a pure
    // performance hint — the accurate path is valid for every input; every 16th
    // call re-tries the fast path).
    std::vector<std::int64_t> hint_q;
    unsigned hint_accurate = 0;
    std::uint64_t hint_calls = 0;
    // Speculative tail (see krp_sum_impl): on while the last call needed no
    // accurate-path fallback.
    bool spec_ok = true;
    // ts_krp_sum_many: child contexts (own stream, staging, history) that share
    // this context's device and Ω cache; created on first use.
    ts_ctx* parent = nullptr;
    std::vector<ts_ctx*> lanes;
    std::mutex omega_mu;
    // CUDA-graph cache of repeated speculative calls (see GraphEntry).
    bool graphs = true;
    std::map<GraphKey, std::unique_ptr<GraphEntry>> graph_cache;
    std::set<GraphKey> graph_seen;
    std::uint64_t graph_clock = 0;
    std::int64_t graph_replays = 0;
};

struct ts_batch {
    ts_ctx* ctx = nullptr;
    int order = 0;
    std::int64_t dims[TS_MAX_ORDER] = {};
    std::int64_t count = 0;
    std::int64_t R[TS_MAX_ORDER] = {};  // stacked columns per mode
    double* F[TS_MAX_ORDER] = {};       // device n_j × R_j column-major
    double* cores = nullptr;
    std::int64_t core_elems = 0;
    std::vector<ts::Atom> atoms;
    ts::Atom* d_atoms = nullptr;
    std::vector<double> core_norm;  // per summand ‖core‖_F (plan energies)
    // First stacked column of summand i in mode j at scol[i*order + j]
    // (i = 0..count; row `count` holds R_j): the column segments of
    // ts_krp_sum_segmented.
    std::vector<std::int64_t> scol;
    int max_shape = 0;
    std::int64_t bytes = 0;
    std::uint64_t id = 0;  // unique per upload (graph-cache key; never reused)
    int* aexp[TS_MAX_ORDER] = {};  // per-column exponent bounds of F_j (Ozaki stages A/E), computed on first use
    int* rexp[TS_MAX_ORDER] = {};  // per-row exponent bounds of F_j (Ozaki stage C), computed on first use
};

struct ts_result {
    int order = 0;
    std::int64_t dims[TS_MAX_ORDER] = {}, ranks[TS_MAX_ORDER] = {};
    double* factors[TS_MAX_ORDER] = {};
    double* core = nullptr;
    int device = 0;
    cudaStream_t stream = nullptr;  // owning context's stream (stream-ordered alloc/free)
    // Debug intermediates (host copies).
    std::vector<double> inter[3][TS_MAX_ORDER];
    std::int64_t inter_rows[3][TS_MAX_ORDER] = {}, inter_cols[3][TS_MAX_ORDER] = {};
    std::vector<double> h;
    // Results of one segmented call live in one shared device block (one
    // allocation instead of (order + 1) per sum); freed with the last of them.
    std::shared_ptr<void> arena;
    ~ts_result() {
        if (arena) return;
        cudaSetDevice(device);
        for (auto* f : factors)
            if (f) cudaFreeAsync(f, stream);
        if (core) cudaFreeAsync(core, stream);
    }
};

namespace {

using ts::CallScratch;
using ts::GemmProblem;
using ts::Layout;

// Ω_n = gaussian_matrix(dims[n], widths[n], {seed, stream}.substream(n)), all
// modes concatenated (column-major each), cached on the device.
constexpr size_t kOmegaMaxEntries = 64;
constexpr std::int64_t kOmegaMaxBytes = std::int64_t(1) << 30;

double* omega_get(ts_ctx* ctx, int order, const std::int64_t* dims, const std::int64_t* widths, std::uint64_t seed,
                  std::uint64_t stream) {
    if (ctx->parent) ctx = ctx->parent;  // lanes share the parent's cache
    std::lock_guard<std::mutex> lock(ctx->omega_mu);
    OmegaKey key{seed, stream, std::vector<std::int64_t>(widths, widths + order),
                 std::vector<std::int64_t>(dims, dims + order)};
    auto it = ctx->omega.find(key);
    if (it != ctx->omega.end()) {
        it->second.last_use = ++ctx->omega_clock;
        return it->second.ptr;
    }
    std::int64_t total = 0;
    for (int n = 0; n < order; ++n) total += dims[n] * widths[n];
    std::vector<double> host(static_cast<size_t>(total));
    std::int64_t off = 0;
    for (int n = 0; n < order; ++n) {
        std::uint64_t s2, t2;
        ts::substream(seed, stream, static_cast<std::uint64_t>(n), &s2, &t2);
        ts::gaussian_fill(dims[n], widths[n], s2, t2, host.data() + off);
        off += dims[n] * widths[n];
    }
    const std::int64_t bytes = static_cast<std::int64_t>(sizeof(double)) * std::max<std::int64_t>(total, 1);
    // Callers with a fresh seed per call (NDG steps, GMRES iterations) would
    // otherwise grow the cache without bound: evict least recently used entries.
    while (ctx->omega.size() + 1 > kOmegaMaxEntries || ctx->omega_bytes + bytes > kOmegaMaxBytes) {
        auto lru = ctx->omega.end();
        for (auto e = ctx->omega.begin(); e != ctx->omega.end(); ++e)
            if (e->second.last_use < ctx->omega_pin && (lru == ctx->omega.end() || e->second.last_use < lru->second.last_use))
                lru = e;
        if (lru == ctx->omega.end()) break;  // everything is in use by a running ts_krp_sum_many
        // Work queued on this context or its lanes may still read it.
        TS_CUDA_CHECK(cudaDeviceSynchronize());
        for (auto g = ctx->graph_cache.begin(); g != ctx->graph_cache.end();)
            g = (g->first.seed == lru->first.seed && g->first.stream == lru->first.stream) ? ctx->graph_cache.erase(g)
                                                                                         : std::next(g);
        {  // its pre-sliced copies go with it
            const double* lo = lru->second.ptr;
            const double* hi = lo + lru->second.bytes / static_cast<std::int64_t>(sizeof(double));
            for (auto c = ctx->oz_cache.begin(); c != ctx->oz_cache.end();)
                if (c->first >= lo && c->first < hi) {
                    cudaFree(c->second.slices);
                    cudaFree(c->second.exp);
                    c = ctx->oz_cache.erase(c);
                } else {
                    ++c;
                }
        }
        TS_CUDA_CHECK(cudaFree(lru->second.ptr));
        ctx->omega_bytes -= lru->second.bytes;
        ctx->omega.erase(lru);
    }
    double* d = nullptr;
    TS_CUDA_CHECK(cudaMalloc(&d, static_cast<size_t>(bytes)));
    TS_CUDA_CHECK(cudaMemcpy(d, host.data(), sizeof(double) * static_cast<size_t>(total), cudaMemcpyHostToDevice));
    ctx->omega.emplace(std::move(key), OmegaEntry{d, bytes, ++ctx->omega_clock});
    ctx->omega_bytes += bytes;
    return d;
}

bool sharded(const ts_ctx* ctx) { return ctx->comm != nullptr || ctx->host_ar != nullptr; }

// Sum `buf` (device, count doubles) over the ranks, in place, ordered on `st`:
// ncclAllReduce on the library stream, or the host callback (D2H, callback, H2D).
void allreduce_sum(ts_ctx* ctx, double* buf, std::int64_t count, cudaStream_t st, const char* what) {
    if (ctx->comm) {
        nccl_check(nccl_api().AllReduce(buf, buf, static_cast<size_t>(count), ncclFloat64, ncclSum, ctx->comm, st), what);
    } else if (ctx->host_ar) {
        std::vector<double> h(static_cast<size_t>(count));
        TS_CUDA_CHECK(cudaMemcpyAsync(h.data(), buf, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, st));
        TS_CUDA_CHECK(cudaStreamSynchronize(st));
        if (ctx->host_ar(ctx->host_ar_user, h.data(), count) != 0)
            throw ts::Error(TS_NCCL, std::string(what) + ": host all-reduce callback failed");
        TS_CUDA_CHECK(cudaMemcpyAsync(buf, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, st));
        TS_CUDA_CHECK(cudaStreamSynchronize(st));
    }
}

void mark(ts_ctx* ctx, int idx) {
    if (ctx->timing && static_cast<size_t>(idx) < ctx->events.size())
        TS_CUDA_CHECK(cudaEventRecord(ctx->events[static_cast<size_t>(idx)], ctx->stream));
}

void copy_to_host(std::vector<double>& dst, const double* src, std::int64_t n, cudaStream_t st) {
    dst.resize(static_cast<size_t>(n));
    if (n > 0) TS_CUDA_CHECK(cudaMemcpyAsync(dst.data(), src, sizeof(double) * static_cast<size_t>(n),
                                             cudaMemcpyDeviceToHost, st));
}

// Reference rank rule of st_hosvd (src/tucker.cpp:255-276) + optional cap.
std::int64_t hosvd_rank(const std::vector<double>& s, double tau, double theta, std::int64_t cap) {
    const std::int64_t count = static_cast<std::int64_t>(s.size());
    std::int64_t rank = 1;
    if (tau == 0.0) {
        const double floor = 1e-14 * s[0];
        rank = count;
        while (rank > 1 && s[static_cast<size_t>(rank - 1)] <= floor) --rank;
    } else {
        std::vector<double> suffix(static_cast<size_t>(count) + 1, 0.0);
        for (std::int64_t j = count - 1; j >= 0; --j)
            suffix[static_cast<size_t>(j)] = suffix[static_cast<size_t>(j) + 1] + s[static_cast<size_t>(j)] * s[static_cast<size_t>(j)];
        rank = count;
        for (std::int64_t r = 1; r <= count; ++r)
            if (suffix[static_cast<size_t>(r)] <= theta) {
                rank = r;
                break;
            }
    }
    if (cap > 0) rank = std::min(rank, cap);
    return rank;
}

// Accurate path: left singular vectors + singular values of the unfolding
// g_(k) (q_k × rest) from X = g_(k)ᵀ via TSQR (R only) and a one-sided Jacobi SVD
// of the small triangular factor.  X is overwritten.
void unfolding_svd_accurate(double* X, std::int64_t rest, std::int64_t qk, double* sigma, double* U, CallScratch& sc,
                            int num_sms) {
    if (qk > ts::max_tsqr_cols()) {  // any width: block one-sided Jacobi on X itself (wide.cu)
        ts::bosj_svd(X, rest, rest, qk, sigma, U, qk, sc, num_sms);
        return;
    }
    ts::TsqrPlan plan = ts::plan_tsqr(X, rest, rest, qk, nullptr, 0, sc);
    ts::run_tsqr({&plan}, sc, false);
    ts::launch_jacobi_svd(plan.Rtop, plan.kk, static_cast<int>(plan.kk), static_cast<int>(qk), sigma, U, sc);
}

// Symmetric eigensolver of the Gram fast paths (reference sym_eig,
// src/kernels.cpp:70-86) for any n: the one-CTA Jacobi (eig.cu / kernels.cu)
// up to 96, beyond that the block one-sided Jacobi of the (PSD) Gram itself,
// whose singular values are its eigenvalues (wide.cu).
void sym_eig_any(const double* C, std::int64_t n, double* lambda, double* V, CallScratch& sc, int num_sms,
                 int* sweeps = nullptr) {
    if (n <= ts::max_tsqr_cols()) {
        ts::launch_sym_jacobi(C, n, static_cast<int>(n), lambda, V, sc, sweeps);
        return;
    }
    ts::bosj_svd(C, n, n, n, lambda, V, n, sc, num_sms);
}

// Stage-D thin Q of a mode the CholeskyQR2 fast path does not take, for any
// width: widths ≤ 96 are planned into one batched Householder TSQR (Y is
// overwritten), wider ones go through wide.cu's BCGS2 (Y is kept).
bool qr_wide_mode(std::int64_t cols) { return cols > ts::max_tsqr_cols(); }

// Stages A and E (C = Sᵀ F_n with a skinny S of ≤ 64 columns: Ω_n, Y_n or Û_n)
// on the int8 tensor cores (ozaki.cu) when the stacked factors are large enough
// for the HBM-bound engine to beat the DMMA one (config 5: 0.55 vs 0.77 ms per
// stage); small sums stay on DMMA (latency).  TS_OZAKI=0 disables it.
bool ozaki_worth(const ts_batch* b) {
    if (!ts::ozaki_enabled()) return false;
    double bytes = 0.0;
    for (int n = 0; n < b->order; ++n) bytes += 8.0 * static_cast<double>(b->dims[n]) * static_cast<double>(b->R[n]);
    return bytes >= 256e6;
}

// ps[i] = {A = S (K × M, M ≤ 64), B = F_{modes[i]}, C (M × R)}; false (nothing
// launched) when a problem does not fit — the caller then runs the DMMA GEMM.
bool ozaki_stage(ts_ctx* ctx, const ts_batch* b, const std::vector<GemmProblem>& ps, const std::vector<int>& modes,
                 CallScratch& sc, bool cached_small = false) {
    if (!ozaki_worth(b)) return false;
    for (size_t i = 0; i < ps.size(); ++i) {
        const GemmProblem& p = ps[i];
        const int n = modes[i];
        if (p.M > 64 || p.B != b->F[n] || p.ldb != b->dims[n] || p.N != b->R[n] || p.alpha != 1.0 || p.beta != 0.0 ||
            p.batch != 1)
            return false;
    }
    auto* bm = const_cast<ts_batch*>(b);
    for (int n = 0; n < b->order; ++n)
        if (!bm->aexp[n] && b->R[n] > 0) {  // once per upload (first call, never inside a graph capture)
            TS_CUDA_CHECK(cudaMallocAsync(&bm->aexp[n], sizeof(int) * static_cast<size_t>(b->R[n]), sc.stream()));
            ts::launch_col_exponents(b->F[n], b->dims[n], b->dims[n], b->R[n], bm->aexp[n], sc);
        }
    std::vector<ts::OzOperand> small;
    if (!cached_small) {  // one launch slices every mode's skinny operand
        std::vector<ts::OzSmall> reqs;
        for (const GemmProblem& p : ps) reqs.push_back(ts::OzSmall{p.A, p.lda, p.K, p.M, false});
        small = ts::prepare_ozaki_b_batch(reqs, sc);
    }
    std::vector<ts::OzProblem> oz;
    for (size_t i = 0; i < ps.size(); ++i) {
        const GemmProblem& p = ps[i];
        const int n = modes[i];
        ts::OzProblem q{};
        q.F = b->F[n];
        q.ldf = b->dims[n];
        q.aexp = b->aexp[n];
        q.M = static_cast<int>(b->R[n]);
        q.K = p.K;
        if (cached_small) {  // Ω_j: sliced once, kept with the Ω cache
            ts_ctx* owner = ctx->parent ? ctx->parent : ctx;
            std::lock_guard<std::mutex> lock(owner->omega_mu);
            auto it = owner->oz_cache.find(p.A);
            if (it == owner->oz_cache.end() || it->second.K != p.K || it->second.N != p.M) {
                if (it != owner->oz_cache.end()) {
                    TS_CUDA_CHECK(cudaStreamSynchronize(sc.stream()));
                    cudaFree(it->second.slices);
                    cudaFree(it->second.exp);
                    owner->oz_cache.erase(it);
                }
                ts::OzOperand o{};
                o.K = p.K;
                o.N = p.M;
                TS_CUDA_CHECK(cudaMalloc(&o.slices, ts::ozaki_b_bytes(p.K)));
                TS_CUDA_CHECK(cudaMalloc(&o.exp, sizeof(int) * 64));
                ts::prepare_ozaki_b_into(p.A, p.lda, p.K, p.M, o, sc);
                it = owner->oz_cache.emplace(p.A, o).first;
            }
            q.B = it->second;
        } else {
            q.B = small[i];
        }
        q.C = p.C;
        q.ldc = p.ldc;
        oz.push_back(q);
    }
    int launched = 0;
    return ts::launch_ozaki_gemm(oz, sc, ctx->num_sms, &launched);
}

// Stage C (Y_n = F_n W_n with W_n stored transposed, ≤ 64 columns) on the same
// engine in its M-contiguous orientation: per-row exponent bounds of F_n.
bool ozaki_stage_c(ts_ctx* ctx, const ts_batch* b, const std::vector<GemmProblem>& ps, CallScratch& sc) {
    if (!ozaki_worth(b)) return false;
    for (size_t n = 0; n < ps.size(); ++n) {
        const GemmProblem& p = ps[n];
        if (p.N > 64 || p.A != b->F[n] || p.lda != b->dims[n] || p.K != b->R[n] || p.alpha != 1.0 || p.beta != 0.0 ||
            p.batch != 1)
            return false;
    }
    auto* bm = const_cast<ts_batch*>(b);
    for (int n = 0; n < b->order; ++n)
        if (!bm->rexp[n] && b->dims[n] > 0) {  // once per upload (first call, never inside a graph capture)
            TS_CUDA_CHECK(cudaMallocAsync(&bm->rexp[n], sizeof(int) * static_cast<size_t>(b->dims[n]), sc.stream()));
            ts::launch_row_exponents(b->F[n], b->dims[n], b->dims[n], b->R[n], bm->rexp[n], sc);
        }
    std::vector<ts::OzSmall> reqs;
    for (const GemmProblem& p : ps) reqs.push_back(ts::OzSmall{p.B, p.ldb, p.K, p.N, true});
    const std::vector<ts::OzOperand> small = ts::prepare_ozaki_b_batch(reqs, sc);
    std::vector<ts::OzProblem> oz;
    for (size_t n = 0; n < ps.size(); ++n) {
        const GemmProblem& p = ps[n];
        ts::OzProblem q{};
        q.F = b->F[n];
        q.ldf = b->dims[n];
        q.aexp = b->rexp[n];
        q.M = p.M;
        q.K = p.K;
        q.B = small[n];
        q.C = p.C;
        q.ldc = p.ldc;
        q.a_mn = true;
        q.c_colmajor = true;
        oz.push_back(q);
    }
    int launched = 0;
    return ts::launch_ozaki_gemm(oz, sc, ctx->num_sms, &launched);
}

// Fast path of the ST-HOSVD rank decision from the eigenvalues lam (descending)
// of the Gram h_(k)h_(k)ᵀ.  The Gram's eigenvalues carry absolute errors of a few
// ulps of λ₁, so the decision (and the kept subspace) is accepted only when it is
// provably the one the exact singular values give; otherwise *ok = false and the
// caller takes the accurate TSQR + one-sided Jacobi path.
std::int64_t gram_rank(const std::vector<double>& lam_in, double tau, double theta, std::int64_t cap, double resid,
                       bool* ok) {
    *ok = false;
    const std::int64_t q = static_cast<std::int64_t>(lam_in.size());
    if (q == 0 || !(lam_in[0] > 0.0)) return 1;
    std::vector<double> lam(lam_in);
    for (double& l : lam) l = std::max(l, 0.0);
    const double l1 = lam[0];
    const double noise = 1e-12 * l1;
    const double resolvable = 1e-8 * l1;  // σ ≥ 1e-4·σ₁: far above both noise and the 1e-14·σ₁ floor
    std::int64_t rank;
    if (tau == 0.0) {
        if (cap > 0 && cap < q) {
            if (lam[static_cast<size_t>(cap - 1)] < resolvable) return 1;
            rank = cap;
        } else {
            if (lam[static_cast<size_t>(q - 1)] < resolvable) return 1;
            rank = q;
        }
    } else {
        std::vector<double> suffix(static_cast<size_t>(q) + 1, 0.0);
        for (std::int64_t j = q - 1; j >= 0; --j) suffix[static_cast<size_t>(j)] = suffix[static_cast<size_t>(j) + 1] + lam[static_cast<size_t>(j)];
        std::int64_t r = q;
        for (std::int64_t i = 1; i <= q; ++i)
            if (suffix[static_cast<size_t>(i)] <= theta) {
                r = i;
                break;
            }
        const double margin = static_cast<double>(q) * noise;
        if (r < q && suffix[static_cast<size_t>(r)] > theta - margin) return 1;
        if (r > 1 && suffix[static_cast<size_t>(r - 1)] <= theta + margin) return 1;
        rank = r;
        if (cap > 0) rank = std::min(rank, cap);
    }
    if (rank < q) {  // the kept subspace must be well separated from the discarded one
        const double gap = lam[static_cast<size_t>(rank - 1)] - lam[static_cast<size_t>(rank)];
        if (!(gap > 0.0)) return 1;
        // Eigenvector error of the kept subspace ≲ residual / gap, with the
        // solver's measured ‖C V − VΛ‖_F (resid ≥ 0) or the Jacobi solver's
        // off(C) ≤ 1e-14·‖C‖; its effect on the truncated tensor is damped by
        // σ_{r+1}/σ₁.  Require it 10× below the 1e-10 parity bar.  (Same
        // arithmetic as the device twins in kernels.cu.)
        const double rabs = resid >= 0.0 ? std::max(resid, 1e-16 * l1) : 1e-14 * l1;
        const double err = rabs / gap * std::sqrt(lam[static_cast<size_t>(rank)] / l1);
        if (err > 1e-11) return 1;
    }
    *ok = true;
    return rank;
}

// Π_{j≠skip} v_j, saturating at 2^50 (reference complement_product, src/sketch.cpp).
std::int64_t complement_product(const std::int64_t* v, int order, int skip) {
    const std::int64_t cap = std::int64_t(1) << 50;
    std::int64_t prod = 1;
    for (int j = 0; j < order; ++j) {
        if (j == skip) continue;
        const std::int64_t f = std::max<std::int64_t>(v[j], 1);
        if (prod > cap / f) return cap;
        prod *= f;
    }
    return prod;
}

// Stage B of the Kron sketch (src/sketch.cpp:132-140): every atom's core block
// is multiplied by M_j = Ω_jᵀU_j (its column slice of Z_j, ow_j × r_j) in every
// mode j ≠ n, ascending — one grouped batched DMMA GEMM launch over all atoms per
// step — and the gather writes w_b·unfold(V, n)ᵀ into Wt_n (C_n × R_n).
void kron_stage_b(const ts_batch* b, double* const* Z, const std::int64_t* ow, double* const* Wt,
                  const std::int64_t* yc, const double* d_w, CallScratch& sc, int num_sms) {
    const int d = b->order;
    const size_t na = b->atoms.size();
    for (int n = 0; n < d; ++n) {
        std::vector<const double*> cur(na);
        std::vector<std::array<std::int64_t, TS_MAX_ORDER>> shp(na);
        for (size_t a = 0; a < na; ++a) {
            cur[a] = b->cores + b->atoms[a].core_off;
            for (int j = 0; j < d; ++j) shp[a][static_cast<size_t>(j)] = b->atoms[a].shape[j];
        }
        for (int m = 0; m < d; ++m) {
            if (m == n) continue;
            std::vector<std::int64_t> outoff(na);
            std::int64_t tot = 0;
            for (size_t a = 0; a < na; ++a) {
                std::int64_t e = ow[m];
                for (int j = 0; j < d; ++j)
                    if (j != m) e *= shp[a][static_cast<size_t>(j)];
                outoff[a] = tot;
                tot += e;
            }
            double* outbuf = sc.alloc_n<double>(static_cast<size_t>(std::max<std::int64_t>(tot, 1)));
            std::vector<GemmProblem> ps;
            ps.reserve(na);
            for (size_t a = 0; a < na; ++a) {
                const ts::Atom& at = b->atoms[a];
                std::int64_t left = 1, right = 1;
                for (int j = 0; j < m; ++j) left *= shp[a][static_cast<size_t>(j)];
                for (int j = m + 1; j < d; ++j) right *= shp[a][static_cast<size_t>(j)];
                const std::int64_t rm = shp[a][static_cast<size_t>(m)];
                double* out = outbuf + outoff[a];
                GemmProblem p{};
                if (m == 0) {
                    // out (ow_0 × right) = M_0 (ow_0 × r_0) · T (r_0 × right)
                    p.A = Z[0] + static_cast<std::int64_t>(at.col[0]) * ow[0];
                    p.lda = ow[0];
                    p.B = cur[a];
                    p.ldb = rm;
                    p.C = out;
                    p.ldc = ow[0];
                    p.M = static_cast<int>(ow[0]);
                    p.N = static_cast<int>(right);
                    p.K = static_cast<int>(rm);
                } else {
                    // per right slice: out (left × ow_m) = T (left × r_m) · M_mᵀ
                    p.A = cur[a];
                    p.lda = left;
                    p.sA = left * rm;
                    p.B = Z[m] + static_cast<std::int64_t>(at.col[m]) * ow[m];
                    p.ldb = ow[m];
                    p.sB = 0;
                    p.C = out;
                    p.ldc = left;
                    p.sC = left * ow[m];
                    p.M = static_cast<int>(left);
                    p.N = static_cast<int>(ow[m]);
                    p.K = static_cast<int>(rm);
                    p.batch = static_cast<int>(right);
                }
                ps.push_back(p);
                cur[a] = out;
                shp[a][static_cast<size_t>(m)] = ow[m];
            }
            ts::launch_grouped_gemm(m == 0 ? Layout::NN : Layout::NT, ps, sc, num_sms);
        }
        std::vector<ts::KronGather> g(na);
        for (size_t a = 0; a < na; ++a) {
            std::int64_t L = 1;
            for (int j = 0; j < n; ++j) L *= shp[a][static_cast<size_t>(j)];
            g[a] = ts::KronGather{cur[a], L, b->atoms[a].shape[n], b->atoms[a].col[n], b->atoms[a].summand, 0};
        }
        ts::launch_kron_gather(g, yc[n], Wt[n], d_w, sc);
    }
}

// Stages F1 + F2 (src/sketch.cpp:152-169): h = Σ_atoms w_b · G_b ×_n P_n[:, cols_b]
// for given projections P_n (q_n × R_n, ld q_n).  Order 3 fuses the chain per
// core slice (ttm3.cu); other orders run a per-atom grouped GEMM chain.  The sum
// over atoms is the K dimension of the final GEMM (deterministic split-K).
double* project_core_f1(ts_ctx* ctx, const ts_batch* b, double* const* P, const std::int64_t* q, const double* d_w,
                        const double* weights, CallScratch& sc, int** rowexp = nullptr) {
    const int d = b->order;
    // ---- Stage F1: per-atom multi-TTM over modes 0..d-2 into T_stack (Q' × R_{d-1})
    std::int64_t Qp = 1;
    for (int j = 0; j < d - 1; ++j) Qp *= q[j];
    double* Tstack = sc.alloc_n<double>(static_cast<size_t>(Qp * b->R[d - 1]));
    bool f1_done = false;
    if (d == 3) {  // fused per-slice chain (ttm3.cu)
        ts::Ttm3Args ta{};
        for (int n = 0; n < d; ++n) {
            ta.P[n] = P[n];
            ta.q[n] = q[n];
        }
        ta.atoms = b->d_atoms;
        ta.cores = b->cores;
        ta.weights = d_w;
        ta.Tstack = Tstack;
        ta.Qp = Qp;
        ta.natoms = static_cast<int>(b->atoms.size());
        int max_r2 = 0;
        for (const auto& at : b->atoms) max_r2 = std::max(max_r2, at.shape[2]);
        if (rowexp) {  // row exponent bounds of T_stack for F2 on the int8 engine
            ta.rowexp = sc.alloc_n<int>(static_cast<size_t>(Qp * ts::kTtmExpBuckets));
            ts::launch_fill_exponents(ta.rowexp, Qp * ts::kTtmExpBuckets, sc);
        }
        f1_done = ts::launch_ttm3(ta, b->max_shape, max_r2, sc);
        if (rowexp && f1_done) ts::launch_reduce_exponents(ta.rowexp, Qp, ts::kTtmExpBuckets, sc);
        if (rowexp) *rowexp = f1_done ? ta.rowexp : nullptr;
    } else if (rowexp) {
        *rowexp = nullptr;
    }
    if (!f1_done) {
        const size_t na = b->atoms.size();
        std::vector<double*> cur(na), nxt(na);
        for (int m = 0; m <= d - 2; ++m) {
            const bool last = (m == d - 2);
            double* outbuf = nullptr;
            std::vector<std::int64_t> outoff(na);
            if (!last) {
                std::int64_t tot = 0;
                for (size_t a = 0; a < na; ++a) {
                    std::int64_t e = 1;
                    for (int j = 0; j <= m; ++j) e *= q[j];
                    for (int j = m + 1; j < d; ++j) e *= b->atoms[a].shape[j];
                    outoff[a] = tot;
                    tot += e;
                }
                outbuf = sc.alloc_n<double>(static_cast<size_t>(tot));
            }
            std::vector<GemmProblem> ps;
            ps.reserve(na);
            for (size_t a = 0; a < na; ++a) {
                const ts::Atom& at = b->atoms[a];
                double* out = last ? Tstack + static_cast<std::int64_t>(at.col[d - 1]) * Qp : outbuf + outoff[a];
                const double alpha = last ? weights[at.summand] : 1.0;
                std::int64_t left = 1, right = 1;
                for (int j = 0; j < m; ++j) left *= q[j];
                for (int j = m + 1; j < d; ++j) right *= at.shape[j];
                GemmProblem p{};
                p.alpha = alpha;
                if (m == 0) {
                    // out (q0 × right) = P_0[:, cols] (q0 × r0) · G_(0) (r0 × right)
                    p.A = P[0] + static_cast<std::int64_t>(at.col[0]) * q[0];
                    p.lda = q[0];
                    p.B = b->cores + at.core_off;
                    p.ldb = at.shape[0];
                    p.C = out;
                    p.ldc = q[0];
                    p.M = static_cast<int>(q[0]);
                    p.N = static_cast<int>(right);
                    p.K = at.shape[0];
                } else {
                    // per right slice: out (left × q_m) = T (left × r_m) · P_m[:, cols]ᵀ
                    p.A = cur[a];
                    p.lda = left;
                    p.sA = left * at.shape[m];
                    p.B = P[m] + static_cast<std::int64_t>(at.col[m]) * q[m];
                    p.ldb = q[m];
                    p.sB = 0;
                    p.C = out;
                    p.ldc = left;
                    p.sC = left * q[m];
                    p.M = static_cast<int>(left);
                    p.N = static_cast<int>(q[m]);
                    p.K = at.shape[m];
                    p.batch = static_cast<int>(right);
                }
                ps.push_back(p);
                nxt[a] = out;
            }
            ts::launch_grouped_gemm(m == 0 ? Layout::NN : Layout::NT, ps, sc, ctx->num_sms);
            std::swap(cur, nxt);
        }
    }
    return Tstack;
}

double* project_core(ts_ctx* ctx, const ts_batch* b, double* const* P, const std::int64_t* q, const double* d_w,
                     const double* weights, CallScratch& sc, std::int64_t* hsize) {
    const int d = b->order;
    std::int64_t Qp = 1;
    for (int j = 0; j < d - 1; ++j) Qp *= q[j];
    // F2 on the int8 engine (ozaki.cu, stage-C orientation: T_stack is M-contiguous),
    // with F1 tracking T_stack's row exponent bounds.  Measured at config 5 (268 MB
    // T_stack): F2 0.150 -> 0.117 ms, but the tracking (32 exponent atomics per
    // thread at the end of each 8-slice CTA) costs F1 0.158 -> 0.198 ms, so it is
    // opt-in (TS_OZAKI_F2=1) and F2 stays on the DMMA GEMM by default.
    ctx->f2_int8 = false;
    static const bool f2_opt_in = [] {
        const char* e = std::getenv("TS_OZAKI_F2");
        return e && e[0] == '1';
    }();
    const bool f2_int8 = f2_opt_in && ts::ozaki_enabled() && q[d - 1] <= 64 && (Qp & 1) == 0 &&
                         8.0 * static_cast<double>(Qp) * static_cast<double>(b->R[d - 1]) >= 128e6;
    int* rowexp = nullptr;
    double* Tstack = project_core_f1(ctx, b, P, q, d_w, weights, sc, f2_int8 ? &rowexp : nullptr);
    mark(ctx, 7);
    // ---- Stage F2: h (Q' × q_{d-1}) = T_stack · P_{d-1}ᵀ
    *hsize = Qp * q[d - 1];
    double* h = sc.alloc_n<double>(static_cast<size_t>(*hsize));
    bool f2_done = false;
    if (rowexp) {
        ts::OzProblem o{};
        o.F = Tstack;
        o.ldf = Qp;
        o.aexp = rowexp;
        o.M = static_cast<int>(Qp);
        o.K = static_cast<int>(b->R[d - 1]);
        o.B = ts::prepare_ozaki_b_batch({ts::OzSmall{P[d - 1], q[d - 1], o.K, static_cast<int>(q[d - 1]), true}}, sc)[0];
        o.C = h;
        o.ldc = Qp;
        o.a_mn = true;
        o.c_colmajor = true;
        int launched = 0;
        f2_done = ts::launch_ozaki_gemm({o}, sc, ctx->num_sms, &launched);
        if (f2_done) ctx->f2_int8 = true;
    }
    if (!f2_done) {
        GemmProblem p{};
        p.A = Tstack;
        p.lda = Qp;
        p.B = P[d - 1];
        p.ldb = q[d - 1];
        p.C = h;
        p.ldc = Qp;
        p.M = static_cast<int>(Qp);
        p.N = static_cast<int>(q[d - 1]);
        p.K = static_cast<int>(b->R[d - 1]);
        ts::launch_grouped_gemm(Layout::NT, {p}, sc, ctx->num_sms);
    }
    return h;
}

enum class Method { Krp, Kron, Lazy };

// Σ_{a∈X, b∈Y} wX_a wY_b ⟨X_a, Y_b⟩ over the atoms of two device batches — the
// reference's tucker_inner (src/tucker.cpp:161-181) with weights, restated for the
// stacked layout: one cross-Gram per mode, M_n = F^Xᵀ_n F^Y_n (one grouped DMMA
// GEMM), then per atom a of X the rows of M_n that belong to it act as stage-E
// projections: h_a = Σ_b wY_b G_b ×_n M_n[a, b] (stage F kernels), and
// ⟨G_a, h_a⟩ is accumulated in atom order (deterministic).
double inner_impl(ts_ctx* ctx, const ts_batch* X, const double* wX, const ts_batch* Y, const double* wY) {
    if (!X || !Y || !wX || !wY) invalid("tucker_inner: null operand");
    if (X->order != Y->order) invalid("tucker_inner: operands must share dims");
    if (X->ctx->device != ctx->device || Y->ctx->device != ctx->device)
        invalid("tucker_inner: operands live on another device than this context's");
    const int d = X->order;
    for (int n = 0; n < d; ++n)
        if (X->dims[n] != Y->dims[n]) invalid("tucker_inner: operands must share dims");
    TS_CUDA_CHECK(cudaSetDevice(ctx->device));
    ctx->stage.reset();
    cudaStream_t st = ctx->stream;
    CallScratch sc(st, ctx->stage);
    auto* d_wY = static_cast<double*>(sc.upload(wY, sizeof(double) * static_cast<size_t>(Y->count)));
    double* M[TS_MAX_ORDER];
    {
        std::vector<GemmProblem> ps;
        for (int n = 0; n < d; ++n) {
            M[n] = sc.alloc_n<double>(static_cast<size_t>(X->R[n] * Y->R[n]));
            GemmProblem p{};
            p.A = X->F[n];
            p.lda = X->dims[n];
            p.B = Y->F[n];
            p.ldb = Y->dims[n];
            p.C = M[n];
            p.ldc = X->R[n];
            p.M = static_cast<int>(X->R[n]);
            p.N = static_cast<int>(Y->R[n]);
            p.K = static_cast<int>(X->dims[n]);
            ps.push_back(p);
        }
        ts::launch_grouped_gemm(Layout::TN, ps, sc, ctx->num_sms);
    }
    double* acc = sc.alloc_n<double>(1);
    TS_CUDA_CHECK(cudaMemsetAsync(acc, 0, sizeof(double), st));
    for (const ts::Atom& a : X->atoms) {
        CallScratch it(st, ctx->stage);  // per-atom buffers go back to the pool each iteration
        double* P[TS_MAX_ORDER];
        std::int64_t q[TS_MAX_ORDER];
        for (int n = 0; n < d; ++n) {
            q[n] = a.shape[n];
            P[n] = it.alloc_n<double>(static_cast<size_t>(q[n] * Y->R[n]));
            TS_CUDA_CHECK(cudaMemcpy2DAsync(P[n], sizeof(double) * static_cast<size_t>(q[n]), M[n] + a.col[n],
                                            sizeof(double) * static_cast<size_t>(X->R[n]),
                                            sizeof(double) * static_cast<size_t>(q[n]), static_cast<size_t>(Y->R[n]),
                                            cudaMemcpyDeviceToDevice, st));
        }
        std::int64_t hs = 0;
        double* h = project_core(ctx, Y, P, q, d_wY, wY, it, &hs);
        ts::launch_dot_accumulate(X->cores + a.core_off, h, hs, wX[a.summand], acc, it);
        sc.launches += it.launches;
    }
    double out = 0.0;
    TS_CUDA_CHECK(cudaMemcpyAsync(&out, acc, sizeof(double), cudaMemcpyDeviceToHost, st));
    TS_CUDA_CHECK(cudaStreamSynchronize(st));
    ctx->launches += sc.launches;
    return out;
}

// A result as a one-summand batch (non-owning view of its device factors and core).
struct ResultView {
    ts_batch b;
    explicit ResultView(ts_ctx* ctx, const ts_result* r) {
        b.ctx = ctx;
        b.order = r->order;
        b.count = 1;
        ts::Atom at{};
        std::int64_t core = 1;
        for (int n = 0; n < r->order; ++n) {
            b.dims[n] = r->dims[n];
            b.R[n] = r->ranks[n];
            b.F[n] = r->factors[n];
            at.col[n] = 0;
            at.shape[n] = static_cast<int>(r->ranks[n]);
            b.max_shape = std::max(b.max_shape, at.shape[n]);
            core *= r->ranks[n];
        }
        b.cores = r->core;
        b.core_elems = core;
        b.atoms.push_back(at);
        TS_CUDA_CHECK(cudaMallocAsync(&b.d_atoms, sizeof(ts::Atom), ctx->stream));
        TS_CUDA_CHECK(cudaMemcpyAsync(b.d_atoms, &b.atoms[0], sizeof(ts::Atom), cudaMemcpyHostToDevice, ctx->stream));
        TS_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    }
    ~ResultView() { cudaFreeAsync(b.d_atoms, b.ctx->stream); }
};

// Krp: krp_sum → sketched_sum(krp=true); Kron: kron_sum → sketched_sum(krp=false)
// (src/sketch.cpp:66-181,360-366).  The two differ in the Ω widths (uniform s vs
// plan widths), stage B and the sketch width of Y_n (s vs C_n = Π_{j≠n} s_j);
// everything from stage D on is shared.  Lazy: tucker_rounding(formal_sum(...))
// (src/sketch.cpp:48-50, src/tucker.cpp:132-159,285-296): the "sketch" Y_n is the
// stacked factor F_n itself (Y_n = F_n, no Ω, stages A-C skipped), so stage D is
// orthogonalize's QR of F_n, stage E gives its R factor (P_n = Q_nᵀF_n), stage F
// absorbs R into the block cores, and stages G/H are the rounding's st_hosvd and
// Q·P.  Needs Σ_k r_n^(k) ≤ 96.
ts_result* sketched_sum_impl(ts_ctx* ctx, const ts_batch* b, const double* weights, const std::int64_t* widths,
                             std::uint64_t seed, std::uint64_t stream, double eps, const std::int64_t* max_rank,
                             Method method, bool allow_spec = true, double* norm_out = nullptr,
                             GraphEntry* ge = nullptr) {
    const bool krp = method == Method::Krp, lazy = method == Method::Lazy;
    // Validation mirrors src/sketch.cpp:16-30,66-87.
    if (b == nullptr || b->count < 1) invalid("sum request needs matching, nonempty summands and weights");
    if (weights == nullptr) invalid("sum request needs matching, nonempty summands and weights");
    if (b->ctx->device != ctx->device) invalid("batch was uploaded to another device than this context's");
    if (!(eps >= 0.0)) invalid("tolerance must be nonnegative");
    const int d = b->order;
    if (d < 2) {
        if (lazy) throw ts::Error(TS_UNSUPPORTED, "lazy rounding of first-order tensors is not on the device path");
        invalid("sketched summation needs order >= 2");
    }
    std::int64_t s = 0;
    if (!lazy) {
        if (widths == nullptr) invalid("plan order does not match summand order");
        for (int n = 0; n < d; ++n)
            if (widths[n] < 1) invalid("plan sketch widths must be positive");
        s = *std::max_element(widths, widths + d);
    }
    std::int64_t ow[TS_MAX_ORDER], yc[TS_MAX_ORDER];  // Ω_n widths, Y_n widths
    for (int n = 0; n < d; ++n) {
        ow[n] = lazy ? 0 : krp ? s : widths[n];
        yc[n] = lazy ? b->R[n] : krp ? s : complement_product(widths, d, n);
    }
    for (std::int64_t i = 0; i < b->count; ++i)
        if (!std::isfinite(weights[i])) invalid("weights must be finite");

    TS_CUDA_CHECK(cudaSetDevice(ctx->device));
    ts::HostStage& hstage = ge ? ge->stage : ctx->stage;
    hstage.reset();
    cudaStream_t st = ctx->stream;
    CallScratch sc(st, hstage);
    const std::int64_t* dims = b->dims;
    if (ctx->timing && ctx->events.empty()) {
        ctx->events.resize(kNumStages + 5);
        for (auto& e : ctx->events) TS_CUDA_CHECK(cudaEventCreate(&e));
    }
    mark(ctx, 0);
    unsigned int8_stages = 0;

    double* omega = lazy ? nullptr : omega_get(ctx, d, dims, ow, seed, stream);
    std::int64_t q[TS_MAX_ORDER];
    std::int64_t ooff[TS_MAX_ORDER], yoff[TS_MAX_ORDER];
    std::int64_t ytot = 0, acc = 0;
    for (int n = 0; n < d; ++n) {
        q[n] = std::min(dims[n], yc[n]);
        ooff[n] = acc;
        acc += dims[n] * ow[n];
        yoff[n] = ytot;
        ytot += dims[n] * yc[n];
    }
    auto* d_w = ge ? ge->d_w : static_cast<double*>(sc.upload(weights, sizeof(double) * static_cast<size_t>(b->count)));

    double* Y = sc.alloc_n<double>(static_cast<size_t>(ytot));
    if (lazy) {
        // Y_n = F_n (copied: stage D factors its input in place).
        for (int n = 0; n < d; ++n)
            TS_CUDA_CHECK(cudaMemcpyAsync(Y + yoff[n], b->F[n], sizeof(double) * static_cast<size_t>(dims[n] * yc[n]),
                                          cudaMemcpyDeviceToDevice, st));
        mark(ctx, 1);
        sc.before_next_gemm = sc.after_next_gemm = nullptr;  // the hooks belong to stage A only
        mark(ctx, 2);
    } else {
        if (ctx->timing) {
        sc.before_next_gemm = ctx->events[kNumStages + 1];
        sc.after_next_gemm = ctx->events[kNumStages + 2];
    }
    // ---- Stage A: Z_j = Ω_jᵀ F_j (s × R_j)
        double* Z[TS_MAX_ORDER];
        {
            std::vector<GemmProblem> ps;
            for (int j = 0; j < d; ++j) {
                Z[j] = sc.alloc_n<double>(static_cast<size_t>(ow[j] * b->R[j]));
                GemmProblem p{};
                p.A = omega + ooff[j];
                p.lda = dims[j];
                p.B = b->F[j];
                p.ldb = dims[j];
                p.C = Z[j];
                p.ldc = ow[j];
                p.M = static_cast<int>(ow[j]);
                p.N = static_cast<int>(b->R[j]);
                p.K = static_cast<int>(dims[j]);
                ps.push_back(p);
            }
            std::vector<int> modes(static_cast<size_t>(d));
            std::iota(modes.begin(), modes.end(), 0);
            const bool a8 = ozaki_stage(ctx, b, ps, modes, sc, true);
            if (!a8) ts::launch_grouped_gemm(Layout::TN, ps, sc, ctx->num_sms);
            int8_stages |= a8 ? 1u : 0u;
        }
        mark(ctx, 1);
        sc.before_next_gemm = sc.after_next_gemm = nullptr;  // the hooks belong to stage A only
        // ---- Stage B: W_n (R_n × s), stored transposed
        double* W[TS_MAX_ORDER];
        if (!krp) {
            for (int n = 0; n < d; ++n) W[n] = sc.alloc_n<double>(static_cast<size_t>(b->R[n] * yc[n]));
            bool fused = false;
            if (d == 3) {  // one fused launch (kron3.cu)
                ts::Kron3Args ka{};
                for (int n = 0; n < 3; ++n) {
                    ka.Z[n] = Z[n];
                    ka.W[n] = W[n];
                    ka.s[n] = static_cast<int>(ow[n]);
                }
                ka.natoms = static_cast<int>(b->atoms.size());
                ka.atoms = b->d_atoms;
                ka.cores = b->cores;
                ka.weights = d_w;
                fused = ts::launch_kron3(ka, b->max_shape, sc);
            }
            if (!fused) kron_stage_b(b, Z, ow, W, yc, d_w, sc, ctx->num_sms);
        } else {
            ts::KrpArgs ka{};
            for (int n = 0; n < d; ++n) {
                W[n] = sc.alloc_n<double>(static_cast<size_t>(b->R[n] * s));
                ka.Z[n] = Z[n];
                ka.W[n] = W[n];
                ka.R[n] = b->R[n];
            }
            ka.order = d;
            ka.s = static_cast<int>(s);
            ka.natoms = static_cast<int>(b->atoms.size());
            ka.atoms = b->d_atoms;
            ka.cores = b->cores;
            ka.weights = d_w;
            ts::launch_krp_contract(ka, b->max_shape, sc);
        }
        mark(ctx, 2);
        if (ctx->timing) {  // stage C's GEMM kernel alone (the roofline kernel of bench.py)
            sc.before_next_gemm = ctx->events[kNumStages + 3];
            sc.after_next_gemm = ctx->events[kNumStages + 4];
        }
        // ---- Stage C: Y_n = F_n W_n (n × s), all modes in one buffer
        {
            std::vector<GemmProblem> ps;
            for (int n = 0; n < d; ++n) {
                GemmProblem p{};
                p.A = b->F[n];
                p.lda = dims[n];
                p.B = W[n];  // stored transposed: Wt_n (yc_n × R_n)
                p.ldb = yc[n];
                p.C = Y + yoff[n];
                p.ldc = dims[n];
                p.M = static_cast<int>(dims[n]);
                p.N = static_cast<int>(yc[n]);
                p.K = static_cast<int>(b->R[n]);
                ps.push_back(p);
            }
            const bool c8 = ozaki_stage_c(ctx, b, ps, sc);
            if (!c8) ts::launch_grouped_gemm(Layout::NT, ps, sc, ctx->num_sms);
            int8_stages |= c8 ? 2u : 0u;
            sc.before_next_gemm = sc.after_next_gemm = nullptr;  // the hooks belong to stage C only
        }
    }
    mark(ctx, 3);
    allreduce_sum(ctx, Y, ytot, st, "ncclAllReduce(Y)");
    mark(ctx, 4);
    auto res = std::make_unique<ts_result>();
    res->device = ctx->device;
    res->stream = st;
    res->order = d;
    if (ctx->debug) {
        for (int n = 0; n < d; ++n) {
            if (omega) copy_to_host(res->inter[0][n], omega + ooff[n], dims[n] * ow[n], st);
            res->inter_rows[0][n] = dims[n];
            res->inter_cols[0][n] = ow[n];
            copy_to_host(res->inter[1][n], Y + yoff[n], dims[n] * yc[n], st);
            res->inter_rows[1][n] = dims[n];
            res->inter_cols[1][n] = yc[n];
        }
    }
    // Speculative tail: the fast paths of stages D and G (CholeskyQR2; Gram +
    // Jacobi with the rank fixed by eps = 0 and the cap) are taken without
    // waiting for their acceptance checks, which run on the device; one sync at
    // the end reads them, and a rejected call is recomputed on the synchronous
    // path (identical results whenever the checks pass).  A context falls back
    // to the synchronous path while its last call needed an accurate path.
    const bool spec = allow_spec && ctx->spec_ok && !ctx->debug;
    int* dflags = nullptr;  // stage-D acceptance (CholQR2 pivots / second Gram)
    int* gflags = nullptr;  // stage-G acceptance (gram_rank checks)
    int* flags_all = nullptr;
    // ---- Stage D: Û_n = thin Q of Y_n.  Fast path CholeskyQR2 (Gram GEMM, small
    // Cholesky + inverse, GEMM, twice); R = R₂R₁ has a positive diagonal, so Û is
    // the Householder Q with R_ii ≥ 0 of the reference.  Modes whose Y is too
    // ill-conditioned (failed pivot, or second Gram far from I) or too short take
    // the Householder TSQR.
    // ---- Stages D + E.  Û_n = thin Q of Y_n (R_ii ≥ 0).  Fast path CholeskyQR2:
    // Gram, small Cholesky + inverse, Q₁ = Y R₁⁻¹, Gram, Cholesky + inverse, so
    // R = R₂R₁ has a positive diagonal and Û = Y R⁻¹ is the Householder Q with
    // R_ii ≥ 0 of the reference.  Û is never formed for such modes ("R form"):
    // stage E computes Pt_n = Y_nᵀF_n and P_n = R_n⁻ᵀPt_n (R_n⁻¹ = R₁⁻¹R₂⁻¹),
    // stage H Ũ_n = Y_n (R_n⁻¹P_k).  Because stage E's big GEMM needs only Y,
    // a speculative call whose modes all take CholeskyQR2 runs the R chain on
    // the side stream concurrently with it ("overlap"); the kernels and their
    // inputs are the same either way, so overlapped and synchronous results are
    // bitwise equal.  Modes whose Y is too ill-conditioned (failed pivot, second
    // Gram far from I) or too short take the Householder TSQR, which forms Û.
    double* Uh[TS_MAX_ORDER] = {};
    double* P[TS_MAX_ORDER];
    double* Rinv[TS_MAX_ORDER] = {};
    std::vector<int> rform(static_cast<size_t>(d), 0);
    bool overlap = spec && !lazy && !ctx->debug && !norm_out;
    for (int n = 0; n < d && overlap; ++n) overlap = dims[n] >= 2 * yc[n] && !qr_wide_mode(yc[n]);
    {
        std::vector<int>& chol = rform;
        // one block for both acceptance-flag sets (stage D: [0, d), stage G: [d, 2d)):
        // one memset and one download per call instead of two each
        int* flags = sc.alloc_n<int>(2 * static_cast<size_t>(d));
        TS_CUDA_CHECK(cudaMemsetAsync(flags, 0, 2 * sizeof(int) * static_cast<size_t>(d), st));
        flags_all = flags;
        bool any = false;
        for (int n = 0; n < d; ++n) {
            chol[static_cast<size_t>(n)] = dims[n] >= 2 * yc[n] && !qr_wide_mode(yc[n]);
            if (!chol[static_cast<size_t>(n)]) continue;
            any = true;
            Rinv[n] = sc.alloc_n<double>(static_cast<size_t>(yc[n] * yc[n]));
        }
        for (int n = 0; n < d; ++n) P[n] = sc.alloc_n<double>(static_cast<size_t>(q[n] * b->R[n]));
        if (overlap) {
            mark(ctx, 5);
            TS_CUDA_CHECK(cudaEventRecord(ctx->ev_fork, st));
            TS_CUDA_CHECK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
        }
        if (any) {
            CallScratch sd(overlap ? ctx->side : st, hstage);
            std::vector<GemmProblem> g1, q1, g2, rr;
            double *G1[TS_MAX_ORDER], *G2[TS_MAX_ORDER], *Ri1[TS_MAX_ORDER], *Ri2[TS_MAX_ORDER], *Q1[TS_MAX_ORDER];
            for (int n = 0; n < d; ++n) {
                if (!chol[static_cast<size_t>(n)]) continue;
                const std::int64_t c = yc[n];
                G1[n] = sd.alloc_n<double>(static_cast<size_t>(c * c));
                G2[n] = sd.alloc_n<double>(static_cast<size_t>(c * c));
                Ri1[n] = sd.alloc_n<double>(static_cast<size_t>(c * c));
                Ri2[n] = sd.alloc_n<double>(static_cast<size_t>(c * c));
                Q1[n] = sd.alloc_n<double>(static_cast<size_t>(dims[n] * c));
                GemmProblem p{};
                p.M = p.N = static_cast<int>(c);
                p.K = static_cast<int>(dims[n]);
                p.A = p.B = Y + yoff[n];
                p.lda = p.ldb = dims[n];
                p.C = G1[n];
                p.ldc = c;
                g1.push_back(p);
                p.A = p.B = Q1[n];
                p.C = G2[n];
                g2.push_back(p);
                GemmProblem m{};
                m.M = static_cast<int>(dims[n]);
                m.N = m.K = static_cast<int>(c);
                m.A = Y + yoff[n];
                m.lda = dims[n];
                m.B = Ri1[n];
                m.ldb = c;
                m.C = Q1[n];
                m.ldc = dims[n];
                q1.push_back(m);
                GemmProblem r{};
                r.M = r.N = r.K = static_cast<int>(c);
                r.A = Ri1[n];
                r.lda = c;
                r.B = Ri2[n];
                r.ldb = c;
                r.C = Rinv[n];
                r.ldc = c;
                rr.push_back(r);
            }
            // One Cholesky batch per distinct sketch width (all modes share it for
            // the KRP sketch).
            std::vector<std::int64_t> cw;
            for (int n = 0; n < d; ++n)
                if (chol[static_cast<size_t>(n)] && std::find(cw.begin(), cw.end(), yc[n]) == cw.end()) cw.push_back(yc[n]);
            auto chol_batches = [&](bool second) {
                for (std::int64_t c : cw) {
                    ts::CholBatch cb{};
                    int nb = 0;
                    for (int n = 0; n < d; ++n) {
                        if (!chol[static_cast<size_t>(n)] || yc[n] != c) continue;
                        cb.G[nb] = second ? G2[n] : G1[n];
                        cb.Rinv[nb] = second ? Ri2[n] : Ri1[n];
                        cb.flag[nb] = flags + n;
                        ++nb;
                    }
                    cb.ldg = cb.ldri = c;
                    cb.n = static_cast<int>(c);
                    cb.check_identity = second ? 1 : 0;
                    ts::launch_chol_inv(cb, nb, sd);
                }
            };
            ts::launch_grouped_gemm(Layout::TN, g1, sd, ctx->num_sms);
            chol_batches(false);
            ts::launch_grouped_gemm(Layout::NN, q1, sd, ctx->num_sms);
            ts::launch_grouped_gemm(Layout::TN, g2, sd, ctx->num_sms);
            chol_batches(true);
            ts::launch_grouped_gemm(Layout::NN, rr, sd, ctx->num_sms);
            for (std::int64_t c : cw) {  // κ(Y) small enough for the R form?
                ts::CholBatch cb{};
                int nb = 0;
                for (int n = 0; n < d; ++n) {
                    if (!chol[static_cast<size_t>(n)] || yc[n] != c) continue;
                    cb.G[nb] = G1[n];
                    cb.Rinv[nb] = Rinv[n];
                    cb.flag[nb] = flags + n;
                    ++nb;
                }
                cb.ldg = cb.ldri = c;
                cb.n = static_cast<int>(c);
                ts::launch_rform_check(cb, nb, sd);
            }
            sc.launches += sd.launches;
        }  // a side-stream scratch is released on the side stream
        if (overlap) TS_CUDA_CHECK(cudaEventRecord(ctx->ev_join, ctx->side));
        if (any) {
            if (spec) {
                dflags = flags;
            } else {
                std::vector<int> hf(static_cast<size_t>(d), 0);
                TS_CUDA_CHECK(cudaMemcpyAsync(hf.data(), flags, sizeof(int) * static_cast<size_t>(d),
                                              cudaMemcpyDeviceToHost, st));
                TS_CUDA_CHECK(cudaStreamSynchronize(st));
                for (int n = 0; n < d; ++n)
                    if (hf[static_cast<size_t>(n)] != 0) chol[static_cast<size_t>(n)] = 0;
            }
        }
        std::vector<ts::TsqrPlan> plans(static_cast<size_t>(d));
        std::vector<ts::TsqrPlan*> pp;
        for (int n = 0; n < d; ++n) {
            if (chol[static_cast<size_t>(n)]) continue;
            Uh[n] = sc.alloc_n<double>(static_cast<size_t>(dims[n] * q[n]));
            if (qr_wide_mode(yc[n])) {
                ts::wide_qr(Y + yoff[n], dims[n], dims[n], yc[n], Uh[n], dims[n], sc, ctx->num_sms);
                continue;
            }
            plans[static_cast<size_t>(n)] = ts::plan_tsqr(Y + yoff[n], dims[n], dims[n], yc[n], Uh[n], dims[n], sc);
            pp.push_back(&plans[static_cast<size_t>(n)]);
        }
        if (!pp.empty()) ts::run_tsqr(pp, sc, true);
        ctx->last_qr_fallbacks = static_cast<int>(pp.size());
    }
    if (!overlap) mark(ctx, 5);
    // ---- Stage E: P_n = Û_nᵀ F_n (q_n × R_n); R-form modes: Pt_n = Y_nᵀF_n, P_n = R_n⁻ᵀPt_n
    {
        double* Pt[TS_MAX_ORDER] = {};
        std::vector<GemmProblem> ps, pr;
        for (int n = 0; n < d; ++n) {
            const bool rf = rform[static_cast<size_t>(n)] != 0;
            if (rf) Pt[n] = sc.alloc_n<double>(static_cast<size_t>(q[n] * b->R[n]));
            GemmProblem p{};
            p.A = rf ? Y + yoff[n] : Uh[n];
            p.lda = dims[n];
            p.B = b->F[n];
            p.ldb = dims[n];
            p.C = rf ? Pt[n] : P[n];
            p.ldc = q[n];
            p.M = static_cast<int>(q[n]);
            p.N = static_cast<int>(b->R[n]);
            p.K = static_cast<int>(dims[n]);
            ps.push_back(p);
            if (rf) {
                GemmProblem r{};
                r.A = Rinv[n];
                r.lda = q[n];
                r.B = Pt[n];
                r.ldb = q[n];
                r.C = P[n];
                r.ldc = q[n];
                r.M = static_cast<int>(q[n]);
                r.N = static_cast<int>(b->R[n]);
                r.K = static_cast<int>(q[n]);
                pr.push_back(r);
            }
        }
        std::vector<int> modes(static_cast<size_t>(d));
        std::iota(modes.begin(), modes.end(), 0);
        const bool e8 = ozaki_stage(ctx, b, ps, modes, sc);
        if (!e8) ts::launch_grouped_gemm(Layout::TN, ps, sc, ctx->num_sms);
        int8_stages |= e8 ? 4u : 0u;
        if (overlap) TS_CUDA_CHECK(cudaStreamWaitEvent(st, ctx->ev_join, 0));
        if (!pr.empty()) ts::launch_grouped_gemm(Layout::TN, pr, sc, ctx->num_sms);
    }
    if (ctx->debug) {  // Û of the R-form modes, for the intermediates only
        std::vector<GemmProblem> ps;
        for (int n = 0; n < d; ++n) {
            if (!rform[static_cast<size_t>(n)]) continue;
            Uh[n] = sc.alloc_n<double>(static_cast<size_t>(dims[n] * q[n]));
            GemmProblem p{};
            p.A = Y + yoff[n];
            p.lda = dims[n];
            p.B = Rinv[n];
            p.ldb = q[n];
            p.C = Uh[n];
            p.ldc = dims[n];
            p.M = static_cast<int>(dims[n]);
            p.N = p.K = static_cast<int>(q[n]);
            ps.push_back(p);
        }
        if (!ps.empty()) ts::launch_grouped_gemm(Layout::NN, ps, sc, ctx->num_sms);
    }
    mark(ctx, 6);
    std::int64_t hsize = 0;
    double* h = project_core(ctx, b, P, q, d_w, weights, sc, &hsize);
    mark(ctx, 8);
    allreduce_sum(ctx, h, hsize, st, "ncclAllReduce(h)");
    mark(ctx, 9);
    if (norm_out) {  // tucker_norm: ‖orthogonalized core‖ (src/tucker.cpp:159), no rounding
        double* d_ss = sc.alloc_n<double>(1);
        ts::launch_sumsq(h, hsize, d_ss, sc);
        double ss = 0.0;
        TS_CUDA_CHECK(cudaMemcpyAsync(&ss, d_ss, sizeof(double), cudaMemcpyDeviceToHost, st));
        TS_CUDA_CHECK(cudaStreamSynchronize(st));
        ctx->launches += sc.launches;
        *norm_out = std::sqrt(ss);
        return nullptr;
    }
    if (ctx->debug) {
        for (int n = 0; n < d; ++n) {
            copy_to_host(res->inter[2][n], Uh[n], dims[n] * q[n], st);
            res->inter_rows[2][n] = dims[n];
            res->inter_cols[2][n] = q[n];
        }
        copy_to_host(res->h, h, hsize, st);
    }
    // ---- Stage G: ST-HOSVD of h (replicated on every GPU)
    std::int64_t cur_shape[TS_MAX_ORDER];
    for (int n = 0; n < d; ++n) cur_shape[n] = q[n];
    double* Pk[TS_MAX_ORDER] = {};  // q_k × q_k left singular vectors (first rank_k columns used)
    std::int64_t rank[TS_MAX_ORDER];
    double* g = h;
    // At ε = 0 the fast-path rank is fixed by the cap (else q); at ε > 0 it is
    // known in advance only for a captured call (the probe run's ranks): then the
    // device re-derives the reference tail rule and flags any difference.
    const std::int64_t* fixed_rank = ge ? ge->ranks : nullptr;
    bool spec_g = spec && (eps == 0.0 || fixed_rank != nullptr);
    for (int n = 0; n < d; ++n) spec_g = spec_g && !qr_wide_mode(q[n]);  // wide eigensolves sync anyway
    if (spec_g) gflags = flags_all + d;  // zeroed with the stage-D flags
    {
        double hss = 0.0;  // θ = ε²‖h‖²/d vanishes at ε = 0
        double* d_hss = nullptr;
        if (eps != 0.0) {
            d_hss = sc.alloc_n<double>(1);
            ts::launch_sumsq(h, hsize, d_hss, sc);
            if (!spec_g) {
                TS_CUDA_CHECK(cudaMemcpyAsync(&hss, d_hss, sizeof(double), cudaMemcpyDeviceToHost, st));
                TS_CUDA_CHECK(cudaStreamSynchronize(st));
            }
        }
        const double theta = eps * eps * hss / static_cast<double>(d);
        ctx->last_svd_fallbacks = 0;
        ctx->last_eig_fallbacks = 0;
        const std::vector<std::int64_t> qv(q, q + d);
        const bool hints = !spec_g && ctx->hint_q == qv && (++ctx->hint_calls % 16) != 0;
        unsigned accurate_modes = 0;
        std::vector<int> mode_order(static_cast<size_t>(d));
        std::iota(mode_order.begin(), mode_order.end(), 0);
        std::stable_sort(mode_order.begin(), mode_order.end(), [&](int x, int y) { return cur_shape[x] < cur_shape[y]; });
        for (int k : mode_order) {
            const std::int64_t qk = cur_shape[k];
            Pk[k] = sc.alloc_n<double>(static_cast<size_t>(qk * qk));
            std::int64_t rest = 1;
            for (int j = 0; j < d; ++j)
                if (j != k) rest *= cur_shape[j];
            // X = g_(k)ᵀ (rest × q_k), formed only where needed: the Gram of the
            // first and last modes reads g directly, the accurate path needs X.
            double* X = nullptr;
            auto need_X = [&]() {
                if (!X) {
                    X = sc.alloc_n<double>(static_cast<size_t>(rest * qk));
                    ts::launch_unfold_t(g, d, cur_shape, k, X, sc);
                }
                return X;
            };
            const bool hinted = hints && (ctx->hint_accurate >> k & 1u);
            // Fast path: Gram C = g_(k)·g_(k)ᵀ (DMMA GEMM) + two-sided Jacobi.
            double* C = sc.alloc_n<double>(static_cast<size_t>(qk * qk));
            double* lam = sc.alloc_n<double>(static_cast<size_t>(qk));
            if (!hinted) {
                GemmProblem p{};
                p.M = p.N = static_cast<int>(qk);
                p.K = static_cast<int>(rest);
                p.C = C;
                p.ldc = qk;
                if (k == 0) {  // g as a q_0 × rest matrix: C = g·gᵀ
                    p.A = p.B = g;
                    p.lda = p.ldb = qk;
                    ts::launch_grouped_gemm(Layout::NT, {p}, sc, ctx->num_sms);
                } else if (k == d - 1) {  // g as a rest × q_last matrix M: C = MᵀM
                    p.A = p.B = g;
                    p.lda = p.ldb = rest;
                    ts::launch_grouped_gemm(Layout::TN, {p}, sc, ctx->num_sms);
                } else {
                    p.A = p.B = need_X();
                    p.lda = p.ldb = rest;
                    ts::launch_grouped_gemm(Layout::TN, {p}, sc, ctx->num_sms);
                }
            }
            static const bool dbg_sweeps = std::getenv("TS_DEBUG_SWEEPS") != nullptr;
            int* dsw = dbg_sweeps ? sc.alloc_n<int>(1) : nullptr;
            const std::int64_t capk = max_rank ? max_rank[k] : 0;
            if (hinted) {
                // Last time this mode's Gram decision was not provably exact: go
                // straight to the accurate TSQR + one-sided Jacobi SVD.
                double* sigma = sc.alloc_n<double>(static_cast<size_t>(qk));
                unfolding_svd_accurate(need_X(), rest, qk, sigma, Pk[k], sc, ctx->num_sms);
                std::vector<double> sig(static_cast<size_t>(qk));
                TS_CUDA_CHECK(cudaMemcpyAsync(sig.data(), sigma, sizeof(double) * static_cast<size_t>(qk),
                                              cudaMemcpyDeviceToHost, st));
                TS_CUDA_CHECK(cudaStreamSynchronize(st));
                rank[k] = hosvd_rank(sig, eps, theta, capk);
                ++ctx->last_svd_fallbacks;
                accurate_modes |= 1u << k;
            } else {
            // Eigensolver: for q ≤ 64 the tridiagonalisation solver (eig_trd.cu)
            // with its device acceptance check and measured residual; on rejection
            // the two-sided Jacobi (eig.cu) recomputes — in the speculative path
            // via the stage-G flag (whole call redone synchronously), otherwise
            // here.  Larger q (and TS_EIG=jacobi) take Jacobi directly.
            const bool use_trd = qk <= 64 && !dsw && !ts::jacobi_eig_forced();
            int* tflag = nullptr;
            double* d_res = nullptr;
            if (use_trd) {
                if (spec_g) {
                    tflag = gflags + k;
                } else {
                    tflag = sc.alloc_n<int>(1);
                    TS_CUDA_CHECK(cudaMemsetAsync(tflag, 0, sizeof(int), st));
                }
                d_res = sc.alloc_n<double>(1);
                ts::launch_sym_trd(C, qk, static_cast<int>(qk), lam, Pk[k], tflag, d_res, sc);
            } else {
                sym_eig_any(C, qk, lam, Pk[k], sc, ctx->num_sms, dsw);
            }
            std::int64_t rk = 0;
            if (spec_g && !dsw) {
                if (eps == 0.0) {
                    // At ε = 0 the fast-path rank is fixed (cap, else q); its checks run on the device.
                    rk = (capk > 0 && capk < qk) ? capk : qk;
                    ts::launch_gram_check(lam, static_cast<int>(qk), static_cast<int>(capk), d_res, gflags + k, sc);
                } else {
                    rk = fixed_rank[k];
                    ts::launch_gram_rank_check(lam, static_cast<int>(qk), static_cast<int>(capk), eps, d, d_hss, d_res,
                                               static_cast<int>(rk), gflags + k, sc);
                }
            } else {
                std::vector<double> lv(static_cast<size_t>(qk));
                TS_CUDA_CHECK(cudaMemcpyAsync(lv.data(), lam, sizeof(double) * static_cast<size_t>(qk),
                                              cudaMemcpyDeviceToHost, st));
                int hsw = 0, htf = 0;
                double hres = -1.0;
                if (dsw) TS_CUDA_CHECK(cudaMemcpyAsync(&hsw, dsw, sizeof(int), cudaMemcpyDeviceToHost, st));
                if (tflag) TS_CUDA_CHECK(cudaMemcpyAsync(&htf, tflag, sizeof(int), cudaMemcpyDeviceToHost, st));
                if (d_res) TS_CUDA_CHECK(cudaMemcpyAsync(&hres, d_res, sizeof(double), cudaMemcpyDeviceToHost, st));
                TS_CUDA_CHECK(cudaStreamSynchronize(st));
                if (htf) {  // the tridiagonalisation solver rejected its own result
                    sym_eig_any(C, qk, lam, Pk[k], sc, ctx->num_sms);
                    TS_CUDA_CHECK(cudaMemcpyAsync(lv.data(), lam, sizeof(double) * static_cast<size_t>(qk),
                                                  cudaMemcpyDeviceToHost, st));
                    TS_CUDA_CHECK(cudaStreamSynchronize(st));
                    hres = -1.0;  // Jacobi: the assumed residual
                    ++ctx->last_eig_fallbacks;
                }
                if (dsw)
                    std::fprintf(stderr, "[ts] st-hosvd mode %d: n=%lld sweeps=%d lam1=%.3e lam_last=%.3e\n", k,
                                 static_cast<long long>(qk), hsw, lv[0], lv.back());
                bool ok = false;
                rk = gram_rank(lv, eps, theta, capk, hres, &ok);
                if (!ok) {
                    double* sigma = sc.alloc_n<double>(static_cast<size_t>(qk));
                    unfolding_svd_accurate(need_X(), rest, qk, sigma, Pk[k], sc, ctx->num_sms);
                    std::vector<double> sig(static_cast<size_t>(qk));
                    TS_CUDA_CHECK(cudaMemcpyAsync(sig.data(), sigma, sizeof(double) * static_cast<size_t>(qk),
                                                  cudaMemcpyDeviceToHost, st));
                    TS_CUDA_CHECK(cudaStreamSynchronize(st));
                    rk = hosvd_rank(sig, eps, theta, capk);
                    ++ctx->last_svd_fallbacks;
                    accurate_modes |= 1u << k;
                }
            }
            rank[k] = rk;
            }
            const std::int64_t rk = rank[k];
            // g ← g ×_k P_kᵀ
            std::int64_t left = 1, right = 1, total_out = rk;
            for (int j = 0; j < d; ++j) {
                if (j < k) left *= cur_shape[j];
                if (j > k) right *= cur_shape[j];
                if (j != k) total_out *= cur_shape[j];
            }
            double* gn = sc.alloc_n<double>(static_cast<size_t>(total_out));
            GemmProblem p{};
            if (k == 0) {
                p.A = Pk[k];
                p.lda = qk;
                p.B = g;
                p.ldb = qk;
                p.C = gn;
                p.ldc = rk;
                p.M = static_cast<int>(rk);
                p.N = static_cast<int>(right);
                p.K = static_cast<int>(qk);
                ts::launch_grouped_gemm(Layout::TN, {p}, sc, ctx->num_sms);
            } else {
                p.A = g;
                p.lda = left;
                p.sA = left * qk;
                p.B = Pk[k];
                p.ldb = qk;
                p.C = gn;
                p.ldc = left;
                p.sC = left * rk;
                p.M = static_cast<int>(left);
                p.N = static_cast<int>(rk);
                p.K = static_cast<int>(qk);
                p.batch = static_cast<int>(right);
                ts::launch_grouped_gemm(Layout::NN, {p}, sc, ctx->num_sms);
            }
            g = gn;
            cur_shape[k] = rk;
        }
        if (!spec_g) {
            ctx->hint_q = qv;
            ctx->hint_accurate = accurate_modes;
        }
    }
    mark(ctx, 10);
    // ---- Stage H: Ũ_n = Û_n · P_n (n × rank_n); the core is g.
    {
        double* Tk[TS_MAX_ORDER] = {};
        {  // R-form modes: Ũ_n = Y_n (R_n⁻¹ P_k), first T_n = R_n⁻¹ P_k (q_n × rank_n)
            std::vector<GemmProblem> ts_;
            for (int n = 0; n < d; ++n) {
                if (!rform[static_cast<size_t>(n)]) continue;
                Tk[n] = sc.alloc_n<double>(static_cast<size_t>(q[n] * rank[n]));
                GemmProblem p{};
                p.A = Rinv[n];
                p.lda = q[n];
                p.B = Pk[n];
                p.ldb = q[n];
                p.C = Tk[n];
                p.ldc = q[n];
                p.M = static_cast<int>(q[n]);
                p.N = static_cast<int>(rank[n]);
                p.K = static_cast<int>(q[n]);
                ts_.push_back(p);
            }
            if (!ts_.empty()) ts::launch_grouped_gemm(Layout::NN, ts_, sc, ctx->num_sms);
        }
        std::vector<GemmProblem> ps;
        for (int n = 0; n < d; ++n) {
            res->dims[n] = dims[n];
            res->ranks[n] = rank[n];
            if (ge) {  // captured call: outputs go to the graph's own buffers
                if (ge->ranks[n] != rank[n]) throw ts::Error(TS_RUNTIME, "graph capture: rank mismatch");
                res->factors[n] = ge->out_f[n];
            } else {
                TS_CUDA_CHECK(cudaMallocAsync(&res->factors[n], sizeof(double) * static_cast<size_t>(dims[n] * rank[n]), st));
            }
            GemmProblem p{};
            p.A = rform[static_cast<size_t>(n)] ? Y + yoff[n] : Uh[n];
            p.lda = dims[n];
            p.B = rform[static_cast<size_t>(n)] ? Tk[n] : Pk[n];
            p.ldb = q[n];
            p.C = res->factors[n];
            p.ldc = dims[n];
            p.M = static_cast<int>(dims[n]);
            p.N = static_cast<int>(rank[n]);
            p.K = static_cast<int>(q[n]);
            ps.push_back(p);
        }
        ts::launch_grouped_gemm(Layout::NN, ps, sc, ctx->num_sms);
        std::int64_t csize = 1;
        for (int n = 0; n < d; ++n) csize *= rank[n];
        if (ge) {
            res->core = ge->out_core;
        } else {
            TS_CUDA_CHECK(cudaMallocAsync(&res->core, sizeof(double) * static_cast<size_t>(csize), st));
        }
        TS_CUDA_CHECK(cudaMemcpyAsync(res->core, g, sizeof(double) * static_cast<size_t>(csize),
                                      cudaMemcpyDeviceToDevice, st));
    }
    mark(ctx, 11);
    if (ge) {  // end of the captured region: flags to pinned host memory, no sync
        ge->launches = sc.launches;
        if (dflags && gflags)
            TS_CUDA_CHECK(cudaMemcpyAsync(ge->h_flags, flags_all, 2 * sizeof(int) * static_cast<size_t>(d), cudaMemcpyDeviceToHost, st));
        else if (dflags)
            TS_CUDA_CHECK(cudaMemcpyAsync(ge->h_flags, dflags, sizeof(int) * static_cast<size_t>(d), cudaMemcpyDeviceToHost, st));
        else if (gflags)
            TS_CUDA_CHECK(cudaMemcpyAsync(ge->h_flags + d, gflags, sizeof(int) * static_cast<size_t>(d),
                                          cudaMemcpyDeviceToHost, st));
        for (int n = 0; n < d; ++n) res->factors[n] = nullptr;  // graph-owned, not the result's
        res->core = nullptr;
        return nullptr;
    }
    ctx->launches += sc.launches;
    if (spec) {
        std::vector<int> hf(2 * static_cast<size_t>(d), 0);
        if (dflags)
            TS_CUDA_CHECK(cudaMemcpyAsync(hf.data(), dflags, sizeof(int) * static_cast<size_t>(d), cudaMemcpyDeviceToHost, st));
        if (gflags)
            TS_CUDA_CHECK(cudaMemcpyAsync(hf.data() + d, gflags, sizeof(int) * static_cast<size_t>(d),
                                          cudaMemcpyDeviceToHost, st));
        TS_CUDA_CHECK(cudaStreamSynchronize(st));
        for (int x : hf)
            if (x != 0) {
                ctx->spec_ok = false;
                res.reset();
                return sketched_sum_impl(ctx, b, weights, widths, seed, stream, eps, max_rank, method, false);
            }
    } else {
        ctx->spec_ok = ctx->last_qr_fallbacks == 0 && ctx->last_svd_fallbacks == 0;
    }
    TS_CUDA_CHECK(cudaStreamSynchronize(st));
    ctx->last_int8_stages = int8_stages | (ctx->f2_int8 ? 8u : 0u);
    if (ctx->timing) {
        ctx->stage_ms.assign(kNumStages + 2, 0.0);
        for (int i = 0; i < kNumStages; ++i) {
            float ms = 0.f;
            TS_CUDA_CHECK(cudaEventElapsedTime(&ms, ctx->events[static_cast<size_t>(i)], ctx->events[static_cast<size_t>(i + 1)]));
            ctx->stage_ms[static_cast<size_t>(i)] = ms;
        }
        {  // stage A's GEMM kernel alone (the two hook events around its launch)
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, ctx->events[kNumStages + 1], ctx->events[kNumStages + 2]) == cudaSuccess && ms > 0.f &&
                ms <= ctx->stage_ms[0] + 1e-3)
                ctx->stage_ms[kNumStages] = ms;
            else
                (void)cudaGetLastError();
        }
        if (!lazy) {  // stage C's GEMM kernel alone
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, ctx->events[kNumStages + 3], ctx->events[kNumStages + 4]) == cudaSuccess && ms > 0.f &&
                ms <= ctx->stage_ms[2] + 1e-3)
                ctx->stage_ms[kNumStages + 1] = ms;
            else
                (void)cudaGetLastError();
        }
    }
    return res.release();
}

// Segmented KRP sums (one round_sum per NDG node with a
// shared plan, src/ndg.cpp:401-462; many GMRES sums, src/cookie.cpp:389-421).
// S independent krp_sum calls whose summands are the consecutive segments
// [seg[s], seg[s+1]) of ONE uploaded batch share the plan widths; every stage
// runs as one launch over all sums — grouped DMMA GEMMs over the (sum, mode)
// problems, the stage-B and stage-F1 kernels over all atoms, one Cholesky CTA
// and one eigensolver CTA per (sum, mode) — so S small sums cost about what one
// does instead of S times its latency.  Sum s computes exactly what
// ts_krp_sum(batch of its summands, its weights, widths, seeds[s], …) computes
// (same kernels per problem, so the same numbers up to the split-K choices of
// the grouped launches).
std::vector<ts_result*> segmented_impl(ts_ctx* ctx, const ts_batch* b, std::int64_t S, const std::int64_t* seg,
                                       const double* weights, const std::int64_t* widths, const std::uint64_t* seeds,
                                       const std::uint64_t* streams, double eps, const std::int64_t* max_rank,
                                       bool allow_spec) {
    if (b == nullptr || b->count < 1 || S < 1 || seg == nullptr || weights == nullptr || seeds == nullptr ||
        streams == nullptr)
        invalid("sum request needs matching, nonempty summands and weights");
    if (b->ctx->device != ctx->device) invalid("batch was uploaded to another device than this context's");
    if (seg[0] != 0 || seg[S] != b->count) invalid("segments must partition the batch's summands");
    for (std::int64_t s = 0; s < S; ++s)
        if (seg[s + 1] <= seg[s]) invalid("sum request needs matching, nonempty summands and weights");
    if (!(eps >= 0.0)) invalid("tolerance must be nonnegative");
    const int d = b->order;
    if (d < 2) invalid("sketched summation needs order >= 2");
    if (widths == nullptr) invalid("plan order does not match summand order");
    for (int n = 0; n < d; ++n)
        if (widths[n] < 1) invalid("plan sketch widths must be positive");
    if (sharded(ctx)) throw ts::Error(TS_UNSUPPORTED, "segmented sums do not shard: use a context without NCCL");
    if (b->scol.empty()) throw ts::Error(TS_UNSUPPORTED, "segmented sums need a batch from ts_batch_upload*");
    for (std::int64_t i = 0; i < b->count; ++i)
        if (!std::isfinite(weights[i])) invalid("weights must be finite");
    const std::int64_t sw = *std::max_element(widths, widths + d);
    TS_CUDA_CHECK(cudaSetDevice(ctx->device));
    ctx->stage.reset();
    cudaStream_t st = ctx->stream;
    CallScratch sc(st, ctx->stage);
    static const bool dbg_seg = std::getenv("TS_DEBUG_SEG") != nullptr;
    auto t_last = std::chrono::steady_clock::now();
    auto tick = [&](const char* what) {
        if (!dbg_seg) return;
        TS_CUDA_CHECK(cudaStreamSynchronize(st));
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[seg] %-8s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(now - t_last).count());
        t_last = now;
    };
    const std::int64_t* dims = b->dims;
    auto col = [&](std::int64_t s, int n) { return b->scol[static_cast<size_t>(seg[s] * d + n)]; };
    auto rsn = [&](std::int64_t s, int n) { return col(s + 1, n) - col(s, n); };
    const size_t SD = static_cast<size_t>(S) * static_cast<size_t>(d);
    auto sn = [&](std::int64_t s, int n) { return static_cast<size_t>(s) * static_cast<size_t>(d) + static_cast<size_t>(n); };
    std::int64_t q[TS_MAX_ORDER], ow[TS_MAX_ORDER], ooff[TS_MAX_ORDER], yoff[TS_MAX_ORDER];
    std::int64_t ysum = 0, oacc = 0;
    for (int n = 0; n < d; ++n) {
        ow[n] = sw;
        q[n] = std::min(dims[n], sw);
        ooff[n] = oacc;
        oacc += dims[n] * sw;
        yoff[n] = ysum;
        ysum += dims[n] * sw;
    }
    std::vector<double*> om(static_cast<size_t>(S));
    for (std::int64_t s = 0; s < S; ++s) om[static_cast<size_t>(s)] = omega_get(ctx, d, dims, ow, seeds[s], streams[s]);
    auto* d_w = static_cast<double*>(sc.upload(weights, sizeof(double) * static_cast<size_t>(b->count)));

    tick("setup");
    // ---- A: Z_n[:, cols_s] = Ω_{s,n}ᵀ F_n[:, cols_s]
    double* Z[TS_MAX_ORDER];
    {
        std::vector<GemmProblem> ps;
        for (int n = 0; n < d; ++n) Z[n] = sc.alloc_n<double>(static_cast<size_t>(sw * b->R[n]));
        for (std::int64_t s = 0; s < S; ++s)
            for (int n = 0; n < d; ++n) {
                GemmProblem p{};
                p.A = om[static_cast<size_t>(s)] + ooff[n];
                p.lda = dims[n];
                p.B = b->F[n] + col(s, n) * dims[n];
                p.ldb = dims[n];
                p.C = Z[n] + col(s, n) * sw;
                p.ldc = sw;
                p.M = static_cast<int>(sw);
                p.N = static_cast<int>(rsn(s, n));
                p.K = static_cast<int>(dims[n]);
                ps.push_back(p);
            }
        ts::launch_grouped_gemm(Layout::TN, ps, sc, ctx->num_sms);
    }
    tick("A");
    // ---- B: one launch over all atoms (each atom reads its own sum's Z columns)
    double* W[TS_MAX_ORDER];
    {
        ts::KrpArgs ka{};
        for (int n = 0; n < d; ++n) {
            W[n] = sc.alloc_n<double>(static_cast<size_t>(b->R[n] * sw));
            ka.Z[n] = Z[n];
            ka.W[n] = W[n];
            ka.R[n] = b->R[n];
        }
        ka.order = d;
        ka.s = static_cast<int>(sw);
        ka.natoms = static_cast<int>(b->atoms.size());
        ka.atoms = b->d_atoms;
        ka.cores = b->cores;
        ka.weights = d_w;
        ts::launch_krp_contract(ka, b->max_shape, sc);
    }
    tick("B");
    // ---- C: Y_{s,n} = F_n[:, cols_s] · W_n[cols_s, :]
    double* Y = sc.alloc_n<double>(static_cast<size_t>(S * ysum));
    auto ypos = [&](std::int64_t s, int n) { return Y + s * ysum + yoff[n]; };
    {
        std::vector<GemmProblem> ps;
        for (std::int64_t s = 0; s < S; ++s)
            for (int n = 0; n < d; ++n) {
                GemmProblem p{};
                p.A = b->F[n] + col(s, n) * dims[n];
                p.lda = dims[n];
                p.B = W[n] + col(s, n) * sw;
                p.ldb = sw;
                p.C = ypos(s, n);
                p.ldc = dims[n];
                p.M = static_cast<int>(dims[n]);
                p.N = static_cast<int>(sw);
                p.K = static_cast<int>(rsn(s, n));
                ps.push_back(p);
            }
        ts::launch_grouped_gemm(Layout::NT, ps, sc, ctx->num_sms);
    }
    const bool spec = allow_spec && ctx->spec_ok;
    int* dflags = nullptr;
    int* gflags = nullptr;
    tick("C");
    // ---- D: CholeskyQR2 R form per (sum, mode) where dims ≥ 2s, Householder TSQR otherwise / on rejection
    std::vector<int> rform(SD, 0);
    std::vector<double*> Rinv(SD, nullptr), Uh(SD, nullptr);
    {
        int* flags = sc.alloc_n<int>(SD);
        TS_CUDA_CHECK(cudaMemsetAsync(flags, 0, sizeof(int) * SD, st));
        std::vector<GemmProblem> g1, q1, g2, rr;
        std::vector<const double*> hG1, hG2;
        std::vector<double*> hR1, hR2, hRi;
        std::vector<int*> hF;
        for (std::int64_t s = 0; s < S; ++s)
            for (int n = 0; n < d; ++n) {
                if (dims[n] < 2 * sw || qr_wide_mode(sw)) continue;
                const size_t i = sn(s, n);
                rform[i] = 1;
                const std::int64_t c = sw;
                double* G1 = sc.alloc_n<double>(static_cast<size_t>(c * c));
                double* G2 = sc.alloc_n<double>(static_cast<size_t>(c * c));
                double* Ri1 = sc.alloc_n<double>(static_cast<size_t>(c * c));
                double* Ri2 = sc.alloc_n<double>(static_cast<size_t>(c * c));
                double* Q1 = sc.alloc_n<double>(static_cast<size_t>(dims[n] * c));
                Rinv[i] = sc.alloc_n<double>(static_cast<size_t>(c * c));
                GemmProblem p{};
                p.M = p.N = static_cast<int>(c);
                p.K = static_cast<int>(dims[n]);
                p.A = p.B = ypos(s, n);
                p.lda = p.ldb = dims[n];
                p.C = G1;
                p.ldc = c;
                g1.push_back(p);
                p.A = p.B = Q1;
                p.C = G2;
                g2.push_back(p);
                GemmProblem m{};
                m.M = static_cast<int>(dims[n]);
                m.N = m.K = static_cast<int>(c);
                m.A = ypos(s, n);
                m.lda = dims[n];
                m.B = Ri1;
                m.ldb = c;
                m.C = Q1;
                m.ldc = dims[n];
                q1.push_back(m);
                GemmProblem r{};
                r.M = r.N = r.K = static_cast<int>(c);
                r.A = Ri1;
                r.lda = c;
                r.B = Ri2;
                r.ldb = c;
                r.C = Rinv[i];
                r.ldc = c;
                rr.push_back(r);
                hG1.push_back(G1);
                hG2.push_back(G2);
                hR1.push_back(Ri1);
                hR2.push_back(Ri2);
                hRi.push_back(Rinv[i]);
                hF.push_back(flags + i);
            }
        const int nb = static_cast<int>(hG1.size());
        if (nb > 0) {
            auto up = [&](const void* src, size_t bytes) { return sc.upload(src, bytes); };
            ts::CholBatch c1{}, c2{}, cr{};
            c1.Gd = static_cast<const double* const*>(up(hG1.data(), sizeof(double*) * hG1.size()));
            c1.Rd = static_cast<double* const*>(up(hR1.data(), sizeof(double*) * hR1.size()));
            c1.Fd = static_cast<int* const*>(up(hF.data(), sizeof(int*) * hF.size()));
            c2 = c1;
            c2.Gd = static_cast<const double* const*>(up(hG2.data(), sizeof(double*) * hG2.size()));
            c2.Rd = static_cast<double* const*>(up(hR2.data(), sizeof(double*) * hR2.size()));
            cr = c1;
            cr.Rd = static_cast<double* const*>(up(hRi.data(), sizeof(double*) * hRi.size()));
            for (ts::CholBatch* cb : {&c1, &c2, &cr}) {
                cb->ldg = cb->ldri = sw;
                cb->n = static_cast<int>(sw);
            }
            c2.check_identity = 1;
            ts::launch_grouped_gemm(Layout::TN, g1, sc, ctx->num_sms);
            ts::launch_chol_inv(c1, nb, sc);
            ts::launch_grouped_gemm(Layout::NN, q1, sc, ctx->num_sms);
            ts::launch_grouped_gemm(Layout::TN, g2, sc, ctx->num_sms);
            ts::launch_chol_inv(c2, nb, sc);
            ts::launch_grouped_gemm(Layout::NN, rr, sc, ctx->num_sms);
            ts::launch_rform_check(cr, nb, sc);
            if (spec) {
                dflags = flags;
            } else {
                std::vector<int> hf(SD, 0);
                TS_CUDA_CHECK(cudaMemcpyAsync(hf.data(), flags, sizeof(int) * SD, cudaMemcpyDeviceToHost, st));
                TS_CUDA_CHECK(cudaStreamSynchronize(st));
                for (size_t i = 0; i < SD; ++i)
                    if (hf[i] != 0) rform[i] = 0;
            }
        }
        std::vector<ts::TsqrPlan> plans(SD);
        std::vector<ts::TsqrPlan*> pp;
        for (std::int64_t s = 0; s < S; ++s)
            for (int n = 0; n < d; ++n) {
                const size_t i = sn(s, n);
                if (rform[i]) continue;
                Uh[i] = sc.alloc_n<double>(static_cast<size_t>(dims[n] * q[n]));
                if (qr_wide_mode(sw)) {
                    ts::wide_qr(ypos(s, n), dims[n], dims[n], sw, Uh[i], dims[n], sc, ctx->num_sms);
                    continue;
                }
                plans[i] = ts::plan_tsqr(ypos(s, n), dims[n], dims[n], sw, Uh[i], dims[n], sc);
                pp.push_back(&plans[i]);
            }
        if (!pp.empty()) ts::run_tsqr(pp, sc, true);
        ctx->last_qr_fallbacks = static_cast<int>(pp.size());
    }
    tick("D");
    // ---- E: P_n[:, cols_s] = Û_{s,n}ᵀ F_n[:, cols_s]  (R form: R⁻ᵀ (Y_{s,n}ᵀ F_n[:, cols_s]))
    double* P[TS_MAX_ORDER];
    {
        for (int n = 0; n < d; ++n) P[n] = sc.alloc_n<double>(static_cast<size_t>(q[n] * b->R[n]));
        std::vector<GemmProblem> ps, pr;
        for (std::int64_t s = 0; s < S; ++s)
            for (int n = 0; n < d; ++n) {
                const size_t i = sn(s, n);
                const bool rf = rform[i] != 0;
                double* Pt = rf ? sc.alloc_n<double>(static_cast<size_t>(q[n] * rsn(s, n))) : nullptr;
                GemmProblem p{};
                p.A = rf ? ypos(s, n) : Uh[i];
                p.lda = dims[n];
                p.B = b->F[n] + col(s, n) * dims[n];
                p.ldb = dims[n];
                p.C = rf ? Pt : P[n] + col(s, n) * q[n];
                p.ldc = q[n];
                p.M = static_cast<int>(q[n]);
                p.N = static_cast<int>(rsn(s, n));
                p.K = static_cast<int>(dims[n]);
                ps.push_back(p);
                if (rf) {
                    GemmProblem r{};
                    r.A = Rinv[i];
                    r.lda = q[n];
                    r.B = Pt;
                    r.ldb = q[n];
                    r.C = P[n] + col(s, n) * q[n];
                    r.ldc = q[n];
                    r.M = static_cast<int>(q[n]);
                    r.N = static_cast<int>(rsn(s, n));
                    r.K = static_cast<int>(q[n]);
                    pr.push_back(r);
                }
            }
        ts::launch_grouped_gemm(Layout::TN, ps, sc, ctx->num_sms);
        if (!pr.empty()) ts::launch_grouped_gemm(Layout::TN, pr, sc, ctx->num_sms);
    }
    tick("E");
    // ---- F: T_stack over all atoms, then h_s = T_stack[:, cols_s] · P_{d-1}[:, cols_s]ᵀ
    std::int64_t Qp = 1;
    for (int j = 0; j < d - 1; ++j) Qp *= q[j];
    const std::int64_t hsz = Qp * q[d - 1];
    double* Tstack = project_core_f1(ctx, b, P, q, d_w, weights, sc);
    double* H = sc.alloc_n<double>(static_cast<size_t>(S * hsz));
    {
        std::vector<GemmProblem> ps;
        for (std::int64_t s = 0; s < S; ++s) {
            GemmProblem p{};
            p.A = Tstack + col(s, d - 1) * Qp;
            p.lda = Qp;
            p.B = P[d - 1] + col(s, d - 1) * q[d - 1];
            p.ldb = q[d - 1];
            p.C = H + s * hsz;
            p.ldc = Qp;
            p.M = static_cast<int>(Qp);
            p.N = static_cast<int>(q[d - 1]);
            p.K = static_cast<int>(rsn(s, d - 1));
            ps.push_back(p);
        }
        ts::launch_grouped_gemm(Layout::NT, ps, sc, ctx->num_sms);
    }
    tick("F");
    // ---- G: ST-HOSVD of every h_s, one mode step at a time for all sums
    std::vector<std::array<std::int64_t, TS_MAX_ORDER>> shp(static_cast<size_t>(S));
    std::vector<std::array<std::int64_t, TS_MAX_ORDER>> rank(static_cast<size_t>(S));
    std::vector<std::array<double*, TS_MAX_ORDER>> Pk(static_cast<size_t>(S));
    std::vector<double*> g(static_cast<size_t>(S));
    for (std::int64_t s = 0; s < S; ++s) {
        for (int n = 0; n < d; ++n) shp[static_cast<size_t>(s)][static_cast<size_t>(n)] = q[n];
        g[static_cast<size_t>(s)] = H + s * hsz;
    }
    bool spec_g = spec && eps == 0.0;
    for (int n = 0; n < d; ++n) spec_g = spec_g && !qr_wide_mode(q[n]);  // wide eigensolves sync anyway
    if (spec_g) {
        gflags = sc.alloc_n<int>(SD);
        TS_CUDA_CHECK(cudaMemsetAsync(gflags, 0, sizeof(int) * SD, st));
    }
    std::vector<double> theta(static_cast<size_t>(S), 0.0);
    if (eps != 0.0) {  // θ_s = ε²‖h_s‖²/d
        double* d_ss = sc.alloc_n<double>(static_cast<size_t>(S));
        for (std::int64_t s = 0; s < S; ++s) ts::launch_sumsq(H + s * hsz, hsz, d_ss + s, sc);
        std::vector<double> hs(static_cast<size_t>(S));
        TS_CUDA_CHECK(cudaMemcpyAsync(hs.data(), d_ss, sizeof(double) * static_cast<size_t>(S), cudaMemcpyDeviceToHost, st));
        TS_CUDA_CHECK(cudaStreamSynchronize(st));
        for (std::int64_t s = 0; s < S; ++s) theta[static_cast<size_t>(s)] = eps * eps * hs[static_cast<size_t>(s)] / static_cast<double>(d);
    }
    ctx->last_svd_fallbacks = 0;
    ctx->last_eig_fallbacks = 0;
    std::vector<int> mode_order(static_cast<size_t>(d));
    std::iota(mode_order.begin(), mode_order.end(), 0);
    std::stable_sort(mode_order.begin(), mode_order.end(), [&](int x, int y) { return q[x] < q[y]; });
    for (int k : mode_order) {
        const std::int64_t qk = q[k];  // mode k is untouched until its step: q_k for every sum
        double* Call = sc.alloc_n<double>(static_cast<size_t>(S * qk * qk));
        double* Lall = sc.alloc_n<double>(static_cast<size_t>(S * qk));
        double* Vall = sc.alloc_n<double>(static_cast<size_t>(S * qk * qk));
        std::vector<double*> X(static_cast<size_t>(S), nullptr);
        std::vector<std::int64_t> rest(static_cast<size_t>(S), 1);
        std::vector<GemmProblem> gnt, gtn;
        for (std::int64_t s = 0; s < S; ++s) {
            auto& cs = shp[static_cast<size_t>(s)];
            for (int j = 0; j < d; ++j)
                if (j != k) rest[static_cast<size_t>(s)] *= cs[static_cast<size_t>(j)];
            Pk[static_cast<size_t>(s)][static_cast<size_t>(k)] = Vall + s * qk * qk;
            GemmProblem p{};
            p.M = p.N = static_cast<int>(qk);
            p.K = static_cast<int>(rest[static_cast<size_t>(s)]);
            p.C = Call + s * qk * qk;
            p.ldc = qk;
            if (k == 0) {
                p.A = p.B = g[static_cast<size_t>(s)];
                p.lda = p.ldb = qk;
                gnt.push_back(p);
            } else {
                if (k != d - 1)
                    X[static_cast<size_t>(s)] = sc.alloc_n<double>(static_cast<size_t>(rest[static_cast<size_t>(s)] * qk));
                p.A = p.B = k == d - 1 ? g[static_cast<size_t>(s)] : X[static_cast<size_t>(s)];
                p.lda = p.ldb = rest[static_cast<size_t>(s)];
                gtn.push_back(p);
            }
        }
        if (k != 0 && k != d - 1) {  // X_s = g_s,(k)ᵀ: one launch per group of sums with the same current shape
            std::vector<bool> done(static_cast<size_t>(S), false);
            for (std::int64_t s0 = 0; s0 < S; ++s0) {
                if (done[static_cast<size_t>(s0)]) continue;
                std::vector<const double*> gsrc;
                std::vector<double*> xdst;
                for (std::int64_t s = s0; s < S; ++s)
                    if (!done[static_cast<size_t>(s)] && shp[static_cast<size_t>(s)] == shp[static_cast<size_t>(s0)]) {
                        done[static_cast<size_t>(s)] = true;
                        gsrc.push_back(g[static_cast<size_t>(s)]);
                        xdst.push_back(X[static_cast<size_t>(s)]);
                    }
                auto* dg = static_cast<const double* const*>(sc.upload(gsrc.data(), sizeof(double*) * gsrc.size()));
                auto* dx = static_cast<double* const*>(sc.upload(xdst.data(), sizeof(double*) * xdst.size()));
                ts::launch_unfold_t_batched(dg, dx, static_cast<int>(gsrc.size()), d, shp[static_cast<size_t>(s0)].data(), k,
                                            sc);
            }
        }
        if (!gnt.empty()) ts::launch_grouped_gemm(Layout::NT, gnt, sc, ctx->num_sms);
        if (!gtn.empty()) ts::launch_grouped_gemm(Layout::TN, gtn, sc, ctx->num_sms);
        const std::int64_t capk = max_rank ? max_rank[k] : 0;
        // speculative: the eigensolver's rejections and the Gram checks of this
        // mode step land in gflags[k·S + s] directly
        int* tflags = spec_g ? gflags + static_cast<size_t>(k) * static_cast<size_t>(S) : sc.alloc_n<int>(static_cast<size_t>(S));
        if (!spec_g) TS_CUDA_CHECK(cudaMemsetAsync(tflags, 0, sizeof(int) * static_cast<size_t>(S), st));
        double* res = sc.alloc_n<double>(static_cast<size_t>(S));
        const bool trd = qk <= 64 && !ts::jacobi_eig_forced();
        if (trd) {
            ts::launch_sym_trd(Call, qk, static_cast<int>(qk), Lall, Vall, tflags, res, sc, static_cast<int>(S), qk * qk,
                               qk, qk * qk);
        } else {
            for (std::int64_t s = 0; s < S; ++s)
                sym_eig_any(Call + s * qk * qk, qk, Lall + s * qk, Vall + s * qk * qk, sc, ctx->num_sms);
        }
        std::vector<std::int64_t> rk(static_cast<size_t>(S), 0);
        if (spec_g) {
            for (std::int64_t s = 0; s < S; ++s) rk[static_cast<size_t>(s)] = (capk > 0 && capk < qk) ? capk : qk;
            ts::launch_gram_check(Lall, static_cast<int>(qk), static_cast<int>(capk), trd ? res : nullptr, tflags, sc,
                                  static_cast<int>(S), qk);
        } else {
            std::vector<double> lv(static_cast<size_t>(S * qk)), hres(static_cast<size_t>(S), -1.0);
            std::vector<int> htf(static_cast<size_t>(S), 0);
            TS_CUDA_CHECK(cudaMemcpyAsync(lv.data(), Lall, sizeof(double) * lv.size(), cudaMemcpyDeviceToHost, st));
            TS_CUDA_CHECK(cudaMemcpyAsync(htf.data(), tflags, sizeof(int) * htf.size(), cudaMemcpyDeviceToHost, st));
            if (trd) TS_CUDA_CHECK(cudaMemcpyAsync(hres.data(), res, sizeof(double) * hres.size(), cudaMemcpyDeviceToHost, st));
            TS_CUDA_CHECK(cudaStreamSynchronize(st));
            for (std::int64_t s = 0; s < S; ++s) {
                const size_t si = static_cast<size_t>(s);
                double* Cs = Call + s * qk * qk;
                double* Ls = Lall + s * qk;
                double* Vs = Vall + s * qk * qk;
                std::vector<double> lam(lv.begin() + static_cast<std::ptrdiff_t>(s * qk),
                                        lv.begin() + static_cast<std::ptrdiff_t>((s + 1) * qk));
                double rres = trd ? hres[si] : -1.0;
                if (trd && htf[si]) {  // the tridiagonalisation solver rejected its own result
                    sym_eig_any(Cs, qk, Ls, Vs, sc, ctx->num_sms);
                    TS_CUDA_CHECK(cudaMemcpyAsync(lam.data(), Ls, sizeof(double) * static_cast<size_t>(qk),
                                                  cudaMemcpyDeviceToHost, st));
                    TS_CUDA_CHECK(cudaStreamSynchronize(st));
                    rres = -1.0;
                    ++ctx->last_eig_fallbacks;
                }
                bool ok = false;
                rk[si] = gram_rank(lam, eps, theta[si], capk, rres, &ok);
                if (!ok) {  // accurate path: TSQR (R only) of h_(k)ᵀ + one-sided Jacobi SVD
                    double* Xs = sc.alloc_n<double>(static_cast<size_t>(rest[si] * qk));
                    ts::launch_unfold_t(g[si], d, shp[si].data(), k, Xs, sc);
                    double* sigma = sc.alloc_n<double>(static_cast<size_t>(qk));
                    unfolding_svd_accurate(Xs, rest[si], qk, sigma, Vs, sc, ctx->num_sms);
                    std::vector<double> sig(static_cast<size_t>(qk));
                    TS_CUDA_CHECK(cudaMemcpyAsync(sig.data(), sigma, sizeof(double) * static_cast<size_t>(qk),
                                                  cudaMemcpyDeviceToHost, st));
                    TS_CUDA_CHECK(cudaStreamSynchronize(st));
                    rk[si] = hosvd_rank(sig, eps, theta[si], capk);
                    ++ctx->last_svd_fallbacks;
                }
            }
        }
        // g_s ← g_s ×_k P_kᵀ (first rank columns)
        std::vector<GemmProblem> t0, t1;
        for (std::int64_t s = 0; s < S; ++s) {
            const size_t si = static_cast<size_t>(s);
            auto& cs = shp[si];
            std::int64_t left = 1, right = 1, total_out = rk[si];
            for (int j = 0; j < d; ++j) {
                if (j < k) left *= cs[static_cast<size_t>(j)];
                if (j > k) right *= cs[static_cast<size_t>(j)];
                if (j != k) total_out *= cs[static_cast<size_t>(j)];
            }
            double* gn = sc.alloc_n<double>(static_cast<size_t>(total_out));
            GemmProblem p{};
            if (k == 0) {
                p.A = Pk[si][static_cast<size_t>(k)];
                p.lda = qk;
                p.B = g[si];
                p.ldb = qk;
                p.C = gn;
                p.ldc = rk[si];
                p.M = static_cast<int>(rk[si]);
                p.N = static_cast<int>(right);
                p.K = static_cast<int>(qk);
                t0.push_back(p);
            } else {
                p.A = g[si];
                p.lda = left;
                p.sA = left * qk;
                p.B = Pk[si][static_cast<size_t>(k)];
                p.ldb = qk;
                p.C = gn;
                p.ldc = left;
                p.sC = left * rk[si];
                p.M = static_cast<int>(left);
                p.N = static_cast<int>(rk[si]);
                p.K = static_cast<int>(qk);
                p.batch = static_cast<int>(right);
                t1.push_back(p);
            }
            g[si] = gn;
            cs[static_cast<size_t>(k)] = rk[si];
            rank[si][static_cast<size_t>(k)] = rk[si];
        }
        if (!t0.empty()) ts::launch_grouped_gemm(Layout::TN, t0, sc, ctx->num_sms);
        if (!t1.empty()) ts::launch_grouped_gemm(Layout::NN, t1, sc, ctx->num_sms);
    }
    tick("G");
    // ---- H: Ũ_{s,n} = Y_{s,n}(R⁻¹P_k) or Û_{s,n}P_k; results
    std::vector<std::unique_ptr<ts_result>> out(static_cast<size_t>(S));
    {
        std::int64_t total = 0;
        for (std::int64_t s = 0; s < S; ++s) {
            std::int64_t csize = 1;
            for (int n = 0; n < d; ++n) {
                const std::int64_t rkn = rank[static_cast<size_t>(s)][static_cast<size_t>(n)];
                total += (dims[n] * rkn + 31) / 32 * 32;
                csize *= rkn;
            }
            total += (csize + 31) / 32 * 32;
        }
        double* block = nullptr;
        TS_CUDA_CHECK(cudaMallocAsync(&block, sizeof(double) * static_cast<size_t>(std::max<std::int64_t>(total, 1)), st));
        const int dev = ctx->device;
        std::shared_ptr<void> arena(block, [dev, st](void* p) {
            cudaSetDevice(dev);
            cudaFreeAsync(p, st);
        });
        double* bump = block;
        std::vector<GemmProblem> tp, up;
        for (std::int64_t s = 0; s < S; ++s) {
            const size_t si = static_cast<size_t>(s);
            out[si] = std::make_unique<ts_result>();
            ts_result* r = out[si].get();
            r->device = ctx->device;
            r->stream = st;
            r->order = d;
            std::int64_t csize = 1;
            for (int n = 0; n < d; ++n) {
                const size_t i = sn(s, n);
                const std::int64_t rkn = rank[si][static_cast<size_t>(n)];
                r->dims[n] = dims[n];
                r->ranks[n] = rkn;
                csize *= rkn;
                r->factors[n] = bump;
                bump += (dims[n] * rkn + 31) / 32 * 32;
                const double* Bm = Pk[si][static_cast<size_t>(n)];
                if (rform[i]) {
                    double* T = sc.alloc_n<double>(static_cast<size_t>(q[n] * rkn));
                    GemmProblem p{};
                    p.A = Rinv[i];
                    p.lda = q[n];
                    p.B = Pk[si][static_cast<size_t>(n)];
                    p.ldb = q[n];
                    p.C = T;
                    p.ldc = q[n];
                    p.M = static_cast<int>(q[n]);
                    p.N = static_cast<int>(rkn);
                    p.K = static_cast<int>(q[n]);
                    tp.push_back(p);
                    Bm = T;
                }
                GemmProblem p{};
                p.A = rform[i] ? ypos(s, n) : Uh[i];
                p.lda = dims[n];
                p.B = Bm;
                p.ldb = q[n];
                p.C = r->factors[n];
                p.ldc = dims[n];
                p.M = static_cast<int>(dims[n]);
                p.N = static_cast<int>(rkn);
                p.K = static_cast<int>(q[n]);
                up.push_back(p);
            }
            r->core = bump;
            bump += (csize + 31) / 32 * 32;
            r->arena = arena;
            TS_CUDA_CHECK(cudaMemcpyAsync(r->core, g[si], sizeof(double) * static_cast<size_t>(csize),
                                          cudaMemcpyDeviceToDevice, st));
        }
        if (!tp.empty()) ts::launch_grouped_gemm(Layout::NN, tp, sc, ctx->num_sms);
        ts::launch_grouped_gemm(Layout::NN, up, sc, ctx->num_sms);
    }
    tick("H");
    ctx->launches += sc.launches;
    if (spec) {
        std::vector<int> hf(2 * SD, 0);
        if (dflags) TS_CUDA_CHECK(cudaMemcpyAsync(hf.data(), dflags, sizeof(int) * SD, cudaMemcpyDeviceToHost, st));
        if (gflags) TS_CUDA_CHECK(cudaMemcpyAsync(hf.data() + SD, gflags, sizeof(int) * SD, cudaMemcpyDeviceToHost, st));
        TS_CUDA_CHECK(cudaStreamSynchronize(st));
        for (int x : hf)
            if (x != 0) {  // speculation rejected: redo every sum on the synchronous path
                ctx->spec_ok = false;
                out.clear();
                return segmented_impl(ctx, b, S, seg, weights, widths, seeds, streams, eps, max_rank, false);
            }
    } else {
        ctx->spec_ok = ctx->last_qr_fallbacks == 0 && ctx->last_svd_fallbacks == 0;
    }
    TS_CUDA_CHECK(cudaStreamSynchronize(st));
    std::vector<ts_result*> res(static_cast<size_t>(S));
    for (std::int64_t s = 0; s < S; ++s) res[static_cast<size_t>(s)] = out[static_cast<size_t>(s)].release();
    return res;
}

// Entry of ts_krp_sum / ts_kron_sum / ts_lazy_sum.  A call that repeats an
// earlier one exactly (same batch upload, method, widths, cap, seed, ε) is
// captured into a CUDA graph the second time and replayed from then on (at
// ε > 0 the captured ranks are those of the probe run, and the replay's device
// checks re-derive the reference rank rule and flag any difference): one cudaGraphLaunch instead of ~40
// launches, memsets and descriptor copies, which is what the latency-bound small
// configurations pay for.  The key includes the weights (some launches carry a
// weight as a host scalar).  A replay whose device
// acceptance checks fail is redone on the synchronous path, like any
// speculative call.
ts_result* run_sum(ts_ctx* ctx, const ts_batch* b, const double* weights, const std::int64_t* widths,
                   std::uint64_t seed, std::uint64_t stream, double eps, const std::int64_t* max_rank, Method method) {
    static const bool env_off = [] {
        const char* e = std::getenv("TS_GRAPHS");
        return (e && e[0] == '0') || std::getenv("TS_DEBUG_SWEEPS") != nullptr;
    }();
    const bool graphable = !env_off && ctx->graphs && b != nullptr && weights != nullptr && eps >= 0.0 &&
                           !sharded(ctx) && !ctx->debug && !ctx->timing && ctx->spec_ok && ctx->parent == nullptr;
    // Generic-width stages (wide.cu) synchronise with the host once per
    // Jacobi sweep: such calls are never captured.
    bool wide = false;
    if (graphable && b->order >= 2) {
        for (int n = 0; n < b->order; ++n) {
            const std::int64_t c = method == Method::Lazy ? b->R[n]
                                   : widths == nullptr    ? 0
                                   : method == Method::Krp ? *std::max_element(widths, widths + b->order)
                                                           : complement_product(widths, b->order, n);
            wide = wide || qr_wide_mode(c);
        }
    }
    if (!graphable || wide)
        return sketched_sum_impl(ctx, b, weights, widths, seed, stream, eps, max_rank, method);
    const int d = b->order;
    GraphKey key{b->id, static_cast<int>(method),
                 widths && method != Method::Lazy ? std::vector<std::int64_t>(widths, widths + d) : std::vector<std::int64_t>{},
                 max_rank ? std::vector<std::int64_t>(max_rank, max_rank + d) : std::vector<std::int64_t>{}, seed, stream,
                 eps, std::vector<double>(weights, weights + b->count)};
    auto it = ctx->graph_cache.find(key);
    if (it == ctx->graph_cache.end()) {
        if (!ctx->graph_seen.count(key)) {  // first sighting: plain call (also does one-time setups)
            if (ctx->graph_seen.size() >= 256) ctx->graph_seen.clear();  // bounded: calls that never repeat
            ctx->graph_seen.insert(key);
            return sketched_sum_impl(ctx, b, weights, widths, seed, stream, eps, max_rank, method);
        }
        // Second sighting: run it plainly once more to learn the output ranks, then capture.
        std::unique_ptr<ts_result> probe(sketched_sum_impl(ctx, b, weights, widths, seed, stream, eps, max_rank, method));
        if (!ctx->spec_ok) return probe.release();  // the speculative path was rejected: no graph
        auto ge = std::make_unique<GraphEntry>();
        ge->order = d;
        ge->count = b->count;
        TS_CUDA_CHECK(cudaMalloc(&ge->d_w, sizeof(double) * static_cast<size_t>(b->count)));
        TS_CUDA_CHECK(cudaMallocHost(&ge->h_w, sizeof(double) * static_cast<size_t>(b->count)));
        TS_CUDA_CHECK(cudaMallocHost(&ge->h_flags, sizeof(int) * 2 * TS_MAX_ORDER));
        std::int64_t csize = 1;
        for (int n = 0; n < d; ++n) {
            ge->dims[n] = probe->dims[n];
            ge->ranks[n] = probe->ranks[n];
            csize *= probe->ranks[n];
            TS_CUDA_CHECK(cudaMalloc(&ge->out_f[n], sizeof(double) * static_cast<size_t>(probe->dims[n] * probe->ranks[n])));
        }
        TS_CUDA_CHECK(cudaMalloc(&ge->out_core, sizeof(double) * static_cast<size_t>(csize)));
        ge->stage.reserve(2 * ctx->stage.footprint() + (size_t(1) << 20));
        TS_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        cudaStream_t st = ctx->stream;
        TS_CUDA_CHECK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        cudaGraph_t graph = nullptr;
        try {
            sketched_sum_impl(ctx, b, weights, widths, seed, stream, eps, max_rank, method, true, nullptr, ge.get());
        } catch (...) {
            cudaStreamEndCapture(st, &graph);
            if (graph) cudaGraphDestroy(graph);
            ctx->graphs = false;  // do not try again on this context
            return probe.release();
        }
        const cudaError_t e1 = cudaStreamEndCapture(st, &graph);
        const cudaError_t e2 = e1 == cudaSuccess ? cudaGraphInstantiate(&ge->exec, graph, 0) : e1;
        if (graph) cudaGraphDestroy(graph);
        if (e2 != cudaSuccess) {  // not capturable here: stay on plain launches
            (void)cudaGetLastError();
            ge->exec = nullptr;
            ctx->graphs = false;
            return probe.release();
        }
        if (ctx->graph_cache.size() >= 8) {  // bounded cache: evict the least recently used
            auto lru = ctx->graph_cache.begin();
            for (auto g = ctx->graph_cache.begin(); g != ctx->graph_cache.end(); ++g)
                if (g->second->last_use < lru->second->last_use) lru = g;
            ctx->graph_cache.erase(lru);
        }
        it = ctx->graph_cache.emplace(key, std::move(ge)).first;
        return probe.release();
    }
    GraphEntry& ge = *it->second;
    if (b->count != ge.count) invalid("sum request needs matching, nonempty summands and weights");
    for (std::int64_t i = 0; i < b->count; ++i)
        if (!std::isfinite(weights[i])) invalid("weights must be finite");
    ge.last_use = ++ctx->graph_clock;
    TS_CUDA_CHECK(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    std::memcpy(ge.h_w, weights, sizeof(double) * static_cast<size_t>(b->count));
    TS_CUDA_CHECK(cudaMemcpyAsync(ge.d_w, ge.h_w, sizeof(double) * static_cast<size_t>(b->count), cudaMemcpyHostToDevice, st));
    std::memset(ge.h_flags, 0, sizeof(int) * 2 * TS_MAX_ORDER);
    TS_CUDA_CHECK(cudaGraphLaunch(ge.exec, st));
    auto res = std::make_unique<ts_result>();
    res->device = ctx->device;
    res->stream = st;
    res->order = d;
    std::int64_t csize = 1;
    for (int n = 0; n < d; ++n) {
        res->dims[n] = ge.dims[n];
        res->ranks[n] = ge.ranks[n];
        csize *= ge.ranks[n];
        const size_t bytes = sizeof(double) * static_cast<size_t>(ge.dims[n] * ge.ranks[n]);
        TS_CUDA_CHECK(cudaMallocAsync(&res->factors[n], bytes, st));
        TS_CUDA_CHECK(cudaMemcpyAsync(res->factors[n], ge.out_f[n], bytes, cudaMemcpyDeviceToDevice, st));
    }
    TS_CUDA_CHECK(cudaMallocAsync(&res->core, sizeof(double) * static_cast<size_t>(csize), st));
    TS_CUDA_CHECK(cudaMemcpyAsync(res->core, ge.out_core, sizeof(double) * static_cast<size_t>(csize),
                                  cudaMemcpyDeviceToDevice, st));
    TS_CUDA_CHECK(cudaStreamSynchronize(st));
    ctx->launches += ge.launches;
    ++ctx->graph_replays;
    for (int i = 0; i < 2 * d; ++i)
        if (ge.h_flags[i] != 0) {  // speculation rejected: redo synchronously
            ctx->spec_ok = false;
            res.reset();
            return sketched_sum_impl(ctx, b, weights, widths, seed, stream, eps, max_rank, method, false);
        }
    return res.release();
}

}  // namespace

extern "C" {

const char* ts_last_error(void) { return g_err.c_str(); }
const char* ts_version(void) { return "tucksum-b200 0.1 (sm_100a)"; }

int ts_ctx_create(int device, ts_ctx** out) {
    return guarded([&] {
        if (out == nullptr) invalid("ts_ctx_create: null out");
        int ndev = 0;
        TS_CUDA_CHECK(cudaGetDeviceCount(&ndev));
        if (device < 0 || device >= ndev) invalid("ts_ctx_create: no such device");
        TS_CUDA_CHECK(cudaSetDevice(device));
        auto ctx = std::make_unique<ts_ctx>();
        ctx->device = device;
        TS_CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        {   // The side stream carries stage D's short latency-bound chain next to stage E's
            // machine-filling GEMM: highest priority, so its CTAs are placed first.
            int lo_prio = 0, hi_prio = 0;
            TS_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
            TS_CUDA_CHECK(cudaStreamCreateWithPriority(&ctx->side, cudaStreamNonBlocking, hi_prio));
        }
        TS_CUDA_CHECK(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
        TS_CUDA_CHECK(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
        TS_CUDA_CHECK(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
        cudaMemPool_t pool;
        TS_CUDA_CHECK(cudaDeviceGetDefaultMemPool(&pool, device));
        std::uint64_t thresh = std::numeric_limits<std::uint64_t>::max();
        TS_CUDA_CHECK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh));
        *out = ctx.release();
    });
}

int ts_ctx_destroy(ts_ctx* ctx) {
    return guarded([&] {
        if (!ctx) return;
        for (ts_ctx* lane : ctx->lanes) ts_ctx_destroy(lane);
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        ctx->graph_cache.clear();
        for (auto& kv : ctx->omega) cudaFree(kv.second.ptr);
        for (auto& kv : ctx->oz_cache) {
            cudaFree(kv.second.slices);
            cudaFree(kv.second.exp);
        }
        for (auto& e : ctx->events) cudaEventDestroy(e);
        if (ctx->comm && nccl_api().CommDestroy) nccl_api().CommDestroy(ctx->comm);
        cudaStreamSynchronize(ctx->side);
        cudaEventDestroy(ctx->ev_fork);
        cudaEventDestroy(ctx->ev_join);
        cudaStreamDestroy(ctx->side);
        cudaStreamDestroy(ctx->stream);
        delete ctx;
    });
}

int ts_nccl_unique_id(void* unique_id_128) {
    return guarded([&] {
        ncclUniqueId id;
        nccl_check(nccl_api().GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(unique_id_128, &id, sizeof(id));
    });
}

int ts_ctx_init_nccl(ts_ctx* ctx, const void* unique_id_128, int nranks, int rank) {
    return guarded([&] {
        if (!ctx || !unique_id_128 || nranks < 1 || rank < 0 || rank >= nranks) invalid("ts_ctx_init_nccl: bad arguments");
        if (ctx->host_ar) invalid("ts_ctx_init_nccl: context already has a host all-reduce");
        TS_CUDA_CHECK(cudaSetDevice(ctx->device));
        ncclUniqueId id;
        std::memcpy(&id, unique_id_128, sizeof(id));
        nccl_check(nccl_api().CommInitRank(&ctx->comm, nranks, id, rank), "ncclCommInitRank");
        ctx->nranks = nranks;
        ctx->rank = rank;
    });
}

int ts_ctx_set_host_allreduce(ts_ctx* ctx, ts_host_allreduce_fn fn, void* user, int nranks, int rank) {
    return guarded([&] {
        if (!ctx || nranks < 1 || rank < 0 || rank >= nranks) invalid("ts_ctx_set_host_allreduce: bad arguments");
        if (ctx->comm) invalid("ts_ctx_set_host_allreduce: context already has a NCCL communicator");
        ctx->host_ar = fn;
        ctx->host_ar_user = fn ? user : nullptr;
        ctx->nranks = fn ? nranks : 1;
        ctx->rank = fn ? rank : 0;
    });
}

int ts_ctx_comm_info(ts_ctx* ctx, int* nranks, int* rank) {
    return guarded([&] {
        if (!ctx || !nranks || !rank) invalid("ts_ctx_comm_info: null argument");
        *nranks = ctx->nranks;
        *rank = ctx->rank;
        if (!ctx->comm) return;
        NcclApi& api = nccl_api();
        if (!api.CommCount || !api.CommUserRank) throw ts::Error(TS_NCCL, "libnccl.so.2 lacks ncclCommCount");
        nccl_check(api.CommCount(ctx->comm, nranks), "ncclCommCount");
        nccl_check(api.CommUserRank(ctx->comm, rank), "ncclCommUserRank");
    });
}

void* ts_ctx_stream(ts_ctx* ctx) { return ctx ? ctx->stream : nullptr; }
int64_t ts_ctx_launch_count(ts_ctx* ctx) { return ctx ? ctx->launches : 0; }

int ts_ctx_last_paths(ts_ctx* ctx, int* qr_fallback_modes, int* svd_fallback_modes) {
    return guarded([&] {
        if (!ctx) invalid("null context");
        if (qr_fallback_modes) *qr_fallback_modes = ctx->last_qr_fallbacks;
        if (svd_fallback_modes) *svd_fallback_modes = ctx->last_svd_fallbacks;
    });
}

int ts_ctx_last_int8_stages(ts_ctx* ctx) { return ctx ? static_cast<int>(ctx->last_int8_stages) : 0; }

int ts_ctx_set_debug(ts_ctx* ctx, int enabled) {
    return guarded([&] {
        if (!ctx) invalid("null context");
        ctx->debug = enabled != 0;
    });
}
int ts_ctx_set_graphs(ts_ctx* ctx, int enabled) {
    return guarded([&] {
        if (!ctx) invalid("ts_ctx_set_graphs: null context");
        ctx->graphs = enabled != 0;
        if (!ctx->graphs) {
            ctx->graph_cache.clear();
            ctx->graph_seen.clear();
        }
    });
}
int64_t ts_ctx_graph_replays(ts_ctx* ctx) { return ctx ? ctx->graph_replays : 0; }
int ts_ctx_set_timing(ts_ctx* ctx, int enabled) {
    return guarded([&] {
        if (!ctx) invalid("null context");
        ctx->timing = enabled != 0;
    });
}
int ts_ctx_stage_times(ts_ctx* ctx, double* ms, int cap) {
    if (!ctx) return 0;
    const int n = std::min<int>(cap, static_cast<int>(ctx->stage_ms.size()));
    for (int i = 0; i < n; ++i) ms[i] = ctx->stage_ms[static_cast<size_t>(i)];
    return n;
}

int ts_batch_upload(ts_ctx* ctx, const ts_tucker_view* xs, int64_t count, ts_batch** out) {
    return guarded([&] {
        if (!ctx || !out) invalid("ts_batch_upload: null argument");
        if (count < 1 || xs == nullptr) invalid("sum request needs matching, nonempty summands and weights");
        const ts_tucker_view& x0 = xs[0];
        const int d = static_cast<int>(x0.order);
        if (d < 1) invalid("TuckerTensor: order must be >= 1");
        if (d > TS_MAX_ORDER) throw ts::Error(TS_UNSUPPORTED, "order exceeds TS_MAX_ORDER");
        auto b = std::make_unique<ts_batch>();
        static std::atomic<std::uint64_t> next_id{1};
        b->id = next_id++;
        b->ctx = ctx;
        b->order = d;
        b->count = count;
        for (int j = 0; j < d; ++j) b->dims[j] = x0.dims[j];
        // Structure validation (src/tucker.cpp:16-55) and dims agreement (src/sketch.cpp:23-28).
        std::int64_t core_elems = 0;
        for (std::int64_t i = 0; i < count; ++i) {
            const ts_tucker_view& x = xs[i];
            if (x.order != d) invalid("sum request summands must share dims");
            for (int j = 0; j < d; ++j) {
                if (x.dims[j] != b->dims[j]) invalid("sum request summands must share dims");
                if (x.dims[j] < 1 || x.ranks[j] < 1) invalid("TuckerTensor: dims and ranks must be positive");
                if (x.factors == nullptr || x.factors[j] == nullptr) invalid("TuckerTensor: one factor matrix per mode required");
            }
            if (x.num_blocks < 1) invalid("TuckerTensor: core needs at least one block");
            std::int64_t cursor[TS_MAX_ORDER] = {};
            for (std::int64_t bl = 0; bl < x.num_blocks; ++bl) {
                std::int64_t e = 1;
                for (int j = 0; j < d; ++j) {
                    if (x.block_offsets[bl * d + j] != cursor[j]) invalid("TuckerTensor: blocks must tile the super-diagonal");
                    const std::int64_t ext = x.block_shapes[bl * d + j];
                    if (ext < 1) invalid("DenseTensor: every dimension must be >= 1");
                    cursor[j] += ext;
                    e *= ext;
                }
                if (x.block_data == nullptr || x.block_data[bl] == nullptr) invalid("TuckerTensor: null block data");
                core_elems += e;
            }
            for (int j = 0; j < d; ++j)
                if (cursor[j] != x.ranks[j]) invalid("TuckerTensor: blocks must span the full rank box");
            for (int j = 0; j < d; ++j) b->R[j] += x.ranks[j];
        }
        b->scol.assign(static_cast<size_t>((count + 1) * d), 0);
        for (std::int64_t i = 0; i < count; ++i)
            for (int j = 0; j < d; ++j)
                b->scol[static_cast<size_t>((i + 1) * d + j)] = b->scol[static_cast<size_t>(i * d + j)] + xs[i].ranks[j];
        TS_CUDA_CHECK(cudaSetDevice(ctx->device));
        cudaStream_t st = ctx->stream;
        std::int64_t bytes = 0;
        for (int j = 0; j < d; ++j) {
            TS_CUDA_CHECK(cudaMallocAsync(&b->F[j], sizeof(double) * static_cast<size_t>(b->dims[j] * b->R[j]), st));
            bytes += sizeof(double) * b->dims[j] * b->R[j];
        }
        TS_CUDA_CHECK(cudaMallocAsync(&b->cores, sizeof(double) * static_cast<size_t>(std::max<std::int64_t>(core_elems, 1)), st));
        bytes += sizeof(double) * core_elems;
        b->core_elems = core_elems;
        // Copies; adjacent host ranges (e.g. one pinned slab per mode) are merged.
        struct Run {
            const double* src = nullptr;
            double* dst = nullptr;
            std::int64_t n = 0;
        };
        auto flush = [&](Run& r) {
            if (r.n > 0)
                TS_CUDA_CHECK(cudaMemcpyAsync(r.dst, r.src, sizeof(double) * static_cast<size_t>(r.n),
                                              cudaMemcpyHostToDevice, st));
            r = Run{};
        };
        auto add = [&](Run& r, const double* src, double* dst, std::int64_t n) {
            if (r.n > 0 && r.src + r.n == src && r.dst + r.n == dst) {
                r.n += n;
                return;
            }
            flush(r);
            r.src = src;
            r.dst = dst;
            r.n = n;
        };
        std::int64_t col[TS_MAX_ORDER] = {};
        for (int j = 0; j < d; ++j) {
            Run run;
            std::int64_t c = 0;
            for (std::int64_t i = 0; i < count; ++i) {
                add(run, xs[i].factors[j], b->F[j] + c * b->dims[j], b->dims[j] * xs[i].ranks[j]);
                c += xs[i].ranks[j];
            }
            flush(run);
        }
        Run crun;
        std::int64_t coff = 0;
        for (std::int64_t i = 0; i < count; ++i) {
            const ts_tucker_view& x = xs[i];
            for (std::int64_t bl = 0; bl < x.num_blocks; ++bl) {
                ts::Atom at{};
                at.summand = static_cast<int>(i);
                at.core_off = coff;
                std::int64_t e = 1;
                for (int j = 0; j < d; ++j) {
                    at.col[j] = static_cast<int>(col[j] + x.block_offsets[bl * d + j]);
                    at.shape[j] = static_cast<int>(x.block_shapes[bl * d + j]);
                    e *= at.shape[j];
                    b->max_shape = std::max(b->max_shape, at.shape[j]);
                }
                add(crun, x.block_data[bl], b->cores + coff, e);
                coff += e;
                b->atoms.push_back(at);
            }
            for (int j = 0; j < d; ++j) col[j] += x.ranks[j];
        }
        flush(crun);
        TS_CUDA_CHECK(cudaMallocAsync(&b->d_atoms, sizeof(ts::Atom) * b->atoms.size(), st));
        TS_CUDA_CHECK(cudaMemcpyAsync(b->d_atoms, b->atoms.data(), sizeof(ts::Atom) * b->atoms.size(),
                                      cudaMemcpyHostToDevice, st));
        bytes += sizeof(ts::Atom) * b->atoms.size();
        TS_CUDA_CHECK(cudaStreamSynchronize(st));
        b->bytes = bytes;
        *out = b.release();
    });
}

// Summands already in the stacked formal-sum layout on the host (per mode one
// n_j × R_j column-major slab, dense cores concatenated in summand order): one
// H2D copy per mode plus one for the cores, no per-summand views.
int ts_batch_upload_stacked(ts_ctx* ctx, int64_t order, const int64_t* dims, int64_t count, const int64_t* ranks,
                            const double* const* factors, const double* cores, ts_batch** out) {
    return guarded([&] {
        if (!ctx || !out || !dims || !ranks || !factors || !cores) invalid("ts_batch_upload_stacked: null argument");
        if (count < 1) invalid("sum request needs matching, nonempty summands and weights");
        if (order < 1) invalid("TuckerTensor: order must be >= 1");
        if (order > TS_MAX_ORDER) throw ts::Error(TS_UNSUPPORTED, "order exceeds TS_MAX_ORDER");
        const int d = static_cast<int>(order);
        auto b = std::make_unique<ts_batch>();
        static std::atomic<std::uint64_t> next_id{1u << 30};
        b->id = next_id++;
        b->ctx = ctx;
        b->order = d;
        b->count = count;
        std::int64_t core_elems = 0;
        b->atoms.resize(static_cast<size_t>(count));
        for (int j = 0; j < d; ++j) {
            if (dims[j] < 1) invalid("TuckerTensor: dims and ranks must be positive");
            if (factors[j] == nullptr) invalid("TuckerTensor: one factor matrix per mode required");
            b->dims[j] = dims[j];
        }
        b->scol.assign(static_cast<size_t>((count + 1) * d), 0);
        for (std::int64_t i = 0; i < count; ++i) {
            ts::Atom& at = b->atoms[static_cast<size_t>(i)];
            at.summand = static_cast<int>(i);
            at.core_off = core_elems;
            std::int64_t e = 1;
            for (int j = 0; j < d; ++j) {
                const std::int64_t r = ranks[i * d + j];
                b->scol[static_cast<size_t>((i + 1) * d + j)] = b->scol[static_cast<size_t>(i * d + j)] + std::max<std::int64_t>(r, 0);
                if (r < 1) invalid("TuckerTensor: dims and ranks must be positive");
                at.col[j] = static_cast<int>(b->R[j]);
                at.shape[j] = static_cast<int>(r);
                b->R[j] += r;
                b->max_shape = std::max(b->max_shape, at.shape[j]);
                e *= r;
            }
            core_elems += e;
        }
        TS_CUDA_CHECK(cudaSetDevice(ctx->device));
        cudaStream_t st = ctx->stream;
        std::int64_t bytes = 0;
        for (int j = 0; j < d; ++j) {
            const size_t n = sizeof(double) * static_cast<size_t>(b->dims[j] * b->R[j]);
            TS_CUDA_CHECK(cudaMallocAsync(&b->F[j], n, st));
            TS_CUDA_CHECK(cudaMemcpyAsync(b->F[j], factors[j], n, cudaMemcpyHostToDevice, st));
            bytes += static_cast<std::int64_t>(n);
        }
        TS_CUDA_CHECK(cudaMallocAsync(&b->cores, sizeof(double) * static_cast<size_t>(core_elems), st));
        TS_CUDA_CHECK(cudaMemcpyAsync(b->cores, cores, sizeof(double) * static_cast<size_t>(core_elems),
                                      cudaMemcpyHostToDevice, st));
        b->core_elems = core_elems;
        bytes += sizeof(double) * core_elems;
        TS_CUDA_CHECK(cudaMallocAsync(&b->d_atoms, sizeof(ts::Atom) * b->atoms.size(), st));
        TS_CUDA_CHECK(cudaMemcpyAsync(b->d_atoms, b->atoms.data(), sizeof(ts::Atom) * b->atoms.size(),
                                      cudaMemcpyHostToDevice, st));
        bytes += sizeof(ts::Atom) * b->atoms.size();
        TS_CUDA_CHECK(cudaStreamSynchronize(st));
        b->bytes = bytes;
        *out = b.release();
    });
}

int ts_batch_free(ts_batch* b) {
    return guarded([&] {
        if (!b) return;
        cudaSetDevice(b->ctx->device);
        // Graphs captured on this batch can never replay again: release them
        // (and the memory their allocation nodes reserve).
        for (auto it = b->ctx->graph_cache.begin(); it != b->ctx->graph_cache.end();)
            it = it->first.batch == b->id ? b->ctx->graph_cache.erase(it) : std::next(it);
        cudaStream_t st = b->ctx->stream;  // stream-ordered: safe while kernels are still queued
        for (auto* f : b->F)
            if (f) cudaFreeAsync(f, st);
        for (auto* e : b->aexp)
            if (e) cudaFreeAsync(e, st);
        for (auto* e : b->rexp)
            if (e) cudaFreeAsync(e, st);
        if (b->cores) cudaFreeAsync(b->cores, st);
        if (b->d_atoms) cudaFreeAsync(b->d_atoms, st);
        delete b;
    });
}

int64_t ts_batch_count(const ts_batch* b) { return b ? b->count : 0; }
int64_t ts_batch_bytes(const ts_batch* b) { return b ? b->bytes : 0; }

void ts_substream(uint64_t seed, uint64_t stream, uint64_t salt, uint64_t* out_seed, uint64_t* out_stream) {
    ts::substream(seed, stream, salt, out_seed, out_stream);
}

int ts_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, uint64_t stream, double* out) {
    return guarded([&] {
        if (rows < 0 || cols < 0) invalid("gaussian_matrix: negative extent");
        ts::gaussian_fill(rows, cols, seed, stream, out);
    });
}

int ts_omega_prepare(ts_ctx* ctx, int64_t order, const int64_t* dims, int64_t width, uint64_t seed, uint64_t stream) {
    return guarded([&] {
        if (!ctx || order < 1 || order > TS_MAX_ORDER || width < 1) invalid("ts_omega_prepare: bad arguments");
        TS_CUDA_CHECK(cudaSetDevice(ctx->device));
        const std::vector<std::int64_t> wv(static_cast<size_t>(order), width);
        omega_get(ctx, static_cast<int>(order), dims, wv.data(), seed, stream);
    });
}

int ts_krp_sum(ts_ctx* ctx, const ts_batch* batch, const double* weights, const int64_t* widths, uint64_t seed,
               uint64_t stream, double eps, const int64_t* max_rank, ts_result** out) {
    return guarded([&] {
        if (!ctx || !out) invalid("ts_krp_sum: null argument");
        *out = run_sum(ctx, batch, weights, widths, seed, stream, eps, max_rank, Method::Krp);
    });
}

int ts_kron_sum(ts_ctx* ctx, const ts_batch* batch, const double* weights, const int64_t* widths, uint64_t seed,
                uint64_t stream, double eps, const int64_t* max_rank, ts_result** out) {
    return guarded([&] {
        if (!ctx || !out) invalid("ts_kron_sum: null argument");
        *out = run_sum(ctx, batch, weights, widths, seed, stream, eps, max_rank, Method::Kron);
    });
}

int ts_krp_sum_segmented(ts_ctx* ctx, const ts_batch* batch, int64_t nsums, const int64_t* segments,
                         const double* weights, const int64_t* widths, const uint64_t* seeds, const uint64_t* streams,
                         double eps, const int64_t* max_rank, ts_result** out) {
    return guarded([&] {
        if (!ctx || !out || !segments) invalid("ts_krp_sum_segmented: null argument");
        for (int64_t i = 0; i < nsums; ++i) out[i] = nullptr;
        std::vector<ts_result*> r =
            segmented_impl(ctx, batch, nsums, segments, weights, widths, seeds, streams, eps, max_rank, true);
        for (int64_t i = 0; i < nsums; ++i) out[i] = r[static_cast<size_t>(i)];
    });
}

int ts_tucker_norm(ts_ctx* ctx, const ts_batch* batch, const double* weights, double* out) {
    return guarded([&] {
        if (!ctx || !out) invalid("ts_tucker_norm: null argument");
        if (sharded(ctx)) throw ts::Error(TS_UNSUPPORTED, "tucker_norm does not shard: use a context without NCCL");
        sketched_sum_impl(ctx, batch, weights, nullptr, 0, 0, 0.0, nullptr, Method::Lazy, false, out);
    });
}

int ts_tucker_inner(ts_ctx* ctx, const ts_batch* x, const double* wx, const ts_batch* y, const double* wy,
                    double* out) {
    return guarded([&] {
        if (!ctx || !out) invalid("ts_tucker_inner: null argument");
        if (sharded(ctx)) throw ts::Error(TS_UNSUPPORTED, "tucker_inner of sharded batches: use a context without NCCL");
        *out = inner_impl(ctx, x, wx, y, wy);
    });
}

int ts_rel_error_to_sum(ts_ctx* ctx, const ts_result* r, const ts_batch* batch, const double* weights, double* out) {
    return guarded([&] {
        if (!ctx || !r || !out) invalid("ts_rel_error_to_sum: null argument");
        if (r->device != ctx->device) invalid("ts_rel_error_to_sum: result lives on another device than this context's");
        if (sharded(ctx)) throw ts::Error(TS_UNSUPPORTED, "rel_error_to_sum of a sharded batch: use a context without NCCL");
        ResultView rv(ctx, r);
        const double one = 1.0;
        const double xx = inner_impl(ctx, &rv.b, &one, &rv.b, &one);
        const double xs = inner_impl(ctx, &rv.b, &one, batch, weights);
        const double ss = inner_impl(ctx, batch, weights, batch, weights);
        const double diff = std::sqrt(std::max(xx - 2.0 * xs + ss, 0.0));
        *out = ss > 0.0 ? diff / std::sqrt(ss) : diff;  // src/tucker.cpp:298-303
    });
}

int ts_lazy_sum(ts_ctx* ctx, const ts_batch* batch, const double* weights, double eps, const int64_t* max_rank,
                ts_result** out) {
    return guarded([&] {
        if (!ctx || !out) invalid("ts_lazy_sum: null argument");
        if (sharded(ctx)) throw ts::Error(TS_UNSUPPORTED, "lazy rounding does not shard: use a context without NCCL");
        *out = run_sum(ctx, batch, weights, nullptr, 0, 0, eps, max_rank, Method::Lazy);
    });
}

// Independent sums (one round_sum per NDG node, many
// GMRES steps).  Small sums are latency-bound — one CTA runs the eigensolver
// while the rest of the GPU idles — so they run side by side: sum i goes to lane
// i mod L, each lane a child context with its own stream driven by its own host
// thread.  Every sum computes exactly what ts_krp_sum computes (bitwise).  With
// a NCCL communicator the sums run in order on the context itself (collectives
// must be issued in the same order on every rank).
int ts_krp_sum_many(ts_ctx* ctx, int64_t count, const ts_batch* const* batches, const double* const* weights,
                    const int64_t* widths, const uint64_t* seeds, const uint64_t* streams, double eps,
                    const int64_t* max_rank, int lanes, ts_result** out) {
    return guarded([&] {
        if (!ctx || !out || count < 0 || (count > 0 && (!batches || !weights || !seeds || !streams)))
            invalid("ts_krp_sum_many: null argument");
        for (int64_t i = 0; i < count; ++i) out[i] = nullptr;
        if (count == 0) return;
        if (sharded(ctx) || count == 1 || lanes <= 1) {
            for (int64_t i = 0; i < count; ++i)
                out[i] = sketched_sum_impl(ctx, batches[i], weights[i], widths, seeds[i], streams[i], eps, max_rank, Method::Krp);
            return;
        }
        const int L = static_cast<int>(std::min<int64_t>(std::min(lanes, 16), count));
        {  // Ω entries fetched by the lanes stay resident until every lane is done
            std::lock_guard<std::mutex> lock(ctx->omega_mu);
            ctx->omega_pin = ctx->omega_clock + 1;
        }
        struct Unpin {
            ts_ctx* c;
            ~Unpin() {
                std::lock_guard<std::mutex> lock(c->omega_mu);
                c->omega_pin = ~std::uint64_t(0);
            }
        } unpin{ctx};
        TS_CUDA_CHECK(cudaSetDevice(ctx->device));
        TS_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));  // batches were uploaded on this stream
        while (static_cast<int>(ctx->lanes.size()) < L) {
            ts_ctx* lane = nullptr;
            if (ts_ctx_create(ctx->device, &lane) != TS_OK) throw ts::Error(TS_RUNTIME, g_err);
            lane->parent = ctx;
            ctx->lanes.push_back(lane);
        }
        std::vector<std::string> errs(static_cast<size_t>(L));
        std::vector<int> codes(static_cast<size_t>(L), TS_OK);
        std::vector<std::thread> workers;
        for (int t = 0; t < L; ++t)
            workers.emplace_back([&, t] {
                ts_ctx* lane = ctx->lanes[static_cast<size_t>(t)];
                codes[static_cast<size_t>(t)] = guarded([&] {
                    TS_CUDA_CHECK(cudaSetDevice(lane->device));
                    for (int64_t i = t; i < count; i += L)
                        out[i] = sketched_sum_impl(lane, batches[i], weights[i], widths, seeds[i], streams[i], eps, max_rank, Method::Krp);
                });
                if (codes[static_cast<size_t>(t)] != TS_OK) errs[static_cast<size_t>(t)] = g_err;
            });
        for (auto& w : workers) w.join();
        for (int t = 0; t < L; ++t)
            if (codes[static_cast<size_t>(t)] != TS_OK) {
                for (int64_t i = 0; i < count; ++i) {
                    delete out[i];
                    out[i] = nullptr;
                }
                throw ts::Error(codes[static_cast<size_t>(t)], errs[static_cast<size_t>(t)]);
            }
    });
}

// Plan stage (src/sketch.cpp:272-349, Strategy::Krp).  The spectrum of the Gram
// of the energy-weighted stacked factors V_n = F_n·diag(e) is obtained as the
// squared singular values of V_n (TSQR + Jacobi on device), with the reference's
// floor / tail rule applied on the returned values.
static void plan_targets(ts_ctx* ctx, const ts_batch* b, const double* weights, double eps, const int64_t* oversampling,
                         int64_t* effective_ranks, int64_t* targets) {
    {
        if (!ctx || !b || !weights || !oversampling) invalid("sum request needs matching, nonempty summands and weights");
        if (b->ctx->device != ctx->device) invalid("batch was uploaded to another device than this context's");
        if (!(eps >= 0.0)) invalid("tolerance must be nonnegative");
        const int d = b->order;
        for (int n = 0; n < d; ++n)
            if (oversampling[n] < 0) invalid("oversampling must be nonnegative");
        TS_CUDA_CHECK(cudaSetDevice(ctx->device));
        ctx->stage.reset();
        CallScratch sc(ctx->stream, ctx->stage);
        if (b->core_norm.empty()) {  // per-summand ‖core‖_F, computed once on the device
            double* d_sq = sc.alloc_n<double>(b->atoms.size());
            ts::launch_atom_sumsq(b->cores, b->d_atoms, static_cast<int>(b->atoms.size()), d, d_sq, sc);
            std::vector<double> sq(b->atoms.size());
            TS_CUDA_CHECK(cudaMemcpyAsync(sq.data(), d_sq, sizeof(double) * sq.size(), cudaMemcpyDeviceToHost, ctx->stream));
            TS_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
            auto* bm = const_cast<ts_batch*>(b);
            bm->core_norm.assign(static_cast<size_t>(b->count), 0.0);
            for (size_t a = 0; a < b->atoms.size(); ++a) bm->core_norm[static_cast<size_t>(b->atoms[a].summand)] += sq[a];
            for (double& v : bm->core_norm) v = std::sqrt(v);
        }
        std::vector<double> energy(static_cast<size_t>(b->count));
        for (std::int64_t i = 0; i < b->count; ++i)
            energy[static_cast<size_t>(i)] = std::fabs(weights[i]) * b->core_norm[static_cast<size_t>(i)];
        for (int n = 0; n < d; ++n) {
            const std::int64_t rows = b->dims[n], R = b->R[n];
            const std::int64_t small = std::min(rows, R);
            // Per-column energy scale.
            std::vector<double> cscale(static_cast<size_t>(R));
            // Column ranges per summand follow the stacking order.
            {
                std::vector<std::int64_t> rk(static_cast<size_t>(b->count), 0);
                for (const auto& at : b->atoms) rk[static_cast<size_t>(at.summand)] += at.shape[n];
                std::int64_t c = 0;
                for (std::int64_t i = 0; i < b->count; ++i)
                    for (std::int64_t t = 0; t < rk[static_cast<size_t>(i)]; ++t) cscale[static_cast<size_t>(c++)] = energy[static_cast<size_t>(i)];
            }
            auto* d_scale = static_cast<double*>(sc.upload(cscale.data(), sizeof(double) * static_cast<size_t>(R)));
            const bool tall = rows >= R;
            double* V = sc.alloc_n<double>(static_cast<size_t>(rows * R));
            ts::launch_scale_columns(b->F[n], rows, R, d_scale, V, !tall, sc);
            const std::int64_t m = tall ? rows : R, cols = tall ? R : rows;
            double* sigma = sc.alloc_n<double>(static_cast<size_t>(cols));
            bool gram_values = false;  // sigma holds Gram eigenvalues (λ = σ²) instead of σ
            if (qr_wide_mode(cols) && cols <= 128) {
                // The reference's own formulation (src/sketch.cpp:311): eigenvalues of
                // the Gram VᵀV (DMMA GEMM) by the one-CTA values-only solver.
                double* G = sc.alloc_n<double>(static_cast<size_t>(cols * cols));
                GemmProblem p{};
                p.A = p.B = V;
                p.lda = p.ldb = m;
                p.C = G;
                p.ldc = cols;
                p.M = p.N = static_cast<int>(cols);
                p.K = static_cast<int>(m);
                ts::launch_grouped_gemm(Layout::TN, {p}, sc, ctx->num_sms);
                ts::launch_sym_eigvals(G, cols, static_cast<int>(cols), sigma, sc);
                gram_values = true;
            } else if (qr_wide_mode(cols)) {  // any width: block one-sided Jacobi on V itself (wide.cu)
                ts::bosj_svd(V, m, m, cols, sigma, nullptr, 0, sc, ctx->num_sms);
            } else {
                ts::TsqrPlan plan = ts::plan_tsqr(V, m, m, cols, nullptr, 0, sc);
                ts::run_tsqr({&plan}, sc, false);
                double* U = sc.alloc_n<double>(static_cast<size_t>(cols * cols));
                ts::launch_jacobi_svd(plan.Rtop, plan.kk, static_cast<int>(plan.kk), static_cast<int>(cols), sigma, U, sc);
            }
            std::vector<double> sig(static_cast<size_t>(cols));
            TS_CUDA_CHECK(cudaMemcpyAsync(sig.data(), sigma, sizeof(double) * static_cast<size_t>(cols),
                                          cudaMemcpyDeviceToHost, ctx->stream));
            TS_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
            // Eigenvalues of VᵀV (R of them; the R - cols missing ones are zero).
            std::vector<double> lam(static_cast<size_t>(R), 0.0);
            for (std::int64_t j = 0; j < cols; ++j)
                lam[static_cast<size_t>(j)] = gram_values ? std::max(sig[static_cast<size_t>(j)], 0.0)  // cwiseMax(0), src/sketch.cpp:312
                                                          : sig[static_cast<size_t>(j)] * sig[static_cast<size_t>(j)];
            const double lmax = lam.empty() ? 0.0 : lam[0];
            const double floor = static_cast<double>(R) * std::numeric_limits<double>::epsilon() * lmax;
            for (double& l : lam)
                if (l < floor) l = 0.0;
            std::vector<double> suffix(static_cast<size_t>(R) + 1, 0.0);
            for (std::int64_t j = R - 1; j >= 0; --j) suffix[static_cast<size_t>(j)] = suffix[static_cast<size_t>(j) + 1] + lam[static_cast<size_t>(j)];
            const double thresh = eps * eps / static_cast<double>(d) * suffix[0];
            std::int64_t keep = R;
            for (std::int64_t r = 1; r <= R; ++r)
                if (suffix[static_cast<size_t>(r)] <= thresh) {
                    keep = r;
                    break;
                }
            effective_ranks[n] = keep;
            std::int64_t target = keep + oversampling[n];
            target = std::min({target, b->dims[n], complement_product(b->dims, d, n)});
            targets[n] = std::max<std::int64_t>(target, 1);
        }
        ctx->launches += sc.launches;
        TS_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    }
}

// Reference kron_sketch_dims (src/sketch.cpp:222-270): balanced widths whose
// complementary products cover the targets, then a deterministic repair.
static std::vector<std::int64_t> kron_sketch_dims(const std::vector<std::int64_t>& targets,
                                                  const std::vector<std::int64_t>& dims) {
    const size_t n = targets.size();
    if (n < 2 || n != dims.size()) invalid("kron_sketch_dims: need order >= 2 and matching dims");
    for (size_t i = 0; i < n; ++i) {
        if (targets[i] < 1 || dims[i] < 1) invalid("kron_sketch_dims: targets and dims must be positive");
        if (targets[i] > complement_product(dims.data(), static_cast<int>(n), static_cast<int>(i)))
            invalid("kron_sketch_dims: target exceeds attainable mode rank");
    }
    long double logp = 0.0L;
    for (std::int64_t t : targets) logp += std::log(static_cast<long double>(t));
    const long double root = std::exp(logp / static_cast<long double>(n - 1));
    std::vector<std::int64_t> s(n);
    for (size_t i = 0; i < n; ++i) {
        long double q = root / static_cast<long double>(targets[i]);
        const long double snapped = std::round(q);
        if (snapped >= 1.0L && std::fabs(q - snapped) < 1e-9L) q = snapped;
        const auto si = static_cast<std::int64_t>(std::ceil(static_cast<double>(q)));
        s[i] = std::clamp<std::int64_t>(si, 1, dims[i]);
    }
    bool changed = true;
    while (changed) {
        changed = false;
        for (size_t m = 0; m < n; ++m) {
            while (complement_product(s.data(), static_cast<int>(n), static_cast<int>(m)) < targets[m]) {
                size_t pick = n;
                for (size_t j = 0; j < n; ++j) {
                    if (j == m || s[j] >= dims[j]) continue;
                    if (pick == n || s[j] < s[pick]) pick = j;
                }
                if (pick == n) throw ts::Error(TS_RUNTIME, "kron_sketch_dims: infeasible despite capped targets");
                ++s[pick];
                changed = true;
            }
        }
    }
    return s;
}

int ts_effective_subrank(ts_ctx* ctx, const ts_batch* b, const double* weights, double eps, const int64_t* oversampling,
                         int64_t* effective_ranks, int64_t* targets, int64_t* widths) {
    return guarded([&] {
        plan_targets(ctx, b, weights, eps, oversampling, effective_ranks, targets);
        const std::int64_t smax = *std::max_element(targets, targets + b->order);  // src/sketch.cpp:342-344
        for (int n = 0; n < b->order; ++n) widths[n] = smax;
    });
}

int ts_effective_subrank_kron(ts_ctx* ctx, const ts_batch* b, const double* weights, double eps,
                              const int64_t* oversampling, int64_t* effective_ranks, int64_t* targets, int64_t* widths) {
    return guarded([&] {
        plan_targets(ctx, b, weights, eps, oversampling, effective_ranks, targets);
        const int d = b->order;
        const std::vector<std::int64_t> w = kron_sketch_dims(std::vector<std::int64_t>(targets, targets + d),
                                                             std::vector<std::int64_t>(b->dims, b->dims + d));
        std::copy(w.begin(), w.end(), widths);  // src/sketch.cpp:340-341
    });
}

int ts_kron_sketch_dims(int64_t order, const int64_t* targets, const int64_t* dims, int64_t* out) {
    return guarded([&] {
        if (order < 0 || (order > 0 && (!targets || !dims || !out))) invalid("kron_sketch_dims: null argument");
        const size_t o = static_cast<size_t>(order);
        const std::vector<std::int64_t> w =
            kron_sketch_dims(std::vector<std::int64_t>(targets, targets + o), std::vector<std::int64_t>(dims, dims + o));
        std::copy(w.begin(), w.end(), out);
    });
}

void tsi_read_eig_profile(long long* out);
// Debug: phase clock totals of the last n ≤ 64 values-kernel run (TS_EIG_PROFILE=1).
int ts_debug_eig_profile(long long* out17) {  // 18 entries
    return guarded([&] { tsi_read_eig_profile(out17); });
}

// Symmetric eigensolver of the ST-HOSVD fast path (reference sym_eig,
// src/kernels.cpp:70-86): host in / host out; also reports sweeps and kernel ms.
int ts_sym_eig(ts_ctx* ctx, int64_t n, const double* a, double* values, double* vectors, int* sweeps, double* ms) {
    return guarded([&] {
        if (!ctx || n < 1) invalid("ts_sym_eig: need n >= 1");
        TS_CUDA_CHECK(cudaSetDevice(ctx->device));
        ctx->stage.reset();
        CallScratch sc(ctx->stream, ctx->stage);
        auto* dA = static_cast<double*>(sc.upload(a, sizeof(double) * static_cast<size_t>(n * n)));
        double* dl = sc.alloc_n<double>(static_cast<size_t>(n));
        double* dV = sc.alloc_n<double>(static_cast<size_t>(n * n));
        int* dsw = sc.alloc_n<int>(1);
        cudaEvent_t e0, e1;
        TS_CUDA_CHECK(cudaEventCreate(&e0));
        TS_CUDA_CHECK(cudaEventCreate(&e1));
        TS_CUDA_CHECK(cudaEventRecord(e0, ctx->stream));
        int hs = 0;
        if (qr_wide_mode(n)) {  // block one-sided Jacobi of the (PSD) matrix (wide.cu)
            hs = ts::bosj_svd(dA, n, n, n, dl, dV, n, sc, ctx->num_sms);
            TS_CUDA_CHECK(cudaMemsetAsync(dsw, 0, sizeof(int), ctx->stream));
        } else {
            ts::launch_sym_jacobi(dA, n, static_cast<int>(n), dl, dV, sc, dsw);
        }
        TS_CUDA_CHECK(cudaEventRecord(e1, ctx->stream));
        const int bosj_sweeps = hs;
        TS_CUDA_CHECK(cudaMemcpyAsync(values, dl, sizeof(double) * static_cast<size_t>(n), cudaMemcpyDeviceToHost, ctx->stream));
        TS_CUDA_CHECK(cudaMemcpyAsync(vectors, dV, sizeof(double) * static_cast<size_t>(n * n), cudaMemcpyDeviceToHost, ctx->stream));
        TS_CUDA_CHECK(cudaMemcpyAsync(&hs, dsw, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        TS_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        float t = 0.f;
        TS_CUDA_CHECK(cudaEventElapsedTime(&t, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (sweeps) *sweeps = qr_wide_mode(n) ? bosj_sweeps : hs;
        if (ms) *ms = t;
    });
}

// Debug / test hook of the Ozaki GEMM (ozaki.cu): out (N × M, ld N) = Fᵀ·B for
// host F (K × M) and B (K × N, N ≤ 64), column-major.  Returns TS_UNSUPPORTED
// when the kernel is disabled (TS_OZAKI=0).
int ts_debug_ozaki_gemm(ts_ctx* ctx, int64_t K, int64_t M, int64_t N, const double* F, const double* B, double* out,
                        double* ms) {
    return guarded([&] {
        if (!ctx || K < 1 || M < 1 || N < 1 || N > 64 || !F || !B || !out) invalid("ts_debug_ozaki_gemm: bad arguments");
        TS_CUDA_CHECK(cudaSetDevice(ctx->device));
        ctx->stage.reset();
        CallScratch sc(ctx->stream, ctx->stage);
        auto* dF = static_cast<double*>(sc.upload(F, sizeof(double) * static_cast<size_t>(K * M)));
        auto* dB = static_cast<double*>(sc.upload(B, sizeof(double) * static_cast<size_t>(K * N)));
        double* dC = sc.alloc_n<double>(static_cast<size_t>(N * M));
        int* aexp = sc.alloc_n<int>(static_cast<size_t>(M));
        ts::launch_col_exponents(dF, K, K, M, aexp, sc);
        ts::OzOperand bo = ts::prepare_ozaki_b(dB, K, static_cast<int>(K), static_cast<int>(N), sc);
        ts::OzProblem p{};
        p.F = dF;
        p.ldf = K;
        p.aexp = aexp;
        p.M = static_cast<int>(M);
        p.K = static_cast<int>(K);
        p.B = bo;
        p.C = dC;
        p.ldc = N;
        cudaEvent_t e0, e1;
        TS_CUDA_CHECK(cudaEventCreate(&e0));
        TS_CUDA_CHECK(cudaEventCreate(&e1));
        TS_CUDA_CHECK(cudaEventRecord(e0, ctx->stream));
        int launched = 0;
        if (!ts::launch_ozaki_gemm({p}, sc, ctx->num_sms, &launched))
            throw ts::Error(TS_UNSUPPORTED, "ozaki GEMM not available for these operands");
        TS_CUDA_CHECK(cudaEventRecord(e1, ctx->stream));
        TS_CUDA_CHECK(cudaMemcpyAsync(out, dC, sizeof(double) * static_cast<size_t>(N * M), cudaMemcpyDeviceToHost,
                                      ctx->stream));
        TS_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        float t = 0.f;
        TS_CUDA_CHECK(cudaEventElapsedTime(&t, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (ms) *ms = t;
    });
}

// Same engine in the stage-C orientation: out (M × N, column-major) = A·Btᵀ for
// host A (M × K, column-major: M contiguous) and Bt (N × K, N ≤ 64).
int ts_debug_ozaki_gemm_nt(ts_ctx* ctx, int64_t M, int64_t K, int64_t N, const double* A, const double* Bt, double* out,
                           double* ms) {
    return guarded([&] {
        if (!ctx || K < 1 || M < 1 || N < 1 || N > 64 || !A || !Bt || !out) invalid("ts_debug_ozaki_gemm_nt: bad arguments");
        TS_CUDA_CHECK(cudaSetDevice(ctx->device));
        ctx->stage.reset();
        CallScratch sc(ctx->stream, ctx->stage);
        auto* dA = static_cast<double*>(sc.upload(A, sizeof(double) * static_cast<size_t>(K * M)));
        auto* dB = static_cast<double*>(sc.upload(Bt, sizeof(double) * static_cast<size_t>(K * N)));
        double* dC = sc.alloc_n<double>(static_cast<size_t>(N * M));
        int* aexp = sc.alloc_n<int>(static_cast<size_t>(M));
        ts::launch_row_exponents(dA, M, M, K, aexp, sc);
        ts::OzOperand bo = ts::prepare_ozaki_b(dB, N, static_cast<int>(K), static_cast<int>(N), sc, true);
        ts::OzProblem p{};
        p.F = dA;
        p.ldf = M;
        p.aexp = aexp;
        p.M = static_cast<int>(M);
        p.K = static_cast<int>(K);
        p.B = bo;
        p.C = dC;
        p.ldc = M;
        p.a_mn = true;
        p.c_colmajor = true;
        cudaEvent_t e0, e1;
        TS_CUDA_CHECK(cudaEventCreate(&e0));
        TS_CUDA_CHECK(cudaEventCreate(&e1));
        TS_CUDA_CHECK(cudaEventRecord(e0, ctx->stream));
        int launched = 0;
        if (!ts::launch_ozaki_gemm({p}, sc, ctx->num_sms, &launched))
            throw ts::Error(TS_UNSUPPORTED, "ozaki GEMM not available for these operands");
        TS_CUDA_CHECK(cudaEventRecord(e1, ctx->stream));
        TS_CUDA_CHECK(cudaMemcpyAsync(out, dC, sizeof(double) * static_cast<size_t>(N * M), cudaMemcpyDeviceToHost,
                                      ctx->stream));
        TS_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        float t = 0.f;
        TS_CUDA_CHECK(cudaEventElapsedTime(&t, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (ms) *ms = t;
    });
}

// The tridiagonalization eigensolver alone (eig_tri.cu), host in / host out;
// *flag = 1 when its acceptance check rejected the result.
int ts_sym_eig_tri(ts_ctx* ctx, int64_t n, const double* a, double* values, double* vectors, int* flag, double* ms) {
    return guarded([&] {
        if (!ctx || n < 1 || n > 64) invalid("ts_sym_eig_tri: need 1 <= n <= 64");
        double* dres = nullptr;
        TS_CUDA_CHECK(cudaSetDevice(ctx->device));
        ctx->stage.reset();
        CallScratch sc(ctx->stream, ctx->stage);
        auto* dA = static_cast<double*>(sc.upload(a, sizeof(double) * static_cast<size_t>(n * n)));
        double* dl = sc.alloc_n<double>(static_cast<size_t>(n));
        double* dV = sc.alloc_n<double>(static_cast<size_t>(n * n));
        int* df = sc.alloc_n<int>(1);
        TS_CUDA_CHECK(cudaMemsetAsync(df, 0, sizeof(int), ctx->stream));
        cudaEvent_t e0, e1;
        TS_CUDA_CHECK(cudaEventCreate(&e0));
        TS_CUDA_CHECK(cudaEventCreate(&e1));
        TS_CUDA_CHECK(cudaEventRecord(e0, ctx->stream));
        dres = sc.alloc_n<double>(1);
        ts::launch_sym_trd(dA, n, static_cast<int>(n), dl, dV, df, dres, sc);
        TS_CUDA_CHECK(cudaEventRecord(e1, ctx->stream));
        int hf = 0;
        TS_CUDA_CHECK(cudaMemcpyAsync(values, dl, sizeof(double) * static_cast<size_t>(n), cudaMemcpyDeviceToHost, ctx->stream));
        TS_CUDA_CHECK(cudaMemcpyAsync(vectors, dV, sizeof(double) * static_cast<size_t>(n * n), cudaMemcpyDeviceToHost, ctx->stream));
        TS_CUDA_CHECK(cudaMemcpyAsync(&hf, df, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        TS_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        float t = 0.f;
        TS_CUDA_CHECK(cudaEventElapsedTime(&t, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (flag) *flag = hf;
        if (ms) *ms = t;
    });
}

int64_t ts_result_order(const ts_result* r) { return r ? r->order : 0; }
void ts_result_dims(const ts_result* r, int64_t* dims) {
    for (int n = 0; n < r->order; ++n) dims[n] = r->dims[n];
}
void ts_result_ranks(const ts_result* r, int64_t* ranks) {
    for (int n = 0; n < r->order; ++n) ranks[n] = r->ranks[n];
}
// Device → caller buffer.  Pageable destinations go through a pinned staging
// buffer (one per thread, grown on demand): a direct pageable copy runs at a
// fraction of the link rate.  Registered / pinned destinations are copied to
// directly.
static void download(double* out, const double* src, size_t n, cudaStream_t st) {
    const size_t bytes = sizeof(double) * n;
    if (bytes == 0) return;
    cudaPointerAttributes attr{};
    const bool pinned = cudaPointerGetAttributes(&attr, out) == cudaSuccess && attr.type == cudaMemoryTypeHost;
    cudaGetLastError();  // pageable pointers may set a sticky-free error on some drivers
    if (pinned || bytes < (64u << 10)) {
        TS_CUDA_CHECK(cudaMemcpyAsync(out, src, bytes, cudaMemcpyDeviceToHost, st));
        TS_CUDA_CHECK(cudaStreamSynchronize(st));
        return;
    }
    struct Staging {
        void* p = nullptr;
        size_t cap = 0;
        ~Staging() {
            if (p) cudaFreeHost(p);
        }
    };
    thread_local Staging stage;
    if (stage.cap < bytes) {
        if (stage.p) TS_CUDA_CHECK(cudaFreeHost(stage.p));
        stage.p = nullptr;
        stage.cap = 0;
        TS_CUDA_CHECK(cudaMallocHost(&stage.p, bytes));
        stage.cap = bytes;
    }
    TS_CUDA_CHECK(cudaMemcpyAsync(stage.p, src, bytes, cudaMemcpyDeviceToHost, st));
    TS_CUDA_CHECK(cudaStreamSynchronize(st));
    std::memcpy(out, stage.p, bytes);
}

int ts_result_factor(const ts_result* r, int64_t mode, double* out) {
    return guarded([&] {
        if (!r || mode < 0 || mode >= r->order) invalid("ts_result_factor: bad mode");
        TS_CUDA_CHECK(cudaSetDevice(r->device));
        download(out, r->factors[mode], static_cast<size_t>(r->dims[mode] * r->ranks[mode]), r->stream);
    });
}
int ts_result_core(const ts_result* r, double* out) {
    return guarded([&] {
        if (!r) invalid("ts_result_core: null result");
        std::int64_t n = 1;
        for (int k = 0; k < r->order; ++k) n *= r->ranks[k];
        TS_CUDA_CHECK(cudaSetDevice(r->device));
        download(out, r->core, static_cast<size_t>(n), r->stream);
    });
}
const double* ts_result_factor_device(const ts_result* r, int64_t mode) {
    return (r && mode >= 0 && mode < r->order) ? r->factors[mode] : nullptr;
}
const double* ts_result_core_device(const ts_result* r) { return r ? r->core : nullptr; }

int64_t ts_result_intermediate(const ts_result* r, int which, int64_t mode, double* out, int64_t* rows, int64_t* cols) {
    if (!r) return -1;
    if (which == 3) {
        if (out) std::memcpy(out, r->h.data(), sizeof(double) * r->h.size());
        if (rows) *rows = static_cast<int64_t>(r->h.size());
        if (cols) *cols = 1;
        return static_cast<int64_t>(r->h.size());
    }
    if (which < 0 || which > 2 || mode < 0 || mode >= r->order) return -1;
    const auto& v = r->inter[which][mode];
    if (out) std::memcpy(out, v.data(), sizeof(double) * v.size());
    if (rows) *rows = r->inter_rows[which][mode];
    if (cols) *cols = r->inter_cols[which][mode];
    return static_cast<int64_t>(v.size());
}

int ts_result_free(ts_result* r) {
    return guarded([&] { delete r; });
}

}  // extern "C"
