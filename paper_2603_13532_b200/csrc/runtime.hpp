// runtime.hpp — per-call scratch memory and error plumbing for the C ABI.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

namespace ts {

// Error carrying a C-ABI status code (include/tucksum_cuda.h).
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line);

#define TS_CUDA_CHECK(x)                                              \
    do {                                                              \
        cudaError_t e__ = (x);                                        \
        if (e__ != cudaSuccess) ::ts::throw_cuda(e__, #x, __FILE__, __LINE__); \
    } while (0)

#define TS_LAUNCH_CHECK() TS_CUDA_CHECK(cudaGetLastError())

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device setting: applied
// once per (current device, kernel), thread-safe (concurrent lanes, one context
// per GPU in one process).  Must not run inside a graph capture: every kernel
// is first launched by a plain call before any call is captured.
void set_max_smem(const void* kernel, int bytes);
template <class K>
inline void set_max_smem(K* kernel, int bytes) {
    set_max_smem(reinterpret_cast<const void*>(kernel), bytes);
}

// Pinned host staging ring for kernel descriptors: written by the host during a
// call, copied to the device with cudaMemcpyAsync on the call's stream.  Every
// call ends with a stream synchronisation, so the ring restarts at each call.
class HostStage {
public:
    ~HostStage();
    // Called at the start of a call (the previous call ended with a stream sync).
    void reset();
    // Returns a pinned pointer holding a copy of src (bytes), 256-aligned.
    void* put(const void* src, size_t bytes);
    // Upper bound of the bytes the calls since the last reset() staged.
    size_t footprint() const;
    // One pinned buffer of at least `bytes` (so a CUDA-graph capture never has
    // to allocate pinned memory mid-capture).
    void reserve(size_t bytes);

private:
    struct Chunk {
        char* p;
        size_t cap;
    };
    std::vector<Chunk> retired_;  // older chunks kept alive until the next call
    char* buf_ = nullptr;
    size_t cap_ = 0, used_ = 0;
};

// Stream-ordered device scratch for one call (cudaMallocAsync from the device's
// default pool, whose release threshold is raised so memory stays cached).
class CallScratch {
public:
    CallScratch(cudaStream_t s, HostStage& stage) : stream_(s), stage_(stage) {}
    ~CallScratch();
    void* alloc(size_t bytes);
    template <class T>
    T* alloc_n(size_t n) {
        return static_cast<T*>(alloc(n * sizeof(T)));
    }
    // Device copy of a host array (via the pinned stage, async on the stream).
    void* upload(const void* src, size_t bytes);
    cudaStream_t stream() const { return stream_; }
    int64_t launches = 0;
    // Timing hook: when set, the next TMA GEMM launch records these events right
    // before and after its GEMM kernel (not its split-K reduction) and clears the
    // hook — the dominant kernel's own duration for bench.py's roofline.
    cudaEvent_t before_next_gemm = nullptr, after_next_gemm = nullptr;

private:
    cudaStream_t stream_;
    HostStage& stage_;
    std::vector<void*> ptrs_;
    char* cur_ = nullptr;  // bump pointer into the current chunk
    char* end_ = nullptr;
};

}  // namespace ts
