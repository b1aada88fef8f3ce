// runtime.cpp — pinned descriptor staging and stream-ordered call scratch.
#include "runtime.hpp"

#include <algorithm>
#include <cstdio>
#include <mutex>
#include <set>
#include <utility>

#include "../../include/tucksum_cuda.h"

namespace ts {

void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
    char buf[512];
    std::snprintf(buf, sizeof buf, "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e), cudaGetErrorString(e), file,
                  line, what);
    throw Error(e == cudaErrorMemoryAllocation ? TS_OOM : TS_CUDA, buf);
}

void set_max_smem(const void* kernel, int bytes) {
    static std::mutex mu;
    static std::set<std::pair<int, const void*>> done;
    int dev = 0;
    TS_CUDA_CHECK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    if (!done.insert({dev, kernel}).second) return;
    const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) {
        done.erase({dev, kernel});
        throw_cuda(e, "cudaFuncSetAttribute(MaxDynamicSharedMemorySize)", __FILE__, __LINE__);
    }
}

HostStage::~HostStage() {
    for (auto& c : retired_) cudaFreeHost(c.p);
    if (buf_) cudaFreeHost(buf_);
}

void HostStage::reset() {
    for (auto& c : retired_) cudaFreeHost(c.p);
    retired_.clear();
    used_ = 0;
}

void* HostStage::put(const void* src, size_t bytes) {
    const size_t need = (bytes + 255) & ~size_t(255);
    if (used_ + need > cap_) {
        if (buf_) retired_.push_back({buf_, cap_});
        cap_ = std::max<size_t>(need, std::max<size_t>(cap_ * 2, size_t(1) << 20));
        TS_CUDA_CHECK(cudaMallocHost(reinterpret_cast<void**>(&buf_), cap_));
        used_ = 0;
    }
    char* p = buf_ + used_;
    used_ += need;
    std::memcpy(p, src, bytes);
    return p;
}

size_t HostStage::footprint() const {
    size_t f = used_;
    for (const auto& c : retired_) f += c.cap;
    return f;
}

void HostStage::reserve(size_t bytes) {
    if (cap_ - used_ >= bytes) return;
    if (buf_) retired_.push_back({buf_, cap_});
    cap_ = std::max<size_t>(bytes, size_t(1) << 20);
    TS_CUDA_CHECK(cudaMallocHost(reinterpret_cast<void**>(&buf_), cap_));
    used_ = 0;
}

CallScratch::~CallScratch() {
    for (void* p : ptrs_) cudaFreeAsync(p, stream_);
}

// Bump allocation from stream-ordered chunks: a call makes hundreds of small
// scratch allocations (segmented sums: thousands), and the cost of each
// cudaMallocAsync grows with the number of live pool allocations (measured: a
// 64-sum segmented call spent ~95 ms of host time in ~2000 of them for ~1 ms of
// kernels).  Large requests keep their own allocation.
void* CallScratch::alloc(size_t bytes) {
    constexpr size_t kChunk = size_t(4) << 20, kAlign = 256;
    bytes = (std::max<size_t>(bytes, 1) + kAlign - 1) & ~(kAlign - 1);
    if (bytes > kChunk / 4) {
        void* p = nullptr;
        TS_CUDA_CHECK(cudaMallocAsync(&p, bytes, stream_));
        ptrs_.push_back(p);
        return p;
    }
    if (cur_ == nullptr || cur_ + bytes > end_) {
        void* c = nullptr;
        TS_CUDA_CHECK(cudaMallocAsync(&c, kChunk, stream_));
        ptrs_.push_back(c);
        cur_ = static_cast<char*>(c);
        end_ = cur_ + kChunk;
    }
    void* p = cur_;
    cur_ += bytes;
    return p;
}

void* CallScratch::upload(const void* src, size_t bytes) {
    void* host = stage_.put(src, bytes);
    void* dev = alloc(bytes);
    TS_CUDA_CHECK(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, stream_));
    return dev;
}

}  // namespace ts
