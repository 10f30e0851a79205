// runtime.h — engine handle and buffer helpers shared by the host-side
// translation units of the C ABI (host_runtime.cpp, host_decide.cpp).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <string>
#include <thread>
#include <vector>

#include "migsched_b200.h"

namespace msgk {

template <class F>
void parallel_for(uint32_t n, uint32_t min_per_thread, F&& f) {
    uint32_t hw = std::max(1u, std::thread::hardware_concurrency());
    uint32_t threads = std::min(hw, std::max(1u, n / std::max(1u, min_per_thread)));
    if (threads <= 1) {
        for (uint32_t i = 0; i < n; ++i) f(i);
        return;
    }
    std::atomic<uint32_t> next{0};
    auto worker = [&]() {
        for (;;) {
            const uint32_t base = next.fetch_add(16);
            if (base >= n) return;
            const uint32_t end = std::min(n, base + 16);
            for (uint32_t i = base; i < end; ++i) f(i);
        }
    };
    std::vector<std::thread> pool;
    for (uint32_t t = 1; t < threads; ++t) pool.emplace_back(worker);
    worker();
    for (auto& th : pool) th.join();
}

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap && p) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        const size_t want = std::max<size_t>(bytes + bytes / 4, 256);
        cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

struct HostBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap && p) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        const size_t want = std::max<size_t>(bytes + bytes / 4, 256);
        cudaError_t e = cudaMallocHost(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    ~HostBuf() {
        if (p) cudaFreeHost(p);
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

}  // namespace msgk

struct msg_staged;

struct msg_engine {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    msgk::DevBuf tables;
    msgk::DevBuf flush;
    uint64_t launches = 0;
    std::string last_error;
    int sm_count = 0;
    char name[256] = {0};
    msg_staged* cached = nullptr;
    msgk::DevBuf dscr[12];  // decision-level scratch (host_decide.cpp)
    msgk::HostBuf hscr[4];
};


namespace msgk {

inline msg_status cuda_fail(msg_engine* e, cudaError_t err, const char* what) {
    if (e) e->last_error = std::string("CudaError: ") + what + ": " + cudaGetErrorString(err);
    return MSG_ERR_CUDA;
}

#define CK(expr)                                                   \
    do {                                                           \
        cudaError_t _e = (expr);                                   \
        if (_e != cudaSuccess) return cuda_fail(eng, _e, #expr);   \
    } while (0)

}  // namespace msgk
