// runtime.h — engine handle and buffer helpers shared by the host-side
// translation units of the C ABI (host_runtime.cpp, host_decide.cpp).
#pragma once
#include <cuda_runtime.h>

#include <sched.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "dev_types.h"
#include "migsched_b200.h"

namespace msgk {

// Persistent fork-join pool for the host-side staging / decoding loops: the
// workers are created once (threads_for_this_process() - 1).  A parallel
// region is published through an atomic generation counter; workers spin on
// it for a short while after each region (kSpinNs) before blocking on a
// condition variable, so the back-to-back regions of one msg_run_batch call
// (a validation pass per pipeline chunk, then the decode) cost no futex
// wake-ups, and an idle engine costs no CPU.  One parallel region at a time
// (calls from several host threads serialise on the pool).
class HostPool {
  public:
    static HostPool& get() {
        static HostPool p;
        return p;
    }
    unsigned size() const { return (unsigned)workers_.size() + 1; }
    // Runs body() on `n` threads (the caller included) and returns when all finished.
    template <class B>
    void run(unsigned n, B&& body) {
        std::lock_guard<std::mutex> one(region_);
        n = std::min(n, size());
        if (n <= 1) {
            body();
            return;
        }
        std::function<void()> fn = [&body]() { body(); };
        body_ = &fn;
        left_.store(n - 1, std::memory_order_relaxed);
        want_.store((int)n - 1, std::memory_order_release);  // publishes body_ and left_ to the claimers
        gen_.fetch_add(1);  // seq_cst with the sleeper count below (Dekker pair with loop())
        if (sleeping_.load() > 0) {
            std::lock_guard<std::mutex> lk(m_);
            cv_.notify_all();
        }
        body();
        while (left_.load(std::memory_order_acquire) != 0) pause();
        body_ = nullptr;
    }
    ~HostPool() {
        stop_.store(true, std::memory_order_release);
        gen_.fetch_add(1, std::memory_order_release);
        {
            std::lock_guard<std::mutex> lk(m_);
            cv_.notify_all();
        }
        for (auto& t : workers_) t.join();
    }

  private:
    static constexpr int64_t kSpinNs = 300000;  // 0.3 ms of spinning after a region
    static void pause() {
#if defined(__x86_64__) || defined(__i386__)
        __builtin_ia32_pause();
#endif
    }
    HostPool() {
        const unsigned hw = threads_for_this_process();
        for (unsigned i = 1; i < hw; ++i) workers_.emplace_back([this] { loop(); });
    }
    // MSG_HOST_THREADS, else the CPUs this process may run on (affinity
    // mask), shared evenly among the processes of one node under torchrun
    // (LOCAL_WORLD_SIZE): one process per GPU must not oversubscribe the host.
    static unsigned threads_for_this_process() {
        if (const char* e = std::getenv("MSG_HOST_THREADS")) {
            const long v = std::strtol(e, nullptr, 10);
            if (v > 0) return (unsigned)std::min(v, 1024L);
        }
        unsigned n = std::max(1u, std::thread::hardware_concurrency());
        cpu_set_t set;
        if (sched_getaffinity(0, sizeof(set), &set) == 0) n = std::max(1, CPU_COUNT(&set));
        if (const char* e = std::getenv("LOCAL_WORLD_SIZE")) {
            const long w = std::strtol(e, nullptr, 10);
            if (w > 1) n = std::max(1u, n / (unsigned)w);
        }
        return n;
    }
    void loop() {
        uint64_t seen = 0;  // the constructor's generation: a region published before this thread ran is still claimed
        for (;;) {
            // wait for the next generation: spin, then block
            uint64_t g = gen_.load(std::memory_order_acquire);
            if (g == seen) {
                const auto t0 = std::chrono::steady_clock::now();
                unsigned k = 0;
                while ((g = gen_.load(std::memory_order_acquire)) == seen) {
                    pause();
                    if ((++k & 255u) == 0 &&
                        std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0)
                                .count() > kSpinNs) {
                        std::unique_lock<std::mutex> lk(m_);
                        sleeping_.fetch_add(1);  // seq_cst: run() either sees the sleeper or we see its generation
                        cv_.wait(lk, [&] { return gen_.load() != seen; });
                        sleeping_.fetch_sub(1, std::memory_order_acq_rel);
                        g = gen_.load(std::memory_order_acquire);
                        break;
                    }
                }
            }
            seen = g;
            if (stop_.load(std::memory_order_acquire)) return;
            if (want_.fetch_sub(1, std::memory_order_acq_rel) <= 0) continue;  // region already fully staffed
            (*body_)();
            left_.fetch_sub(1, std::memory_order_acq_rel);
        }
    }
    std::vector<std::thread> workers_;
    std::mutex m_, region_;
    std::condition_variable cv_;
    std::function<void()>* body_ = nullptr;
    std::atomic<uint64_t> gen_{0};
    std::atomic<int> want_{0};
    std::atomic<unsigned> left_{0};
    std::atomic<int> sleeping_{0};
    std::atomic<bool> stop_{false};
};

template <class F>
void parallel_for(uint32_t n, uint32_t min_per_thread, F&& f) {
    HostPool& pool = HostPool::get();
    const uint32_t threads = std::min(pool.size(), std::max(1u, n / std::max(1u, min_per_thread)));
    if (threads <= 1) {
        for (uint32_t i = 0; i < n; ++i) f(i);
        return;
    }
    std::atomic<uint32_t> next{0};
    pool.run(threads, [&]() {
        for (;;) {
            const uint32_t base = next.fetch_add(16);
            if (base >= n) return;
            const uint32_t end = std::min(n, base + 16);
            for (uint32_t i = base; i < end; ++i) f(i);
        }
    });
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
        if (e != cudaSuccess) return e;
        // Defined contents from the start: result buffers are copied back
        // by capacity (event / scratch records a run did not write), and
        // compute-sanitizer initcheck holds every copied byte to that.
        // Only on growth; ordered before any stream's later work.
        e = cudaMemset(p, 0, want);
        if (e == cudaSuccess) e = cudaStreamSynchronize(cudaStreamLegacy);
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

namespace msgk {
// Device pointers of one multi-GPU launch (host_peer.cpp): every group's
// inbox (peer-mapped), and group 0's job rows / summary / timeline.
struct PeerBinding {
    uint32_t world = 1, rank = 0, epoch = 0;
    void* inbox[kMaxDev] = {};
    void* jobs = nullptr;
    void* summary = nullptr;
    void* timeline = nullptr;
};
}  // namespace msgk

struct msg_engine {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t staged = nullptr;  // stage_impl's copies on `stream` (the pipelined path waits on it)
    msgk::DevBuf tables;
    msgk::DevBuf score_tab;  // the arrival scorer's per-word table (host_tables.h, build_score_table)
    msgk::DevBuf flush;
    uint64_t launches = 0;
    std::string last_error;
    int sm_count = 0;
    char name[256] = {0};
    msg_staged* cached = nullptr;
    cudaStream_t pstream[8] = {};  // pipelined msg_run_batch (host_runtime.cpp, run_pipelined)
    cudaEvent_t pevent[8] = {};
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
