// Shared host-side helpers for the B200 FlashSinkhorn engine.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <thread>
#include <vector>
#include <cstdlib>
#include <stdexcept>
#include <string>

namespace fskb {

// Exceptions used inside the library; capi.cpp maps them to status codes.
struct ValidationFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NumericalFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw CudaFailure(std::string(what) + ": " + cudaGetErrorString(e));
}
#define FSKB_CUDA(call) ::fskb::cuda_check((call), #call)

// Device-status bits written by kernels (atomicOr into a device int).
enum : int {
    kFlagNonFinitePotential = 1,
    kFlagTransportOverflow = 2,
    kFlagNonFiniteTransport = 4,
    kFlagNonFiniteRowMarginal = 8,
    kFlagNonFiniteColMarginal = 16,
};

// Large caller-buffer copies through pooled pinned staging (hostcopy.cpp);
// synchronous with respect to the host buffer (it may be reused on return).
void copy_host_to_device(void* dst, const void* src, std::size_t bytes, cudaStream_t s);
void copy_device_to_host(void* dst, const void* src, std::size_t bytes, cudaStream_t s);
// true for page-locked host memory (cudaHostAlloc / cudaHostRegister): copies DMA directly
bool host_pinned(const void* p);
// pooled page-locked host buffers (hostcopy.cpp; C ABI fsk_host_alloc / fsk_host_free)
void* host_alloc(std::size_t bytes);
void host_free(void* p);
// RAII page-locked host array from that pool
template <typename T>
class PinnedHost {
public:
    PinnedHost() = default;
    explicit PinnedHost(std::size_t n) : p_(static_cast<T*>(host_alloc(n * sizeof(T)))) {}
    ~PinnedHost() { host_free(p_); }
    PinnedHost(const PinnedHost&) = delete;
    PinnedHost& operator=(const PinnedHost&) = delete;
    PinnedHost(PinnedHost&& o) noexcept : p_(o.p_) { o.p_ = nullptr; }
    PinnedHost& operator=(PinnedHost&& o) noexcept {
        if (this != &o) {
            host_free(p_);
            p_ = o.p_;
            o.p_ = nullptr;
        }
        return *this;
    }
    T* get() const { return p_; }

private:
    T* p_ = nullptr;
};

// Faults in and page-locks a caller's output buffer (>= 64 MB) from a background
// host thread (hostcopy.cpp). join() before writing it; pinned() then says whether a
// plain cudaMemcpyAsync may DMA into it; release() (also in the destructor) unlocks.
class HostPrefault {
public:
    HostPrefault() = default;
    HostPrefault(const HostPrefault&) = delete;
    HostPrefault& operator=(const HostPrefault&) = delete;
    ~HostPrefault() { release(); }
    void start(void* p, std::size_t bytes);
    void join();
    bool pinned() const { return pinned_; }
    void release();

private:
    std::thread th_;
    void* p_ = nullptr;
    std::size_t bytes_ = 0;
    bool pinned_ = false;
    bool external_ = false;   // page-locked by the caller: never unregistered here
};

// Owner teardown after a full device synchronize: the buffers may have been
// allocated on caller streams that no longer exist, so frees inside the scope go
// to the legacy default stream.
struct DevBufTeardown {
    bool prev;
    DevBufTeardown() : prev(active()) { active() = true; }
    ~DevBufTeardown() { active() = prev; }
    static bool& active() {
        thread_local bool a = false;
        return a;
    }
};

// Plain owning device buffer (stream-ordered allocation). A regrow frees the old
// block on the stream of the regrowing call: callers that switch streams order
// the new stream after the old one first (the engine's stream fence).
template <typename T>
class DevBuf {
public:
    DevBuf() = default;
    DevBuf(std::size_t n, cudaStream_t s) { alloc(n, s); }
    ~DevBuf() { release(); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_), s_(o.s_) { o.p_ = nullptr; o.n_ = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p_ = o.p_;
            n_ = o.n_;
            s_ = o.s_;
            o.p_ = nullptr;
            o.n_ = 0;
        }
        return *this;
    }
    void alloc(std::size_t n, cudaStream_t s) {
        release(s);
        s_ = s;
        n_ = n;
        if (n) FSKB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p_), n * sizeof(T), s));
    }
    void release() { release(s_); }
    void release(cudaStream_t s) {
        if (p_) cudaFreeAsync(p_, DevBufTeardown::active() ? cudaStream_t(nullptr) : s);
        p_ = nullptr;
        n_ = 0;
    }
    T* get() const { return p_; }
    std::size_t size() const { return n_; }
    void upload(const T* host, std::size_t n) {
        if (n) copy_host_to_device(p_, host, n * sizeof(T), s_);
    }
    // completes before returning for large copies (staged), else stream-ordered
    void download(T* host, std::size_t n) const {
        if (n) copy_device_to_host(host, p_, n * sizeof(T), s_);
    }
    void zero() {
        if (n_) FSKB_CUDA(cudaMemsetAsync(p_, 0, n_ * sizeof(T), s_));
    }

private:
    T* p_ = nullptr;
    std::size_t n_ = 0;
    cudaStream_t s_ = nullptr;
};

// Grow-only device scratch per host thread and device for the large per-call
// partial buffers of the transport kernels (GBs at cfg3): a fresh stream-ordered
// allocation of that size can make the pool map new memory (measured 0-400 ms per
// call through the C ABI). Uses on different streams are ordered by an event.
class Scratch {
public:
    // pointer to >= bytes of device memory, ordered after the previous use
    void* get(std::size_t bytes, cudaStream_t s);
    // marks the end of this use (enqueued work on s that reads or writes it)
    void done(cudaStream_t s);
    static Scratch& local();   // this thread's scratch on the current device
    ~Scratch();

private:
    void* p_ = nullptr;
    std::size_t n_ = 0;
    int dev_ = -1;
    cudaEvent_t ev_ = nullptr;
    bool pending_ = false;
};

// Global launch counter (the bench reports how many of our kernels ran).
std::atomic<int64_t>& launch_counter();   // (batch workers launch from several threads)
inline void count_launch(int k = 1) { launch_counter().fetch_add(k, std::memory_order_relaxed); }

// Negative-control toggle (fsk::stream::debug_break_lse).
bool& break_lse_flag();

int num_sms();

// FSK_TIMING=1: host wall-clock per solve phase on stderr (synchronizes the stream).
struct PhaseTimer {
    bool on;
    cudaStream_t s;
    std::chrono::steady_clock::time_point t0;
    explicit PhaseTimer(cudaStream_t st)
        : on(std::getenv("FSK_TIMING") && std::getenv("FSK_TIMING")[0] != '0'), s(st) {
        t0 = std::chrono::steady_clock::now();
    }
    void mark(const char* what) {
        if (!on) return;
        cudaStreamSynchronize(s);
        const auto t1 = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[fsk timing] %-24s %9.3f ms\n", what,
                     std::chrono::duration<double, std::milli>(t1 - t0).count());
        t0 = t1;
    }
};


}  // namespace fskb
