// Host <-> device copies of large caller buffers through pooled pinned staging.
//
// The C ABI receives and returns pageable host doubles (the reference API's
// std::vector / Mat). A plain cudaMemcpy from pageable memory is staged by the
// driver through a bounce buffer with one CPU thread (~6-10 GB/s here). These
// copies stage through our own pinned buffers instead: several host threads fill
// (or drain) one group of staging chunks while the copy engine moves the other
// group, so the host link, not one memcpy thread, sets the pace.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <stdexcept>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "common.h"

namespace fskb {
namespace {

constexpr size_t kChunk = size_t(16) << 20;   // one DMA
constexpr int kPerGroup = 4;                  // chunks per group
constexpr int kGroups = 2;                    // double-buffered groups

struct Staging {
    int dev = -1;
    char* buf[kGroups][kPerGroup] = {};
    cudaEvent_t ev[kGroups][kPerGroup] = {};
};

std::mutex g_mu;
std::vector<Staging*> g_free;

Staging* acquire() {
    int dev = 0;
    FSKB_CUDA(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> lk(g_mu);
        for (size_t i = 0; i < g_free.size(); ++i)
            if (g_free[i]->dev == dev) {
                Staging* s = g_free[i];
                g_free.erase(g_free.begin() + long(i));
                return s;
            }
    }
    auto* s = new Staging();
    s->dev = dev;
    for (int g = 0; g < kGroups; ++g)
        for (int c = 0; c < kPerGroup; ++c) {
            FSKB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s->buf[g][c]), kChunk,
                                    cudaHostAllocDefault));
            FSKB_CUDA(cudaEventCreateWithFlags(&s->ev[g][c], cudaEventDisableTiming));
        }
    return s;
}

void release(Staging* s) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_free.push_back(s);
}

int host_threads() {
    static const int n = int(std::max(1u, std::min(8u, std::thread::hardware_concurrency())));
    return n;
}

// copy bytes [0, len) of the pieces (dst_i, src_i, len_i) with up to T threads
struct Piece {
    char* dst;
    const char* src;
    size_t len;
};
void parallel_copy(const std::vector<Piece>& pieces) {
    size_t total = 0;
    for (auto& p : pieces) total += p.len;
    const int T = int(std::min<size_t>(size_t(host_threads()), (total + (2 << 20) - 1) >> 21));
    auto work = [&](int t) {
        // thread t copies the byte range [t * total / T, (t + 1) * total / T) of the
        // concatenated pieces
        const size_t lo = total * size_t(t) / size_t(T), hi = total * size_t(t + 1) / size_t(T);
        size_t base = 0;
        for (auto& p : pieces) {
            const size_t a = std::max(lo, base), b = std::min(hi, base + p.len);
            if (a < b) std::memcpy(p.dst + (a - base), p.src + (a - base), b - a);
            base += p.len;
        }
    };
    if (T <= 1) {
        work(0);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
}

}  // namespace

bool host_pinned(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

void copy_host_to_device(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes >= (size_t(8) << 20) && host_pinned(src)) {
        // page-locked caller buffer (fsk_host_alloc, cudaHostRegister): one DMA
        FSKB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        FSKB_CUDA(cudaStreamSynchronize(s));
        return;
    }
    if (bytes < (size_t(8) << 20)) {
        FSKB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        return;
    }
    Staging* st = acquire();
    const char* h = static_cast<const char*>(src);
    char* d = static_cast<char*>(dst);
    const size_t group_bytes = kChunk * kPerGroup;
    int g = 0;
    for (size_t off = 0; off < bytes; off += group_bytes, g ^= 1) {
        for (int c = 0; c < kPerGroup; ++c) FSKB_CUDA(cudaEventSynchronize(st->ev[g][c]));
        std::vector<Piece> pieces;
        for (int c = 0; c < kPerGroup; ++c) {
            const size_t o = off + size_t(c) * kChunk;
            if (o >= bytes) break;
            pieces.push_back({st->buf[g][c], h + o, std::min(kChunk, bytes - o)});
        }
        parallel_copy(pieces);
        for (size_t c = 0; c < pieces.size(); ++c) {
            const size_t o = off + c * kChunk;
            FSKB_CUDA(cudaMemcpyAsync(d + o, st->buf[g][c], pieces[c].len, cudaMemcpyHostToDevice,
                                      s));
            FSKB_CUDA(cudaEventRecord(st->ev[g][c], s));
        }
    }
    // the staging buffers go back to the pool only once their copies have landed
    for (int gg = 0; gg < kGroups; ++gg)
        for (int c = 0; c < kPerGroup; ++c) FSKB_CUDA(cudaEventSynchronize(st->ev[gg][c]));
    release(st);
}

void copy_device_to_host(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes < (size_t(8) << 20) || host_pinned(dst)) {
        FSKB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
        FSKB_CUDA(cudaStreamSynchronize(s));
        return;
    }
    Staging* st = acquire();
    char* h = static_cast<char*>(dst);
    const char* d = static_cast<const char*>(src);
    const size_t group_bytes = kChunk * kPerGroup;
    const size_t groups = (bytes + group_bytes - 1) / group_bytes;
    auto issue = [&](size_t gi) {
        const int g = int(gi & 1);
        for (int c = 0; c < kPerGroup; ++c) {
            const size_t o = gi * group_bytes + size_t(c) * kChunk;
            if (o >= bytes) break;
            FSKB_CUDA(cudaMemcpyAsync(st->buf[g][c], d + o, std::min(kChunk, bytes - o),
                                      cudaMemcpyDeviceToHost, s));
            FSKB_CUDA(cudaEventRecord(st->ev[g][c], s));
        }
    };
    issue(0);
    for (size_t gi = 0; gi < groups; ++gi) {
        if (gi + 1 < groups) issue(gi + 1);   // the copy engine runs ahead one group
        const int g = int(gi & 1);
        std::vector<Piece> pieces;
        for (int c = 0; c < kPerGroup; ++c) {
            const size_t o = gi * group_bytes + size_t(c) * kChunk;
            if (o >= bytes) break;
            FSKB_CUDA(cudaEventSynchronize(st->ev[g][c]));
            pieces.push_back({h + o, st->buf[g][c], std::min(kChunk, bytes - o)});
        }
        parallel_copy(pieces);
    }
    release(st);
}

// A fresh output buffer of the caller (e.g. a just-allocated numpy array) is mapped
// page by page on first touch, and a staged download then costs a host memcpy of
// the whole buffer: both land on the critical path and both vary with the host's
// load (0.02-0.5 s for 0.5 GB measured). A background thread faults the pages in
// (with helpers) while the device iterates; with FSK_PIN_OUTPUT=1 it also page-locks
// the buffer so the download is one DMA straight into it (see pinned()).
void HostPrefault::start(void* p, std::size_t bytes) {
    join();
    if (!p || bytes < (std::size_t(64) << 20)) return;
    if (host_pinned(p)) {
        // already page-locked (e.g. from fsk_host_alloc): resident, DMA-able
        pinned_ = true;
        external_ = true;
        return;
    }
    p_ = p;
    bytes_ = bytes;
    pinned_ = false;
    int dev = 0;
    FSKB_CUDA(cudaGetDevice(&dev));
    th_ = std::thread([this, dev] {
        const int nt = int(std::max(1u, std::min(4u, std::thread::hardware_concurrency())));
        char* c = static_cast<char*>(p_);
        const std::size_t page = 4096, per = (bytes_ / page + nt - 1) / nt * page;
        std::vector<std::thread> helpers;
        for (int t = 0; t < nt; ++t)
            helpers.emplace_back([c, page, per, t, this] {
                const std::size_t lo = std::size_t(t) * per, hi = std::min(bytes_, lo + per);
                for (std::size_t o = lo; o < hi; o += page) reinterpret_cast<volatile char*>(c)[o] = 0;
            });
        for (auto& h : helpers) h.join();
        // page-locking the buffer for a direct DMA measured slower end to end (the
        // register / unregister of 0.5 GB outweighs the staged copy): off by default
        static const bool lock = [] {
            const char* e = std::getenv("FSK_PIN_OUTPUT");
            return e && e[0] == '1';
        }();
        if (lock && cudaSetDevice(dev) == cudaSuccess &&
            cudaHostRegister(p_, bytes_, cudaHostRegisterDefault) == cudaSuccess)
            pinned_ = true;
        else
            cudaGetLastError();   // (not fatal: the staged download is the fallback)
    });
}

void HostPrefault::join() {
    if (th_.joinable()) th_.join();
}

void HostPrefault::release() {
    join();
    if (pinned_ && !external_) cudaHostUnregister(p_);
    pinned_ = false;
    external_ = false;
}

// ---- pooled page-locked host buffers (fsk_host_alloc / fsk_host_free) ---------
namespace {
struct HostPool {
    std::mutex mu;
    std::multimap<size_t, void*> free_;   // size -> block
    std::map<void*, size_t> live;
    size_t cached = 0;
};
HostPool& host_pool() {
    static HostPool* p = new HostPool();   // never destroyed (process-lifetime cache)
    return *p;
}
constexpr size_t kHostPoolCap = size_t(8) << 30;
}  // namespace

void* host_alloc(size_t bytes) {
    if (!bytes) bytes = 1;
    auto& P = host_pool();
    {
        std::lock_guard<std::mutex> lk(P.mu);
        // smallest cached block that fits without wasting more than half of it
        auto it = P.free_.lower_bound(bytes);
        if (it != P.free_.end() && it->first <= 2 * bytes) {
            void* b = it->second;
            P.live[b] = it->first;
            P.cached -= it->first;
            P.free_.erase(it);
            return b;
        }
    }
    void* b = nullptr;
    if (cudaHostAlloc(&b, bytes, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        // release the cache and retry once
        std::vector<void*> drop;
        {
            std::lock_guard<std::mutex> lk(P.mu);
            for (auto& [sz, q] : P.free_) drop.push_back(q);
            P.free_.clear();
            P.cached = 0;
        }
        for (void* q : drop) cudaFreeHost(q);
        FSKB_CUDA(cudaHostAlloc(&b, bytes, cudaHostAllocPortable));
    }
    std::lock_guard<std::mutex> lk(P.mu);
    P.live[b] = bytes;
    return b;
}

void host_free(void* p) {
    if (!p) return;
    auto& P = host_pool();
    std::vector<void*> drop;
    {
        std::lock_guard<std::mutex> lk(P.mu);
        auto it = P.live.find(p);
        if (it == P.live.end()) throw std::invalid_argument("fsk_host_free: not an fsk_host_alloc block");
        const size_t sz = it->second;
        P.live.erase(it);
        P.free_.emplace(sz, p);
        P.cached += sz;
        // over the cap: drop the largest cached blocks
        while (P.cached > kHostPoolCap && !P.free_.empty()) {
            auto last = std::prev(P.free_.end());
            P.cached -= last->first;
            drop.push_back(last->second);
            P.free_.erase(last);
        }
    }
    for (void* q : drop) cudaFreeHost(q);
}

Scratch& Scratch::local() {
    int dev = 0;
    FSKB_CUDA(cudaGetDevice(&dev));
    thread_local std::vector<std::unique_ptr<Scratch>> per_dev;
    if (per_dev.size() <= size_t(dev)) per_dev.resize(size_t(dev) + 1);
    if (!per_dev[size_t(dev)]) {
        per_dev[size_t(dev)] = std::make_unique<Scratch>();
        per_dev[size_t(dev)]->dev_ = dev;
    }
    return *per_dev[size_t(dev)];
}

void* Scratch::get(std::size_t bytes, cudaStream_t s) {
    if (!ev_) FSKB_CUDA(cudaEventCreateWithFlags(&ev_, cudaEventDisableTiming));
    if (pending_) FSKB_CUDA(cudaStreamWaitEvent(s, ev_, 0));
    if (bytes > n_) {
        if (p_) FSKB_CUDA(cudaFreeAsync(p_, s));
        p_ = nullptr;
        n_ = 0;
        FSKB_CUDA(cudaMallocAsync(&p_, bytes, s));
        n_ = bytes;
    }
    return p_;
}

void Scratch::done(cudaStream_t s) {
    FSKB_CUDA(cudaEventRecord(ev_, s));
    pending_ = true;
}

Scratch::~Scratch() {
    // thread exit: the device may already be torn down; best effort
    if (p_) {
        cudaSetDevice(dev_);
        cudaDeviceSynchronize();
        cudaFree(p_);
    }
    if (ev_) cudaEventDestroy(ev_);
}

}  // namespace fskb
