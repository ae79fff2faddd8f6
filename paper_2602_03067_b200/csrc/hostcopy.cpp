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
#include <cstring>
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

void copy_host_to_device(void* dst, const void* src, size_t bytes, cudaStream_t s) {
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
    if (bytes < (size_t(8) << 20)) {
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

}  // namespace fskb
