// hostcopy.cu -- the host-array entry points' transfers (srt_trace_rays,
// srt_transmittance_rays, srt_exact_rays, srt_biased_rays, srt_render into
// caller arrays): pageable <-> device copies at PCIe speed.
//
// A cudaMemcpy from pageable memory goes through the driver's small staging
// buffer, one thread, synchronously (about a third of the link's rate here).
// Instead, large copies are cut into 8 MB chunks that move through a ring of
// two page-locked buffers owned by the scene: host threads copy chunk c+1
// between the caller's array and one buffer while the copy engine moves
// chunk c through the other.  Pinned caller memory (srt_host_alloc,
// registered) and small copies take one cudaMemcpyAsync.
#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <functional>
#include <mutex>
#include <thread>

#include "srt_internal.h"

namespace srt {

namespace {

constexpr size_t kChunk = 8u << 20;       // bytes per staged chunk
constexpr size_t kDirectMax = 2u << 20;   // smaller copies go straight through the driver

// Worker threads for the host-side memcpy of a chunk (a process-wide pool:
// each task is one slice of one chunk; the caller runs a slice itself and
// waits for the rest).
class CopyPool {
  public:
    static CopyPool &get() {
        static CopyPool pool;
        return pool;
    }
    int width() const { return (int)workers_.size() + 1; }
    // at most `threads` host threads (the caller included) on one chunk
    void memcpy_parallel(void *dst, const void *src, size_t n, int threads) {
        const int parts = (int)std::min<size_t>((size_t)std::min(threads, width()), std::max<size_t>(1, n >> 20));
        if (parts <= 1) {
            std::memcpy(dst, src, n);
            return;
        }
        const size_t piece = ((n + parts - 1) / parts + 63) & ~(size_t)63;
        // completion count, guarded by dm: a worker touches dm / dcv only while
        // holding dm, so once the caller sees zero (under dm) no worker will
        // touch them again and they may go out of scope
        int left = parts - 1;
        std::mutex dm;
        std::condition_variable dcv;
        {
            std::lock_guard<std::mutex> lk(m_);
            for (int p = 1; p < parts; ++p) {
                const size_t off = std::min(n, piece * p), len = std::min(n - off, piece);
                tasks_.push_back([=, &left, &dm, &dcv] {
                    std::memcpy((char *)dst + off, (const char *)src + off, len);
                    std::lock_guard<std::mutex> g(dm);
                    if (--left == 0) dcv.notify_one();
                });
            }
        }
        cv_.notify_all();
        std::memcpy(dst, src, std::min(n, piece));
        std::unique_lock<std::mutex> lk(dm);
        dcv.wait(lk, [&] { return left == 0; });
    }

  private:
    CopyPool() {
        const unsigned hw = std::thread::hardware_concurrency();
        const int n = (int)std::max(1u, std::min(32u, hw > 2 ? hw / 2 : 1u)) - 1;
        for (int i = 0; i < n; ++i) workers_.emplace_back([this] { run(); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto &t : workers_) t.join();
    }
    void run() {
        while (true) {
            std::function<void()> f;
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] { return stop_ || !tasks_.empty(); });
                if (stop_ && tasks_.empty()) return;
                f = std::move(tasks_.front());
                tasks_.pop_front();
            }
            f();
        }
    }
    std::vector<std::thread> workers_;
    std::deque<std::function<void()>> tasks_;
    std::mutex m_;
    std::condition_variable cv_;
    bool stop_ = false;
};

// Uploads read the caller's (already resident) arrays: memory-bound, a
// quarter of the host threads copies fastest (2M rays: 5.5 -> 4.6 ms over
// half).  Downloads write fresh numpy arrays whose first touch faults pages
// in: half the threads (a biased 1080p frame: 9.5 -> 7.9 ms over a quarter).
int h2d_threads() {
    const unsigned hw = std::thread::hardware_concurrency();
    return (int)std::max(1u, hw / 4);
}
int d2h_threads() {
    const unsigned hw = std::thread::hardware_concurrency();
    return (int)std::max(1u, hw / 2);
}

bool pinned(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

srt_status stage_reserve(SrtScene *s) {
    if (s->h_stage[0]) return SRT_OK;
    for (int b = 0; b < 2; ++b) {
        srt_status rc = cuda_status(cudaHostAlloc(&s->h_stage[b], kChunk, cudaHostAllocPortable), "staging alloc");
        if (!rc) rc = cuda_status(cudaEventCreateWithFlags(&s->stage_ev[b], cudaEventDisableTiming), "staging event");
        if (rc) return rc;
    }
    return SRT_OK;
}

}  // namespace

srt_status copy_h2d(SrtScene *s, void *dst, const void *src, size_t bytes, cudaStream_t st) {
    if (bytes == 0) return SRT_OK;
    if (bytes <= kDirectMax || pinned(src))
        return cuda_status(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st), "upload");
    srt_status rc = stage_reserve(s);
    if (rc) return rc;
    CopyPool &pool = CopyPool::get();
    for (size_t off = 0, c = 0; off < bytes && !rc; off += kChunk, ++c) {
        const int b = (int)(c & 1);
        const size_t n = std::min(kChunk, bytes - off);
        // the buffer's previous chunk has left for the device
        if (c >= 2) rc = cuda_status(cudaEventSynchronize(s->stage_ev[b]), "staging wait");
        if (rc) break;
        pool.memcpy_parallel(s->h_stage[b], (const char *)src + off, n, h2d_threads());
        rc = cuda_status(cudaMemcpyAsync((char *)dst + off, s->h_stage[b], n, cudaMemcpyHostToDevice, st), "upload");
        if (!rc) rc = cuda_status(cudaEventRecord(s->stage_ev[b], st), "staging event");
    }
    // the ring is reused by the next call: its chunks must have left
    for (int b = 0; b < 2 && !rc; ++b) rc = cuda_status(cudaEventSynchronize(s->stage_ev[b]), "staging wait");
    return rc;
}

srt_status copy_d2h(SrtScene *s, void *dst, const void *src, size_t bytes, cudaStream_t st) {
    if (bytes == 0) return SRT_OK;
    if (bytes <= kDirectMax || pinned(dst))
        return cuda_status(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st), "download");
    srt_status rc = stage_reserve(s);
    if (rc) return rc;
    CopyPool &pool = CopyPool::get();
    const size_t nchunk = (bytes + kChunk - 1) / kChunk;
    for (size_t c = 0; c <= nchunk && !rc; ++c) {
        if (c < nchunk) {  // chunk c -> buffer c & 1 on the copy engine
            const int b = (int)(c & 1);
            const size_t off = c * kChunk, n = std::min(kChunk, bytes - off);
            rc = cuda_status(cudaMemcpyAsync(s->h_stage[b], (const char *)src + off, n, cudaMemcpyDeviceToHost, st),
                             "download");
            if (!rc) rc = cuda_status(cudaEventRecord(s->stage_ev[b], st), "staging event");
        }
        if (c >= 1 && !rc) {  // meanwhile chunk c-1 -> the caller's array
            const int b = (int)((c - 1) & 1);
            const size_t off = (c - 1) * kChunk, n = std::min(kChunk, bytes - off);
            rc = cuda_status(cudaEventSynchronize(s->stage_ev[b]), "staging wait");
            if (!rc) pool.memcpy_parallel((char *)dst + off, s->h_stage[b], n, d2h_threads());
        }
    }
    return rc;
}

void stage_release(SrtScene *s) {
    for (int b = 0; b < 2; ++b) {
        if (s->stage_ev[b]) cudaEventDestroy(s->stage_ev[b]);
        if (s->h_stage[b]) cudaFreeHost(s->h_stage[b]);
        s->stage_ev[b] = nullptr;
        s->h_stage[b] = nullptr;
    }
}

}  // namespace srt
