// Staged H2D copies from pageable host memory (see host_stage.cuh).
#include "host_stage.cuh"

#include <algorithm>
#include <atomic>
#include <cstring>
#include <functional>

#include "common.cuh"

namespace smx {

bool is_pageable(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();   // (older drivers report unregistered memory as an error)
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

namespace {

// Fixed pool of memcpy workers (created on first use, joined at exit).
class CopyPool {
public:
    static CopyPool& get() {
        static CopyPool pool;
        return pool;
    }
    // memcpy(dst, src, bytes) split over the workers; returns when done.
    // One job at a time (concurrent callers queue on job_mu_).
    void copy(char* dst, const char* src, size_t bytes) {
        std::lock_guard<std::mutex> job(job_mu_);
        std::unique_lock<std::mutex> lk(mu_);
        dst_ = dst;
        src_ = src;
        bytes_ = bytes;
        pending_ = (int)workers_.size();
        ++gen_;
        cv_.notify_all();
        done_cv_.wait(lk, [&] { return pending_ == 0; });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }

private:
    CopyPool() {
        const unsigned hw = std::thread::hardware_concurrency();
        const int n = (int)std::max(1u, std::min(12u, hw > 2 ? hw - 2 : 1u));
        for (int i = 0; i < n; ++i) workers_.emplace_back([this, i, n] { loop(i, n); });
    }
    void loop(int i, int n) {
        unsigned long long seen = 0;
        for (;;) {
            char* d;
            const char* s;
            size_t b;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
                d = dst_;
                s = src_;
                b = bytes_;
            }
            // 4 KB-aligned slices, one per worker
            const size_t per = ((b + n - 1) / n + 4095) & ~size_t(4095);
            const size_t lo = std::min(b, per * i), hi = std::min(b, lo + per);
            if (hi > lo) std::memcpy(d + lo, s + lo, hi - lo);
            std::lock_guard<std::mutex> lk(mu_);
            if (--pending_ == 0) done_cv_.notify_all();
        }
    }
    std::vector<std::thread> workers_;
    std::mutex job_mu_, mu_;
    std::condition_variable cv_, done_cv_;
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    size_t bytes_ = 0;
    int pending_ = 0;
    unsigned long long gen_ = 0;
    bool stop_ = false;
};

// Page-locked staging ring: kSlots x kSlotBytes, allocated once per process
// (256 MB; cudaHostAlloc of 2 GB took 2.1 s on the pool's hosts).
constexpr int kSlots = 4;
constexpr size_t kSlotBytes = 64ull << 20;
struct Ring {
    char* base = nullptr;
    cudaEvent_t ev[kSlots] = {};
    int device = -1;
};
std::mutex g_ring_mu;
int ring_for(int device, Ring** out) {
    static Ring rings[64];
    if (device < 0 || device >= 64) return SMX_E_ARG;
    Ring& r = rings[device];
    if (!r.base) {
        cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&r.base), kSlots * kSlotBytes, cudaHostAllocPortable);
        if (e != cudaSuccess) {
            r.base = nullptr;
            return (int)e;
        }
        for (int i = 0; i < kSlots; ++i)
            if ((e = cudaEventCreateWithFlags(&r.ev[i], cudaEventDisableTiming)) != cudaSuccess) return (int)e;
        r.device = device;
    }
    *out = &r;
    return SMX_OK;
}

}  // namespace

int HostStager::start(const void* src, void* dst, size_t row_bytes, const std::vector<int>& ends,
                      const cudaEvent_t* ev, cudaStream_t in) {
    src_ = static_cast<const char*>(src);
    dst_ = static_cast<char*>(dst);
    ends_.clear();
    for (int e : ends) ends_.push_back((size_t)e * row_bytes);
    ev_ = ev;
    in_ = in;
    recorded_ = 0;
    status_ = 0;
    cudaError_t e = cudaGetDevice(&device_);
    if (e != cudaSuccess) return (int)e;
    th_ = std::thread([this] { run(); });
    return SMX_OK;
}

int HostStager::start_bytes(const void* src, void* dst, size_t bytes, const cudaEvent_t* ev, cudaStream_t in) {
    src_ = static_cast<const char*>(src);
    dst_ = static_cast<char*>(dst);
    ends_.assign(1, bytes);
    ev_ = ev;
    in_ = in;
    recorded_ = 0;
    status_ = 0;
    cudaError_t e = cudaGetDevice(&device_);
    if (e != cudaSuccess) return (int)e;
    th_ = std::thread([this] { run(); });
    return SMX_OK;
}

void HostStager::run() {
    int rc = SMX_OK;
    cudaSetDevice(device_);
    Ring* ring = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_ring_mu);   // one staged call per ring at a time
        rc = ring_for(device_, &ring);
        if (rc == SMX_OK) {
            CopyPool& pool = CopyPool::get();
            size_t chunk = 0;
            for (size_t g = 0, b0 = 0; g < ends_.size() && rc == SMX_OK; b0 = ends_[g], ++g) {
                size_t off = b0;
                const size_t end = ends_[g];
                while (off < end && rc == SMX_OK) {
                    const int slot = (int)(chunk % kSlots);
                    const size_t bytes = std::min(kSlotBytes, end - off);
                    cudaError_t e = cudaSuccess;
                    // the slot's previous H2D (this call's, or a previous call's
                    // still in flight) must be done before it is overwritten; an
                    // event never recorded completes at once
                    e = cudaEventSynchronize(ring->ev[slot]);
                    if (e == cudaSuccess) {
                        char* s = ring->base + slot * kSlotBytes;
                        pool.copy(s, src_ + off, bytes);
                        e = cudaMemcpyAsync(dst_ + off, s, bytes, cudaMemcpyHostToDevice, in_);
                    }
                    if (e == cudaSuccess) e = cudaEventRecord(ring->ev[slot], in_);
                    if (e != cudaSuccess) rc = (int)e;
                    off += bytes;
                    ++chunk;
                }
                if (rc == SMX_OK) {
                    cudaError_t e = cudaEventRecord(ev_[g], in_);
                    if (e != cudaSuccess) rc = (int)e;
                }
                if (rc == SMX_OK) {
                    std::lock_guard<std::mutex> lk(mu_);
                    recorded_ = (int)g + 1;
                    cv_.notify_all();
                }
            }
        }
    }
    std::lock_guard<std::mutex> lk(mu_);
    status_ = rc;
    if (rc != SMX_OK) recorded_ = (int)ends_.size();   // release every waiter
    cv_.notify_all();
}

int HostStager::wait_recorded(int g) {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return recorded_ > g; });
    return status_;
}

int HostStager::finish() {
    if (th_.joinable()) th_.join();
    return status_;
}

int HostEgress::start(const void* src, void* dst, cudaStream_t out) {
    src_ = static_cast<const char*>(src);
    dst_ = static_cast<char*>(dst);
    out_ = out;
    queue_.clear();
    next_ = 0;
    closed_ = false;
    status_ = 0;
    cudaError_t e = cudaGetDevice(&device_);
    if (e != cudaSuccess) return (int)e;
    th_ = std::thread([this] { run(); });
    return SMX_OK;
}

void HostEgress::push(size_t b0, size_t b1, cudaEvent_t ev) {
    std::lock_guard<std::mutex> lk(mu_);
    queue_.push_back({b0, b1, ev});
    cv_.notify_all();
}

int HostEgress::finish() {
    {
        std::lock_guard<std::mutex> lk(mu_);
        closed_ = true;
        cv_.notify_all();
    }
    if (th_.joinable()) th_.join();
    return status_;
}

void HostEgress::run() {
    int rc = SMX_OK;
    cudaSetDevice(device_);
    {
        // The ring is taken when the first piece arrives, not before: the
        // same call's ingest stager holds it until every input group has
        // been issued, and the first piece is pushed only after that.
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return !queue_.empty() || closed_; });
    }
    std::lock_guard<std::mutex> ring_lock(g_ring_mu);
    Ring* ring = nullptr;
    rc = ring_for(device_, &ring);
    CopyPool& pool = CopyPool::get();
    // slots in flight: (slot, destination offset, bytes), oldest first
    struct Flight { int slot; size_t off, bytes; };
    std::vector<Flight> flight;
    size_t slot_seq = 0;
    auto drain_one = [&]() -> int {
        const Flight f = flight.front();
        flight.erase(flight.begin());
        cudaError_t e = cudaEventSynchronize(ring->ev[f.slot]);
        if (e != cudaSuccess) return (int)e;
        pool.copy(dst_ + f.off, ring->base + f.slot * kSlotBytes, f.bytes);
        return SMX_OK;
    };
    for (;;) {
        Piece pc;
        {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return next_ < queue_.size() || closed_; });
            if (next_ >= queue_.size()) break;   // closed and drained
            pc = queue_[next_++];
        }
        if (rc != SMX_OK) continue;          // (keep consuming so finish() returns)
        cudaError_t e = cudaStreamWaitEvent(out_, pc.ev, 0);
        for (size_t off = pc.b0; off < pc.b1 && e == cudaSuccess && rc == SMX_OK;) {
            const size_t bytes = std::min(kSlotBytes, pc.b1 - off);
            if (flight.size() == (size_t)kSlots) rc = drain_one();   // the slot we are about to reuse
            if (rc != SMX_OK) break;
            const int slot = (int)(slot_seq++ % kSlots);
            // the slot's last H2D (the ingest of this call) must have read it
            e = cudaStreamWaitEvent(out_, ring->ev[slot], 0);
            if (e != cudaSuccess) break;
            e = cudaMemcpyAsync(ring->base + slot * kSlotBytes, src_ + off, bytes, cudaMemcpyDeviceToHost, out_);
            if (e == cudaSuccess) e = cudaEventRecord(ring->ev[slot], out_);
            if (e == cudaSuccess) flight.push_back({slot, off, bytes});
            off += bytes;
        }
        if (e != cudaSuccess && rc == SMX_OK) rc = (int)e;
    }
    while (rc == SMX_OK && !flight.empty()) rc = drain_one();
    std::lock_guard<std::mutex> lk(mu_);
    status_ = rc;
}

namespace {
struct StageStream {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, done = nullptr;
    std::mutex mu;
};
int stage_stream(StageStream** out) {
    static StageStream per_dev[64];
    static std::mutex mu;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return (int)e;
    if (dev < 0 || dev >= 64) return SMX_E_ARG;
    std::lock_guard<std::mutex> lk(mu);
    StageStream& st = per_dev[dev];
    if (!st.s) {
        if ((e = cudaStreamCreateWithFlags(&st.s, cudaStreamNonBlocking)) != cudaSuccess) return (int)e;
        if ((e = cudaEventCreateWithFlags(&st.fork, cudaEventDisableTiming)) != cudaSuccess) return (int)e;
        if ((e = cudaEventCreateWithFlags(&st.done, cudaEventDisableTiming)) != cudaSuccess) return (int)e;
    }
    *out = &st;
    return SMX_OK;
}
}  // namespace

int h2d_staged(void* dst, const void* src, size_t bytes, cudaStream_t stream) {
    if (bytes == 0) return SMX_OK;
    if (dst == nullptr || src == nullptr) return SMX_E_ARG;
    cudaError_t e;
    // small pageable: one ordinary copy (the driver has read the source when
    // it returns); page-locked: one async copy, then wait for it, since the
    // contract is that `src` may be reused or freed once this returns
    const bool pageable = is_pageable(src);
    if (!pageable || bytes < (8u << 20)) {
        e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream);
        if (e == cudaSuccess && !pageable) e = cudaStreamSynchronize(stream);
        return e == cudaSuccess ? SMX_OK : (int)e;
    }
    StageStream* st = nullptr;
    SMX_TRY(stage_stream(&st));
    std::lock_guard<std::mutex> lk(st->mu);
    // the copy stream starts after the caller's prior work (dst may be in use)
    if ((e = cudaEventRecord(st->fork, stream)) != cudaSuccess) return (int)e;
    if ((e = cudaStreamWaitEvent(st->s, st->fork, 0)) != cudaSuccess) return (int)e;
    HostStager stager;
    SMX_TRY(stager.start_bytes(src, dst, bytes, &st->done, st->s));
    SMX_TRY(stager.finish());
    e = cudaStreamWaitEvent(stream, st->done, 0);
    return e == cudaSuccess ? SMX_OK : (int)e;
}

}  // namespace smx

using namespace smx;

extern "C" int smx_copy_h2d(void* dst, const void* src, size_t bytes, void* stream) {
    return h2d_staged(dst, src, bytes, as_stream(stream));
}

namespace smx {

}  // namespace smx
