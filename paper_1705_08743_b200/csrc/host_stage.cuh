// Staged host -> device copies from pageable memory.
//
// The reference's user-visible closure takes an ordinary numpy array
// (AntidistMatrix(n, n, w, data).transitive_closure(), antidist.py:263-273),
// i.e. pageable memory.  cudaMemcpyAsync from pageable memory runs at ~11
// GB/s on the pool's B200 hosts and blocks the launching thread until each
// copy is staged, so the host-buffer closure could not issue its compute
// while the input streams in.  Here a coordinator thread copies the input
// through a ring of page-locked slots: a pool of worker threads memcpy each
// chunk into a slot (~47 GB/s on 16 cores, tools/perf_host_io.py), the
// coordinator issues the slot's H2D on the copy stream (55 GB/s) and
// records the caller's per-group event when a group's last chunk is in.
// The launching thread only waits (on the host) until a group's event has
// been recorded before it makes its stream wait on that event.
#pragma once
#include <cuda_runtime.h>

#include <condition_variable>
#include <cstddef>
#include <mutex>
#include <thread>
#include <vector>

namespace smx {

bool is_pageable(const void* p);

class HostStager {
public:
    // rows [ends[g-1], ends[g]) of `src` (row_bytes each) form group g; its
    // H2D into dst lands before ev[g] is recorded on `in`.
    int start(const void* src, void* dst, size_t row_bytes, const std::vector<int>& ends,
              const cudaEvent_t* ev, cudaStream_t in);
    // One group of `bytes` bytes (ev[0] recorded after it).
    int start_bytes(const void* src, void* dst, size_t bytes, const cudaEvent_t* ev, cudaStream_t in);
    // Blocks until group g's event has been recorded (or the stager failed).
    int wait_recorded(int g);
    // Joins the coordinator; returns its status.
    int finish();
    ~HostStager() { finish(); }

private:
    void run();
    const char* src_ = nullptr;
    char* dst_ = nullptr;
    std::vector<size_t> ends_;   // byte offsets
    const cudaEvent_t* ev_ = nullptr;
    cudaStream_t in_ = nullptr;
    int device_ = 0;
    std::thread th_;
    std::mutex mu_;
    std::condition_variable cv_;
    int recorded_ = 0;   // groups whose event is recorded
    int status_ = 0;
};

// Staged D2H copies into pageable host memory: the mirror of HostStager for
// the closure's egress.  The caller hands over (byte range, event) pieces in
// order as their rows become final; a coordinator thread copies each piece
// into the page-locked ring on the copy stream once its event has fired,
// and the memcpy pool moves it from the slot into `dst` (up to four slots in
// flight).  finish() returns when every byte is in `dst`.
class HostEgress {
public:
    int start(const void* src, void* dst, cudaStream_t out);
    // rows [b0, b1) of the flat buffers are final once `ev` fires (ev must be
    // recorded before this call; it is consumed in order)
    void push(size_t b0, size_t b1, cudaEvent_t ev);
    int finish();
    ~HostEgress() { finish(); }

private:
    struct Piece { size_t b0, b1; cudaEvent_t ev; };
    void run();
    const char* src_ = nullptr;
    char* dst_ = nullptr;
    cudaStream_t out_ = nullptr;
    int device_ = 0;
    std::thread th_;
    std::mutex mu_;
    std::condition_variable cv_;
    std::vector<Piece> queue_;
    size_t next_ = 0;
    bool closed_ = false;
    int status_ = 0;
};

// dst (device) <- src (host), `bytes`, ordered on `stream`: page-locked
// sources are one async copy; pageable ones go through the staging ring
// (~4x the pageable cudaMemcpy rate) and this call returns once every byte
// has been copied out of `src` (so the caller may reuse it).
int h2d_staged(void* dst, const void* src, size_t bytes, cudaStream_t stream);

}  // namespace smx
