// staging.cu -- host <-> device copies of pageable host memory through
// pinned staging buffers ("pinned-host
// staging for H2D/D2H", the counterpart of the reference's host<->device
// copy arms, algorithms.hpp:388-407).
//
// A reference user's data lives in std::vector, i.e. pageable memory, for
// which cudaMemcpyAsync stages through the driver's own small bounce
// buffer: 11 GB/s H2D and 21 GB/s D2H on the B200 boxes against 55/51 GB/s
// from pinned memory.  Here a large pageable copy is cut into chunks that
// several host threads copy into (or out of) a ring of pinned,
// huge-page-backed staging buffers while the copy engine moves the
// previous chunk, so host copying and DMA overlap.
//
// Semantics match cudaMemcpyAsync on pageable memory: H2D first waits for
// the work already on `stream`, then returns once the source has been
// consumed (the DMA of the last chunk may still be in flight, ordered on
// `stream`); D2H returns once the data is in `dst`.
#include "common.h"
#include "staging.h"

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include <immintrin.h>

namespace coloc_cuda {
namespace {

constexpr std::size_t kChunk = std::size_t(32) << 20;

// memcpy with non-temporal 32-byte stores for the aligned middle: a large
// destination that is not read back soon (the user's buffer of a D2H copy)
// then costs no read-for-ownership traffic.
__attribute__((target("avx2"))) void copy_nt_avx2(char* dst, char const* src, std::size_t n)
{
    std::size_t const head = std::min(n, (32 - reinterpret_cast<std::uintptr_t>(dst) % 32) % 32);
    std::memcpy(dst, src, head);
    std::size_t i = head;
    for (; i + 128 <= n; i += 128)
    {
        __m256i const a = _mm256_loadu_si256(reinterpret_cast<__m256i const*>(src + i));
        __m256i const b = _mm256_loadu_si256(reinterpret_cast<__m256i const*>(src + i + 32));
        __m256i const c = _mm256_loadu_si256(reinterpret_cast<__m256i const*>(src + i + 64));
        __m256i const e = _mm256_loadu_si256(reinterpret_cast<__m256i const*>(src + i + 96));
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), a);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 32), b);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 64), c);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 96), e);
    }
    std::memcpy(dst + i, src + i, n - i);
    _mm_sfence();
}

void copy_range(char* dst, char const* src, std::size_t n, bool streaming)
{
    static bool const avx2 = __builtin_cpu_supports("avx2");
    if (streaming && avx2)
        copy_nt_avx2(dst, src, n);
    else
        std::memcpy(dst, src, n);
}
constexpr int kRing = 3;

// Persistent helper threads for the host side of a staged copy: the
// caller's thread takes one slice, the workers the others.
class copy_team
{
public:
    copy_team()
    {
        unsigned const hw = std::max(1u, std::thread::hardware_concurrency());
        nthreads_ = int(std::clamp(hw / 2, 1u, 8u));
        for (int i = 1; i < nthreads_; ++i)
            workers_.emplace_back([this, i] { run(i); });
    }

    ~copy_team()
    {
        {
            std::lock_guard<std::mutex> lock(mu_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto& t : workers_)
            t.join();
    }

    void copy(void* dst, void const* src, std::size_t n, bool streaming)
    {
        if (nthreads_ == 1 || n < (std::size_t(1) << 20))
        {
            copy_range(static_cast<char*>(dst), static_cast<char const*>(src), n, streaming);
            return;
        }
        std::lock_guard<std::mutex> one_at_a_time(busy_);
        {
            std::lock_guard<std::mutex> lock(mu_);
            dst_ = static_cast<char*>(dst);
            src_ = static_cast<char const*>(src);
            n_ = n;
            streaming_ = streaming;
            pending_ = nthreads_ - 1;
            ++gen_;
        }
        cv_.notify_all();
        slice(0);
        std::unique_lock<std::mutex> lock(mu_);
        done_cv_.wait(lock, [this] { return pending_ == 0; });
    }

private:
    void slice(int i) const
    {
        std::size_t const t = std::size_t(nthreads_);
        std::size_t const per = ((n_ + t - 1) / t + 63) & ~std::size_t(63);    // covers n_
        std::size_t const lo = std::min(n_, per * std::size_t(i));
        std::size_t const hi = std::min(n_, lo + per);
        if (hi > lo)
            copy_range(dst_ + lo, src_ + lo, hi - lo, streaming_);
    }

    void run(int i)
    {
        std::uint64_t seen = 0;
        for (;;)
        {
            {
                std::unique_lock<std::mutex> lock(mu_);
                cv_.wait(lock, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_)
                    return;
            }
            slice(i);
            {
                std::lock_guard<std::mutex> lock(mu_);
                if (--pending_ == 0)
                    done_cv_.notify_one();
            }
        }
    }

    int nthreads_ = 1;
    std::vector<std::thread> workers_;
    std::mutex busy_;    // one copy at a time (rings of several devices share the team)
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    std::uint64_t gen_ = 0;
    bool stop_ = false;
    char* dst_ = nullptr;
    char const* src_ = nullptr;
    std::size_t n_ = 0;
    bool streaming_ = false;
    int pending_ = 0;
};

struct staging_ring
{
    std::mutex mu;    // one staged copy at a time per device
    bool ready = false;
    void* buf[kRing] = {};
    cudaEvent_t ev[kRing] = {};
    bool busy[kRing] = {};
    copy_team* team = nullptr;
};

staging_ring& ring_of(int dev)
{
    static staging_ring rings[64];
    return rings[dev];
}

int ensure_ring(staging_ring& r, int dev)
{
    if (r.ready)
        return COLOC_OK;
    for (int k = 0; k < kRing; ++k)
    {
        COLOC_TRY(coloc_cuda_host_alloc(kChunk, &r.buf[k]));
        COLOC_TRY_CUDA(cudaEventCreateWithFlags(&r.ev[k], cudaEventDisableTiming), "cudaEventCreate");
    }
    static copy_team team;    // shared by every device's ring
    r.team = &team;
    r.ready = true;
    (void) dev;
    return COLOC_OK;
}

}    // namespace

bool is_pageable_host(void const* p)
{
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess)
    {
        (void) cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

bool is_device_memory(void const* p)
{
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess)
    {
        (void) cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int staged_h2d(int dev, cudaStream_t stream, void* dst, void const* src, std::size_t bytes)
{
    staging_ring& r = ring_of(dev);
    std::lock_guard<std::mutex> lock(r.mu);
    COLOC_TRY(ensure_ring(r, dev));
    // as cudaMemcpyAsync from pageable memory: the source is read after the
    // work already queued on the stream
    COLOC_TRY_CUDA(cudaStreamSynchronize(stream), "staging: cudaStreamSynchronize");
    auto* d = static_cast<char*>(dst);
    auto const* s = static_cast<char const*>(src);
    for (std::size_t off = 0, i = 0; off < bytes; off += kChunk, ++i)
    {
        int const k = int(i % kRing);
        std::size_t const len = std::min(kChunk, bytes - off);
        if (r.busy[k])    // the DMA that last read this buffer has finished
            COLOC_TRY_CUDA(cudaEventSynchronize(r.ev[k]), "staging: cudaEventSynchronize");
        r.team->copy(r.buf[k], s + off, len, /*streaming=*/false);    // the DMA reads it next
        COLOC_TRY_CUDA(cudaMemcpyAsync(d + off, r.buf[k], len, cudaMemcpyHostToDevice, stream),
            "staging: cudaMemcpyAsync H2D");
        COLOC_TRY_CUDA(cudaEventRecord(r.ev[k], stream), "staging: cudaEventRecord");
        r.busy[k] = true;
    }
    return COLOC_OK;
}

int staged_d2h(int dev, cudaStream_t stream, void* dst, void const* src, std::size_t bytes)
{
    staging_ring& r = ring_of(dev);
    std::lock_guard<std::mutex> lock(r.mu);
    COLOC_TRY(ensure_ring(r, dev));
    auto* d = static_cast<char*>(dst);
    auto const* s = static_cast<char const*>(src);
    std::size_t const nchunks = (bytes + kChunk - 1) / kChunk;
    auto enqueue = [&](std::size_t i) -> int {
        int const k = int(i % kRing);
        std::size_t const off = i * kChunk;
        COLOC_TRY_CUDA(cudaMemcpyAsync(r.buf[k], s + off, std::min(kChunk, bytes - off),
                           cudaMemcpyDeviceToHost, stream),
            "staging: cudaMemcpyAsync D2H");
        COLOC_TRY_CUDA(cudaEventRecord(r.ev[k], stream), "staging: cudaEventRecord");
        r.busy[k] = true;
        return COLOC_OK;
    };
    for (std::size_t i = 0; i < std::min<std::size_t>(kRing, nchunks); ++i)
        COLOC_TRY(enqueue(i));
    for (std::size_t i = 0; i < nchunks; ++i)
    {
        int const k = int(i % kRing);
        COLOC_TRY_CUDA(cudaEventSynchronize(r.ev[k]), "staging: cudaEventSynchronize");
        std::size_t const off = i * kChunk;
        r.team->copy(d + off, r.buf[k], std::min(kChunk, bytes - off), /*streaming=*/true);
        if (i + kRing < nchunks)
            COLOC_TRY(enqueue(i + kRing));
    }
    return COLOC_OK;
}

}    // namespace coloc_cuda
