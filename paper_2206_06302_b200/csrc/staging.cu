// staging.cu -- host <-> device copies of pageable host memory through
// pinned staging buffers ("pinned-host
// staging for H2D/D2H", the counterpart of the reference's host<->device
// copy arms, algorithms.hpp:388-407).
//
// A reference user's data lives in std::vector, i.e. pageable memory, for
// which cudaMemcpyAsync stages through the driver's own small bounce
// buffer: 11 GB/s H2D and 21 GB/s D2H on the B200 boxes against 55/51 GB/s
// from pinned memory.  Here a large pageable copy is cut into 32 MiB
// chunks that a per-(device, direction) staging worker copies into (or out
// of) a ring of pinned buffers with a team of host threads, while the copy
// engine moves other chunks.
//
// Every chunk is ordered on the caller's stream, never on the host thread
// that enqueued it:
//
//   H2D chunk t (slot k):   [GPU waits flag[k] >= t]  [DMA buf[k] -> dst]  [event]
//     worker: waits for the stream to reach the copy (event recorded when
//             it was enqueued), for the DMA of the slot's previous chunk
//             (its event), copies src -> buf[k], then sets flag[k] = t.
//   D2H chunk t (slot k):   [GPU waits flag[k] >= t - ring]  [DMA src -> buf[k]]  [event]
//     worker: waits for the event, copies buf[k] -> dst, sets flag[k] = t.
//     After the last chunk the stream waits flag[k_last] >= t_last, so
//     the stream completes only once dst holds the data.
//
// The GPU-side waits are stream memory operations (cuStreamWaitValue32 on
// mapped pinned host memory, reached through cudaGetDriverEntryPoint, so
// libcuda is not a link dependency); the flags are monotonically
// increasing tickets, so a slot never needs resetting.  Each worker takes
// its chunks in enqueue order and every wait refers to work enqueued
// earlier, so the earliest unfinished chunk can always progress (no
// deadlock between the two directions, any number of streams).
//
// Two entry points share this machinery:
//   staged_enqueue  stream-ordered (pinned-memory semantics): returns at
//                   once; the host buffer must stay valid (and, for H2D,
//                   unmodified) until the stream has passed the copy.
//   staged_h2d/d2h  cudaMemcpyAsync's pageable semantics: H2D reads the
//                   source after the stream's earlier work and returns
//                   once it has been consumed; D2H returns once the data
//                   is in dst.
#include "common.h"
#include "staging.h"

#include <cuda.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include <immintrin.h>

namespace coloc_cuda {
namespace {

// Chunk size and ring depth per (device, direction).  Defaults: 32 MiB x
// 4; COLOC_STAGING_CHUNK_KB / COLOC_STAGING_RING override them and
// COLOC_STAGING_H2D_NT=0 makes the host->staging copies plain (cached)
// stores (measurement knobs, read once).
constexpr int kMaxRing = 32;

struct staging_params
{
    std::size_t chunk = std::size_t(32) << 20;
    int ring = 4;
    bool h2d_nt = true;
};

staging_params const& params()
{
    static staging_params const p = [] {
        staging_params q;
        if (char const* e = std::getenv("COLOC_STAGING_CHUNK_KB"))
            q.chunk = std::clamp<std::size_t>(std::strtoull(e, nullptr, 10), 64, 1 << 20) << 10;
        if (char const* e = std::getenv("COLOC_STAGING_RING"))
            q.ring = std::clamp(std::atoi(e), 2, kMaxRing);
        if (char const* e = std::getenv("COLOC_STAGING_H2D_NT"))
            q.h2d_nt = std::atoi(e) != 0;
        return q;
    }();
    return p;
}
constexpr int kMaxDevices = 64;

// memcpy with non-temporal 32-byte stores for the aligned middle: a large
// destination that is not read back soon (the user's buffer of a D2H copy,
// or a staging buffer the DMA reads next) then costs no
// read-for-ownership traffic.
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

// Persistent helper threads for the host side of a staged chunk: the
// calling worker takes one slice, the helpers the others.
class copy_team
{
public:
    explicit copy_team(int nthreads)
      : nthreads_(std::max(1, nthreads))
    {
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
        std::lock_guard<std::mutex> one_at_a_time(busy_);    // stagers of several devices share a team
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
    std::mutex busy_;
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

// Stream memory operations from the driver API, resolved at first use.
struct memops
{
    CUresult(CUDAAPI* wait32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
    bool ok = false;
    std::string why;
};

memops const& drv()
{
    static memops m;
    static std::once_flag once;
    std::call_once(once, [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
        cudaError_t e = cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &fn, 12000,
            cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
        {
            (void) cudaGetLastError();
            m.why = "cuStreamWaitValue32 unavailable from the driver";
            return;
        }
        m.wait32 = reinterpret_cast<decltype(m.wait32)>(fn);
        m.ok = true;
    });
    return m;
}

// One chunk handed to a worker.
struct job
{
    std::uint32_t ticket = 0;
    int slot = 0;
    char* host = nullptr;              // H2D: source; D2H: destination
    std::size_t len = 0;
    cudaEvent_t before = nullptr;      // wait before touching the staging buffer
    cudaEvent_t before2 = nullptr;     // H2D: the stream reaching the copy
    bool skip = false;                 // the chunk's GPU side failed: only advance the flag
};

// Ring of pinned buffers + worker for one device and one direction.
class stager
{
public:
    stager(int dev, bool h2d)
      : dev_(dev)
      , h2d_(h2d)
    {
    }

    ~stager() = delete;    // process lifetime (see ring_of)

    int init()
    {
        if (ready_)
            return COLOC_OK;
        if (!drv().ok)
            return fail(COLOC_ERR_UNSUPPORTED, "staging: " + drv().why);
        COLOC_TRY(use_device(dev_));
        // resumes after a partial failure: slots already set up are kept
        for (; nbuf_ < params().ring; ++nbuf_)
            COLOC_TRY(coloc_cuda_host_alloc(params().chunk, &buf_[nbuf_]));
        if (!flags_)
        {
            void* f = nullptr;
            COLOC_TRY_CUDA(cudaHostAlloc(&f, kMaxRing * sizeof(std::uint32_t),
                               cudaHostAllocMapped | cudaHostAllocPortable),
                "staging: flag allocation");
            std::memset(f, 0, kMaxRing * sizeof(std::uint32_t));
            void* d = nullptr;
            cudaError_t e = cudaHostGetDevicePointer(&d, f, 0);
            if (e != cudaSuccess)
            {
                (void) cudaFreeHost(f);
                return fail_cuda(e, "staging: cudaHostGetDevicePointer");
            }
            flags_ = static_cast<std::uint32_t*>(f);
            flags_dev_ = reinterpret_cast<CUdeviceptr>(d);
        }
        // one team per direction, shared by every device's stager of that
        // direction, so H2D and D2H chunks are copied concurrently
        static copy_team* teams[2] = {};
        static std::mutex team_mu;
        {
            std::lock_guard<std::mutex> lock(team_mu);
            copy_team*& t = teams[h2d_ ? 1 : 0];
            if (!t)
            {
                unsigned const hw = std::max(1u, std::thread::hardware_concurrency());
                int nt = int(std::clamp(hw / 2, 1u, 8u));
                if (char const* e = std::getenv("COLOC_STAGING_THREADS"))
                    nt = std::clamp(std::atoi(e), 1, 64);
                t = new copy_team(nt);
            }
            team_ = t;
        }
        if (!worker_started_)
        {
            worker_ = std::thread([this] { run(); });
            worker_.detach();
            worker_started_ = true;
        }
        ready_ = true;
        return COLOC_OK;
    }

    // Enqueues the chunks of one copy on `stream` (caller holds mu()).
    // *last receives the ticket of the copy's final chunk.  Once a ticket
    // is drawn its job always reaches the worker (marked `skip` if the
    // chunk's GPU side failed), so no later wait on its slot can hang.
    int enqueue(cudaStream_t stream, char* dst, char const* src, std::size_t bytes,
        std::uint32_t* last)
    {
        if (int st = take_error(); st != COLOC_OK)
            return st;
        auto const& m = drv();
        auto wait = [&](int k, std::uint32_t v) -> int {
            CUresult r = m.wait32(reinterpret_cast<CUstream>(stream),
                flags_dev_ + CUdeviceptr(k) * sizeof(std::uint32_t), v, CU_STREAM_WAIT_VALUE_GEQ);
            if (r != CUDA_SUCCESS)
                return fail(COLOC_ERR_CUDA, "staging: cuStreamWaitValue32 failed (CUresult " +
                        std::to_string(int(r)) + ")");
            return COLOC_OK;
        };
        cudaEvent_t reach = nullptr;
        if (h2d_)
        {
            // the source is read after the stream's earlier work (which may
            // be a D2H copy into the same host buffer)
            COLOC_TRY(get_event(&reach));
            cudaError_t e = cudaEventRecord(reach, stream);
            if (e != cudaSuccess)
            {
                put_event(reach);
                return fail_cuda(e, "staging: cudaEventRecord");
            }
        }
        int st = COLOC_OK;
        job tail;
        std::size_t const chunk = params().chunk;
        std::uint32_t const ring = std::uint32_t(params().ring);
        for (std::size_t off = 0; off < bytes && st == COLOC_OK; off += chunk)
        {
            cudaEvent_t done = nullptr;
            st = get_event(&done);
            if (st != COLOC_OK)
                break;
            job j;
            j.ticket = next_++;
            j.slot = int(j.ticket % ring);
            j.len = std::min(chunk, bytes - off);
            int const k = j.slot;
            if (h2d_)
            {
                j.host = const_cast<char*>(src + off);
                j.before = slot_free_[k];    // DMA of the slot's previous chunk
                j.before2 = reach;
                reach = nullptr;
                slot_free_[k] = done;
                st = wait(k, j.ticket);
                if (st == COLOC_OK)
                {
                    cudaError_t e = cudaMemcpyAsync(dst + off, buf_[k], j.len, cudaMemcpyHostToDevice, stream);
                    if (e == cudaSuccess)
                        e = cudaEventRecord(done, stream);
                    if (e != cudaSuccess)
                        st = fail_cuda(e, "staging: H2D chunk");
                }
            }
            else
            {
                j.host = dst + off;
                j.before = done;
                // the worker has emptied the slot's previous chunk
                if (j.ticket > ring)
                    st = wait(k, j.ticket - ring);
                if (st == COLOC_OK)
                {
                    cudaError_t e = cudaMemcpyAsync(buf_[k], src + off, j.len, cudaMemcpyDeviceToHost, stream);
                    if (e == cudaSuccess)
                        e = cudaEventRecord(done, stream);
                    if (e != cudaSuccess)
                        st = fail_cuda(e, "staging: D2H chunk");
                }
            }
            j.skip = st != COLOC_OK;
            push(j);
            tail = j;
            *last = j.ticket;
        }
        put_event(reach);    // only left over when bytes == 0
        COLOC_TRY(st);
        // D2H: the stream completes only once dst holds the data
        if (!h2d_ && tail.ticket != 0)
            COLOC_TRY(wait(tail.slot, tail.ticket));
        return COLOC_OK;
    }

    // Frees the ring once every enqueued chunk is done (caller holds mu());
    // the next copy sets it up again, tickets restarting with the zeroed
    // flags.  The worker thread stays (it idles on the empty queue).
    int release()
    {
        if (!ready_)
            return COLOC_OK;
        if (next_ > 1)
            COLOC_TRY(wait_done(next_ - 1));
        for (int k = 0; k < nbuf_; ++k)
        {
            (void) coloc_cuda_host_free(buf_[k]);
            buf_[k] = nullptr;
        }
        nbuf_ = 0;
        if (flags_)
            (void) cudaFreeHost(flags_);
        flags_ = nullptr;
        flags_dev_ = 0;
        for (auto& e : slot_free_)
        {
            if (e)
                (void) cudaEventDestroy(e);
            e = nullptr;
        }
        {
            std::lock_guard<std::mutex> lock(pool_mu_);
            for (cudaEvent_t e : pool_)
                (void) cudaEventDestroy(e);
            pool_.clear();
        }
        {
            std::lock_guard<std::mutex> lock(qmu_);
            completed_ = 0;
        }
        next_ = 1;
        ready_ = false;
        return COLOC_OK;
    }

    // Blocks until the worker has finished chunk `ticket`.
    int wait_done(std::uint32_t ticket)
    {
        std::unique_lock<std::mutex> lock(qmu_);
        dcv_.wait(lock, [&] { return std::int32_t(completed_ - ticket) >= 0; });
        lock.unlock();
        return take_error();
    }

    std::mutex& mu() { return mu_; }

private:
    int get_event(cudaEvent_t* out)
    {
        {
            std::lock_guard<std::mutex> lock(pool_mu_);
            if (!pool_.empty())
            {
                *out = pool_.back();
                pool_.pop_back();
                return COLOC_OK;
            }
        }
        COLOC_TRY_CUDA(cudaEventCreateWithFlags(out, cudaEventDisableTiming), "staging: cudaEventCreate");
        return COLOC_OK;
    }

    void push(job const& j)
    {
        {
            std::lock_guard<std::mutex> lock(qmu_);
            queue_.push_back(j);
        }
        qcv_.notify_one();
    }

    void put_event(cudaEvent_t e)
    {
        if (!e)
            return;
        std::lock_guard<std::mutex> lock(pool_mu_);
        pool_.push_back(e);
    }

    int take_error()
    {
        std::lock_guard<std::mutex> lock(err_mu_);
        if (err_ == COLOC_OK)
            return COLOC_OK;
        int const st = err_;
        err_ = COLOC_OK;
        return fail(st, err_msg_);
    }

    void note_error(cudaError_t e, char const* what)
    {
        (void) cudaGetLastError();
        std::lock_guard<std::mutex> lock(err_mu_);
        if (err_ == COLOC_OK)
        {
            err_ = status_of(e);
            err_msg_ = std::string("staging worker: ") + what + ": " + cudaGetErrorString(e);
        }
    }

    void run()
    {
        (void) cudaSetDevice(dev_);
        for (;;)
        {
            job j;
            {
                std::unique_lock<std::mutex> lock(qmu_);
                qcv_.wait(lock, [&] { return !queue_.empty(); });
                j = queue_.front();
                queue_.pop_front();
            }
            bool ok = true;
            for (cudaEvent_t e : {j.before2, j.before})
                if (e)
                {
                    cudaError_t r = cudaEventSynchronize(e);
                    if (r != cudaSuccess)
                    {
                        note_error(r, "cudaEventSynchronize");
                        ok = false;
                    }
                }
            if (ok && !j.skip)
            {
                if (h2d_)
                    team_->copy(buf_[j.slot], j.host, j.len, /*streaming=*/params().h2d_nt);
                else
                    team_->copy(j.host, buf_[j.slot], j.len, /*streaming=*/true);
            }
            // D2H: the chunk's event is done with; H2D: j.before belonged
            // to the slot's previous chunk, j.before2 to the stream point
            put_event(j.before);
            put_event(j.before2);
            // the flag is set even after an error, so the stream never hangs
            __atomic_store_n(&flags_[j.slot], j.ticket, __ATOMIC_RELEASE);
            {
                std::lock_guard<std::mutex> lock(qmu_);
                completed_ = j.ticket;
            }
            dcv_.notify_all();
        }
    }

    int dev_;
    bool h2d_;
    bool ready_ = false;
    int nbuf_ = 0;
    void* buf_[kMaxRing] = {};
    std::uint32_t* flags_ = nullptr;    // flag[k] = ticket of the slot's last finished chunk
    CUdeviceptr flags_dev_ = 0;
    cudaEvent_t slot_free_[kMaxRing] = {};    // H2D: event after the slot's last DMA
    std::uint32_t next_ = 1;
    copy_team* team_ = nullptr;
    std::thread worker_;
    bool worker_started_ = false;
    std::mutex mu_;                      // one enqueue at a time
    std::mutex qmu_;
    std::condition_variable qcv_, dcv_;
    std::deque<job> queue_;
    std::uint32_t completed_ = 0;
    std::mutex pool_mu_;
    std::vector<cudaEvent_t> pool_;
    std::mutex err_mu_;
    int err_ = COLOC_OK;
    std::string err_msg_;
};

// Process-lifetime stagers (never destroyed: their workers may be blocked
// in CUDA calls while the runtime shuts down at exit).
int stager_of(int dev, bool h2d, stager** out, bool create = true)
{
    if (dev < 0 || dev >= kMaxDevices)
        return fail(COLOC_ERR_INVALID_TARGET, "staging: device ordinal " + std::to_string(dev) + " out of range");
    static std::mutex mu;
    static stager* all[kMaxDevices][2] = {};
    std::lock_guard<std::mutex> lock(mu);
    stager*& s = all[dev][h2d ? 1 : 0];
    if (!s && create)
        s = new stager(dev, h2d);
    *out = s;
    return COLOC_OK;
}

// Every stager created so far (for coloc_cuda_staging_release).
std::vector<stager*> all_stagers()
{
    std::vector<stager*> out;
    for (int dev = 0; dev < kMaxDevices; ++dev)
        for (bool h2d : {false, true})
        {
            stager* s = nullptr;
            if (stager_of(dev, h2d, &s, /*create=*/false) == COLOC_OK && s)
                out.push_back(s);
        }
    return out;
}

int enqueue_locked(stager& s, cudaStream_t stream, void* dst, void const* src, std::size_t bytes,
    std::uint32_t* last)
{
    COLOC_TRY(s.init());
    return s.enqueue(stream, static_cast<char*>(dst), static_cast<char const*>(src), bytes, last);
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

int staged_enqueue(int dev, cudaStream_t stream, void* dst, void const* src, std::size_t bytes, bool h2d)
{
    stager* s = nullptr;
    COLOC_TRY(stager_of(dev, h2d, &s));
    std::lock_guard<std::mutex> lock(s->mu());
    std::uint32_t last = 0;
    return enqueue_locked(*s, stream, dst, src, bytes, &last);
}

int staging_release()
{
    int st = COLOC_OK;
    for (stager* s : all_stagers())
    {
        std::lock_guard<std::mutex> lock(s->mu());
        int const e = s->release();
        st = st == COLOC_OK ? e : st;
    }
    return st;
}

int staged_h2d(int dev, cudaStream_t stream, void* dst, void const* src, std::size_t bytes)
{
    stager* s = nullptr;
    COLOC_TRY(stager_of(dev, true, &s));
    std::uint32_t last = 0;
    {
        std::lock_guard<std::mutex> lock(s->mu());
        COLOC_TRY(enqueue_locked(*s, stream, dst, src, bytes, &last));
    }
    // returns once the source has been consumed (the DMA of the last chunks
    // may still be in flight, ordered on the stream)
    return s->wait_done(last);
}

int staged_d2h(int dev, cudaStream_t stream, void* dst, void const* src, std::size_t bytes)
{
    stager* s = nullptr;
    COLOC_TRY(stager_of(dev, false, &s));
    std::uint32_t last = 0;
    {
        std::lock_guard<std::mutex> lock(s->mu());
        COLOC_TRY(enqueue_locked(*s, stream, dst, src, bytes, &last));
    }
    return s->wait_done(last);    // dst holds the data
}

}    // namespace coloc_cuda
