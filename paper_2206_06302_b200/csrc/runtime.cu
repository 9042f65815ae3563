// runtime.cu -- targets, streams, memory, events: the real CUDA runtime in
// place of the reference's mock discrete device.
//
//   reference (mock)                              here
//   device::target{device_id, queue_id}           (ordinal, cudaStream_t)
//     device.hpp:29-41
//   mock_device::new_queue (src/device.cpp:109)   coloc_cuda_stream_create
//   fifo_queue::wait_idle (device.hpp:73-74)      coloc_cuda_stream_sync
//   mock_device::arena_allocate (device.cpp:78)   coloc_cuda_malloc
//   capacity overflow -> allocation_error          cudaErrorMemoryAllocation ->
//     (device.cpp:85-86)                            COLOC_ERR_ALLOCATION
//   unknown device -> invalid_target_error         cudaErrorInvalidDevice ->
//     (device.cpp:153-160)                          COLOC_ERR_INVALID_TARGET
#include "common.h"
#include "staging.h"

#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>
#include <unordered_map>

#include <sys/mman.h>

namespace coloc_cuda {

namespace {
thread_local std::string t_last_error;
}

std::atomic<std::uint64_t> g_launches{0};

void set_error(std::string msg) { t_last_error = std::move(msg); }
void clear_error() { t_last_error.clear(); }

int status_of(cudaError_t e)
{
    switch (e)
    {
    case cudaSuccess:
        return COLOC_OK;
    case cudaErrorMemoryAllocation:
        return COLOC_ERR_ALLOCATION;
    case cudaErrorInvalidDevice:
    case cudaErrorNoDevice:
    case cudaErrorInsufficientDriver:
    case cudaErrorDevicesUnavailable:
        return COLOC_ERR_INVALID_TARGET;
    case cudaErrorInvalidValue:
    case cudaErrorInvalidDevicePointer:
    case cudaErrorInvalidResourceHandle:
        return COLOC_ERR_INVALID_ARGUMENT;
    case cudaErrorLaunchFailure:
    case cudaErrorLaunchOutOfResources:
    case cudaErrorInvalidConfiguration:
    case cudaErrorNoKernelImageForDevice:
        return COLOC_ERR_SUBMISSION;
    default:
        return COLOC_ERR_CUDA;
    }
}

int fail(int status, std::string const& msg)
{
    set_error(msg);
    return status;
}

int fail_cuda(cudaError_t e, char const* what)
{
    // Sticky launch errors must not leak into the next call.
    (void) cudaGetLastError();
    return fail(status_of(e),
        std::string(what) + ": " + cudaGetErrorName(e) + " (" +
            cudaGetErrorString(e) + ")");
}

int use_device(int dev)
{
    int cur = -1;
    cudaError_t e = cudaGetDevice(&cur);
    if (e == cudaSuccess && cur == dev)
        return COLOC_OK;
    e = cudaSetDevice(dev);
    if (e != cudaSuccess)
    {
        (void) cudaGetLastError();    // keep the failure out of later launches
        return fail(status_of(e) == COLOC_ERR_INVALID_ARGUMENT ?
                COLOC_ERR_INVALID_TARGET :
                status_of(e),
            "cuda device " + std::to_string(dev) + ": " + cudaGetErrorString(e));
    }
    return COLOC_OK;
}

device_props const* props(int dev)
{
    // Fixed storage: a returned pointer stays valid while other threads
    // query further devices (a growing vector would move the entries).
    constexpr int kMaxDevices = 64;
    static std::mutex mu;
    static device_props cache[kMaxDevices];
    static std::atomic<bool> have[kMaxDevices];
    if (dev < 0 || dev >= kMaxDevices)
        return nullptr;
    if (have[dev].load(std::memory_order_acquire))
        return &cache[dev];
    std::lock_guard<std::mutex> lock(mu);
    if (!have[dev].load(std::memory_order_relaxed))
    {
        device_props p;
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        {
            (void) cudaGetLastError();
            return nullptr;
        }
        p.sm_count = v;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxThreadsPerMultiProcessor, dev) == cudaSuccess)
            p.max_threads_per_sm = v;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, dev) == cudaSuccess)
            p.l2_bytes = std::size_t(v);
        (void) cudaGetLastError();
        cache[dev] = p;
        have[dev].store(true, std::memory_order_release);
    }
    return &cache[dev];
}

}    // namespace coloc_cuda

using namespace coloc_cuda;

namespace coloc_cuda {
namespace {

constexpr std::size_t kHugePage = std::size_t(2) << 20;
constexpr std::size_t kThpMinBytes = std::size_t(64) << 20;

std::mutex& thp_mu()
{
    static std::mutex m;
    return m;
}

std::unordered_map<void*, std::size_t>& thp_blocks()
{
    static std::unordered_map<void*, std::size_t> m;    // pointer -> mapped length
    return m;
}

// mmap an aligned anonymous region, ask for huge pages before the first
// touch, then let cudaHostRegister fault in and pin it.  nullptr on any
// failure (the caller falls back to cudaHostAlloc).
void* thp_pinned_alloc(std::size_t bytes)
{
    std::size_t const len = (bytes + kHugePage - 1) / kHugePage * kHugePage;
    void* raw = mmap(nullptr, len + kHugePage, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (raw == MAP_FAILED)
        return nullptr;
    auto const r = reinterpret_cast<std::uintptr_t>(raw);
    auto const a = (r + kHugePage - 1) / kHugePage * kHugePage;
    if (a > r)
        munmap(raw, a - r);
    if (std::size_t const tail = (r + len + kHugePage) - (a + len))
        munmap(reinterpret_cast<void*>(a + len), tail);
    void* p = reinterpret_cast<void*>(a);
    (void) madvise(p, len, MADV_HUGEPAGE);
    if (cudaHostRegister(p, len, cudaHostRegisterPortable | cudaHostRegisterMapped) != cudaSuccess)
    {
        (void) cudaGetLastError();
        munmap(p, len);
        return nullptr;
    }
    std::lock_guard<std::mutex> lock(thp_mu());
    thp_blocks()[p] = len;
    return p;
}

bool thp_pinned_free(void* p)
{
    std::size_t len = 0;
    {
        std::lock_guard<std::mutex> lock(thp_mu());
        auto it = thp_blocks().find(p);
        if (it == thp_blocks().end())
            return false;
        len = it->second;
        thp_blocks().erase(it);
    }
    (void) cudaHostUnregister(p);
    (void) cudaGetLastError();
    munmap(p, len);
    return true;
}

}    // namespace
}    // namespace coloc_cuda

extern "C" {

const char* coloc_cuda_last_error(void)
{
    return t_last_error.c_str();
}

int coloc_cuda_abi_version(void)
{
    return COLOC_CUDA_ABI_VERSION;
}

uint64_t coloc_cuda_launch_count(void)
{
    return g_launches.load(std::memory_order_relaxed);
}

int coloc_cuda_device_count(int* count)
{
    if (!count)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "device_count: null out");
    *count = 0;
    cudaError_t e = cudaGetDeviceCount(count);
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver)
    {
        (void) cudaGetLastError();
        *count = 0;
        return COLOC_OK;
    }
    COLOC_TRY_CUDA(e, "cudaGetDeviceCount");
    return COLOC_OK;
}

int coloc_cuda_device_info_get(int dev, coloc_cuda_device_info* out)
{
    if (!out)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "device_info: null out");
    cudaDeviceProp p;
    cudaError_t e = cudaGetDeviceProperties(&p, dev);
    if (e != cudaSuccess)
        return (void) cudaGetLastError(), fail(COLOC_ERR_INVALID_TARGET,
            "cuda device " + std::to_string(dev) + ": " + cudaGetErrorString(e));
    std::memset(out, 0, sizeof *out);
    out->ordinal = dev;
    out->sm_count = p.multiProcessorCount;
    out->cc_major = p.major;
    out->cc_minor = p.minor;
    out->max_threads_per_sm = p.maxThreadsPerMultiProcessor;
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrClockRate, dev);
    out->sm_clock_khz = v;
    cudaDeviceGetAttribute(&v, cudaDevAttrMemoryClockRate, dev);
    out->mem_clock_khz = v;
    cudaDeviceGetAttribute(&v, cudaDevAttrGlobalMemoryBusWidth, dev);
    out->mem_bus_width_bits = v;
    out->l2_bytes = std::size_t(p.l2CacheSize);
    out->hbm_bytes = p.totalGlobalMem;
    std::snprintf(out->name, sizeof out->name, "%.127s", p.name);
    return COLOC_OK;
}

int coloc_cuda_stream_create(int dev, void** stream)
{
    if (!stream)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "stream_create: null out");
    COLOC_TRY(use_device(dev));
    cudaStream_t s = nullptr;
    COLOC_TRY_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking),
        "cudaStreamCreateWithFlags");
    *stream = s;
    return COLOC_OK;
}

int coloc_cuda_stream_destroy(int dev, void* stream)
{
    if (!stream)
        return COLOC_OK;
    COLOC_TRY(use_device(dev));
    chain_forget(dev, stream);
    COLOC_TRY_CUDA(cudaStreamDestroy(static_cast<cudaStream_t>(stream)),
        "cudaStreamDestroy");
    return COLOC_OK;
}

int coloc_cuda_stream_sync(int dev, void* stream)
{
    COLOC_TRY(use_device(dev));
    COLOC_TRY_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)),
        "cudaStreamSynchronize");
    return COLOC_OK;
}

int coloc_cuda_stream_query(int dev, void* stream, int* done)
{
    if (!done)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "stream_query: null out");
    COLOC_TRY(use_device(dev));
    cudaError_t e = cudaStreamQuery(static_cast<cudaStream_t>(stream));
    if (e == cudaErrorNotReady)
    {
        (void) cudaGetLastError();    // not an error: keep it out of later launch checks
        *done = 0;
        return COLOC_OK;
    }
    COLOC_TRY_CUDA(e, "cudaStreamQuery");
    *done = 1;
    return COLOC_OK;
}

int coloc_cuda_device_sync(int dev)
{
    COLOC_TRY(use_device(dev));
    COLOC_TRY_CUDA(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
    return COLOC_OK;
}

int coloc_cuda_malloc(int dev, size_t bytes, void** ptr)
{
    if (!ptr)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "malloc: null out");
    *ptr = nullptr;
    COLOC_TRY(use_device(dev));
    if (bytes == 0)
        return COLOC_OK;
    cudaError_t e = cudaMalloc(ptr, bytes);
    if (e != cudaSuccess)
    {
        (void) cudaGetLastError();
        *ptr = nullptr;
        return fail(status_of(e),
            "allocation of " + std::to_string(bytes) + " bytes failed on cuda:" +
                std::to_string(dev) + " (" + cudaGetErrorString(e) + ")");
    }
    return COLOC_OK;
}

int coloc_cuda_free(int dev, void* ptr)
{
    if (!ptr)
        return COLOC_OK;
    COLOC_TRY(use_device(dev));
    COLOC_TRY_CUDA(cudaFree(ptr), "cudaFree");
    return COLOC_OK;
}

int coloc_cuda_mem_info(int dev, size_t* free_bytes, size_t* total_bytes)
{
    if (!free_bytes || !total_bytes)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "mem_info: null out");
    COLOC_TRY(use_device(dev));
    COLOC_TRY_CUDA(cudaMemGetInfo(free_bytes, total_bytes), "cudaMemGetInfo");
    return COLOC_OK;
}

int coloc_cuda_host_alloc(size_t bytes, void** ptr)
{
    if (!ptr)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "host_alloc: null out");
    *ptr = nullptr;
    if (bytes == 0)
        return COLOC_OK;
    // Large buffers: transparent-huge-page backed anonymous memory pinned
    // with cudaHostRegister.  2 MiB pages need 512x fewer IOMMU/GPU
    // translations than cudaHostAlloc's 4 KiB ones; both directions at
    // once over PCIe move 3-6% more (profiles/r01_probe_link_thp.jsonl).
    if (bytes >= kThpMinBytes)
        if (void* p = thp_pinned_alloc(bytes))
        {
            *ptr = p;
            return COLOC_OK;
        }
    cudaError_t e = cudaHostAlloc(ptr, bytes, cudaHostAllocPortable);
    if (e != cudaSuccess)
    {
        (void) cudaGetLastError();
        *ptr = nullptr;
        return fail(status_of(e) == COLOC_ERR_CUDA ? COLOC_ERR_ALLOCATION : status_of(e),
            "pinned host allocation of " + std::to_string(bytes) +
                " bytes failed (" + cudaGetErrorString(e) + ")");
    }
    return COLOC_OK;
}

int coloc_cuda_host_free(void* ptr)
{
    if (!ptr)
        return COLOC_OK;
    if (thp_pinned_free(ptr))
        return COLOC_OK;
    COLOC_TRY_CUDA(cudaFreeHost(ptr), "cudaFreeHost");
    return COLOC_OK;
}

int coloc_cuda_host_register(void* ptr, size_t bytes)
{
    if (!ptr || bytes == 0)
        return COLOC_OK;
    COLOC_TRY_CUDA(cudaHostRegister(ptr, bytes, cudaHostRegisterPortable),
        "cudaHostRegister");
    return COLOC_OK;
}

int coloc_cuda_host_unregister(void* ptr)
{
    if (!ptr)
        return COLOC_OK;
    COLOC_TRY_CUDA(cudaHostUnregister(ptr), "cudaHostUnregister");
    return COLOC_OK;
}

int coloc_cuda_memcpy_async(int dev, void* stream, void* dst, const void* src,
    size_t bytes)
{
    if (bytes == 0)
        return COLOC_OK;
    if (!dst || !src)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "memcpy_async: null pointer");
    COLOC_TRY(use_device(dev));
    auto* s = static_cast<cudaStream_t>(stream);
    if (bytes >= kStageMinBytes)
    {
        // pageable host side: pinned staging ring (staging.cu), unless the
        // stream is being captured into a graph (host copies cannot be)
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(s, &cap) != cudaSuccess)
            (void) cudaGetLastError();
        if (cap == cudaStreamCaptureStatusNone)
        {
            if (is_pageable_host(src) && is_device_memory(dst))
                return staged_h2d(dev, s, dst, src, bytes);
            if (is_pageable_host(dst) && is_device_memory(src))
                return staged_d2h(dev, s, dst, src, bytes);
        }
    }
    COLOC_TRY_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s), "cudaMemcpyAsync");
    return COLOC_OK;
}

int coloc_cuda_memcpy_stream_ordered(int dev, void* stream, void* dst, const void* src,
    size_t bytes)
{
    if (bytes == 0)
        return COLOC_OK;
    if (!dst || !src)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "memcpy_stream_ordered: null pointer");
    COLOC_TRY(use_device(dev));
    auto* s = static_cast<cudaStream_t>(stream);
    if (bytes >= kStageMinBytes)
    {
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(s, &cap) != cudaSuccess)
            (void) cudaGetLastError();
        if (cap == cudaStreamCaptureStatusNone)
        {
            if (is_pageable_host(src) && is_device_memory(dst))
                return staged_enqueue(dev, s, dst, src, bytes, /*h2d=*/true);
            if (is_pageable_host(dst) && is_device_memory(src))
                return staged_enqueue(dev, s, dst, src, bytes, /*h2d=*/false);
        }
    }
    COLOC_TRY_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s), "cudaMemcpyAsync");
    return COLOC_OK;
}

int coloc_cuda_staging_release(void)
{
    return staging_release();
}

int coloc_cuda_memcpy_peer_async(int dst_dev, void* dst, int src_dev,
    const void* src, size_t bytes, void* stream)
{
    if (bytes == 0)
        return COLOC_OK;
    if (!dst || !src)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "memcpy_peer_async: null pointer");
    COLOC_TRY(use_device(dst_dev));
    COLOC_TRY_CUDA(cudaMemcpyPeerAsync(dst, dst_dev, src, src_dev, bytes,
                       static_cast<cudaStream_t>(stream)),
        "cudaMemcpyPeerAsync");
    return COLOC_OK;
}

int coloc_cuda_enable_peer_access(int dev, int peer_dev)
{
    if (dev == peer_dev)
        return COLOC_OK;
    int can = 0;
    COLOC_TRY_CUDA(cudaDeviceCanAccessPeer(&can, dev, peer_dev),
        "cudaDeviceCanAccessPeer");
    if (!can)
        return fail(COLOC_ERR_UNSUPPORTED,
            "cuda:" + std::to_string(dev) + " cannot access cuda:" +
                std::to_string(peer_dev));
    COLOC_TRY(use_device(dev));
    cudaError_t e = cudaDeviceEnablePeerAccess(peer_dev, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled)
    {
        (void) cudaGetLastError();
        return COLOC_OK;
    }
    COLOC_TRY_CUDA(e, "cudaDeviceEnablePeerAccess");
    return COLOC_OK;
}

int coloc_cuda_event_create(int dev, void** event)
{
    if (!event)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "event_create: null out");
    COLOC_TRY(use_device(dev));
    cudaEvent_t ev = nullptr;
    COLOC_TRY_CUDA(cudaEventCreate(&ev), "cudaEventCreate");
    *event = ev;
    return COLOC_OK;
}

int coloc_cuda_event_destroy(int dev, void* event)
{
    if (!event)
        return COLOC_OK;
    COLOC_TRY(use_device(dev));
    COLOC_TRY_CUDA(cudaEventDestroy(static_cast<cudaEvent_t>(event)),
        "cudaEventDestroy");
    return COLOC_OK;
}

int coloc_cuda_event_record(int dev, void* event, void* stream)
{
    COLOC_TRY(use_device(dev));
    auto s = static_cast<cudaStream_t>(stream);
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    COLOC_TRY_CUDA(cudaStreamIsCapturing(s, &cap), "cudaStreamIsCapturing");
    // Inside a graph capture the record becomes an event-record node, so
    // replays timestamp it like an eager record.
    if (cap == cudaStreamCaptureStatusActive)
        COLOC_TRY_CUDA(cudaEventRecordWithFlags(static_cast<cudaEvent_t>(event), s,
                           cudaEventRecordExternal),
            "cudaEventRecordWithFlags");
    else
        COLOC_TRY_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(event), s), "cudaEventRecord");
    return COLOC_OK;
}

int coloc_cuda_graph_capture_begin(int dev, void* stream)
{
    COLOC_TRY(use_device(dev));
    COLOC_TRY_CUDA(cudaStreamBeginCapture(static_cast<cudaStream_t>(stream),
                       cudaStreamCaptureModeThreadLocal),
        "cudaStreamBeginCapture");
    return COLOC_OK;
}

int coloc_cuda_graph_capture_end(int dev, void* stream, void** graph_exec)
{
    if (!graph_exec)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "graph_capture_end: null out");
    *graph_exec = nullptr;
    COLOC_TRY(use_device(dev));
    cudaGraph_t g = nullptr;
    COLOC_TRY_CUDA(cudaStreamEndCapture(static_cast<cudaStream_t>(stream), &g),
        "cudaStreamEndCapture");
    cudaGraphExec_t ex = nullptr;
    cudaError_t e = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    COLOC_TRY_CUDA(e, "cudaGraphInstantiate");
    *graph_exec = ex;
    return COLOC_OK;
}

int coloc_cuda_graph_capture_end_many(int n, const int* devs, void* const* streams,
    void** graph_execs)
{
    if (n < 0 || (n > 0 && (!devs || !streams || !graph_execs)))
        return fail(COLOC_ERR_INVALID_ARGUMENT, "graph_capture_end_many: bad arguments");
    // End every capture before instantiating anything: instantiation is
    // not permitted while another stream of this thread is still capturing.
    std::vector<cudaGraph_t> graphs(std::size_t(n), nullptr);
    int st = COLOC_OK;
    for (int i = 0; i < n; ++i)
    {
        graph_execs[i] = nullptr;
        int const u = use_device(devs[i]);
        cudaError_t e = u == COLOC_OK ?
            cudaStreamEndCapture(static_cast<cudaStream_t>(streams[i]), &graphs[std::size_t(i)]) :
            cudaSuccess;
        if (st == COLOC_OK && u != COLOC_OK)
            st = u;
        else if (st == COLOC_OK && e != cudaSuccess)
            st = fail_cuda(e, "cudaStreamEndCapture");
        else if (e != cudaSuccess)
            (void) cudaGetLastError();
    }
    for (int i = 0; i < n && st == COLOC_OK; ++i)
    {
        st = use_device(devs[i]);
        if (st != COLOC_OK)
            break;
        cudaGraphExec_t ex = nullptr;
        cudaError_t e = cudaGraphInstantiate(&ex, graphs[std::size_t(i)], 0);
        if (e != cudaSuccess)
            st = fail_cuda(e, "cudaGraphInstantiate");
        else
            graph_execs[i] = ex;
    }
    for (int i = 0; i < n; ++i)
    {
        if (graphs[std::size_t(i)])
            (void) cudaGraphDestroy(graphs[std::size_t(i)]);
        if (st != COLOC_OK && graph_execs[i])
        {
            (void) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(graph_execs[i]));
            graph_execs[i] = nullptr;
        }
    }
    return st;
}

int coloc_cuda_graph_launch(int dev, void* graph_exec, void* stream)
{
    COLOC_TRY(use_device(dev));
    COLOC_TRY_CUDA(cudaGraphLaunch(static_cast<cudaGraphExec_t>(graph_exec),
                       static_cast<cudaStream_t>(stream)),
        "cudaGraphLaunch");
    return COLOC_OK;
}

int coloc_cuda_graph_destroy(int dev, void* graph_exec)
{
    if (!graph_exec)
        return COLOC_OK;
    COLOC_TRY(use_device(dev));
    COLOC_TRY_CUDA(cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(graph_exec)),
        "cudaGraphExecDestroy");
    return COLOC_OK;
}

int coloc_cuda_event_sync(void* event)
{
    COLOC_TRY_CUDA(cudaEventSynchronize(static_cast<cudaEvent_t>(event)),
        "cudaEventSynchronize");
    return COLOC_OK;
}

int coloc_cuda_event_query(void* event, int* done)
{
    if (!done)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "event_query: null out");
    cudaError_t e = cudaEventQuery(static_cast<cudaEvent_t>(event));
    if (e == cudaErrorNotReady)
    {
        (void) cudaGetLastError();    // not an error: keep it out of later launch checks
        *done = 0;
        return COLOC_OK;
    }
    COLOC_TRY_CUDA(e, "cudaEventQuery");
    *done = 1;
    return COLOC_OK;
}

int coloc_cuda_event_elapsed_ms(void* start, void* stop, float* ms)
{
    if (!ms)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "event_elapsed: null out");
    COLOC_TRY_CUDA(cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(start),
                       static_cast<cudaEvent_t>(stop)),
        "cudaEventElapsedTime");
    return COLOC_OK;
}

int coloc_cuda_stream_fork_timestamp(int dev, void* stream, void* side, void* event)
{
    if (!event || !side)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "stream_fork_timestamp: null side stream or event");
    COLOC_TRY(use_device(dev));
    auto* s = static_cast<cudaStream_t>(stream);
    auto* q = static_cast<cudaStream_t>(side);
    // a dependency token only (plain record, also inside a capture), then
    // the timing record on the side stream: later work on `stream` does
    // not wait for it
    cudaEvent_t fork = nullptr;
    COLOC_TRY_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming), "cudaEventCreate");
    cudaError_t e = cudaEventRecord(fork, s);
    if (e == cudaSuccess)
        e = cudaStreamWaitEvent(q, fork, 0);
    (void) cudaEventDestroy(fork);
    COLOC_TRY_CUDA(e, "stream_fork_timestamp: fork");
    return coloc_cuda_event_record(dev, event, side);
}

int coloc_cuda_stream_join(int dev, void* stream, void* side)
{
    if (!side)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "stream_join: null side stream");
    COLOC_TRY(use_device(dev));
    cudaEvent_t join = nullptr;
    COLOC_TRY_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming), "cudaEventCreate");
    cudaError_t e = cudaEventRecord(join, static_cast<cudaStream_t>(side));
    if (e == cudaSuccess)
        e = cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), join, 0);
    (void) cudaEventDestroy(join);
    COLOC_TRY_CUDA(e, "stream_join");
    return COLOC_OK;
}

int coloc_cuda_stream_wait_event(int dev, void* stream, void* event)
{
    COLOC_TRY(use_device(dev));
    COLOC_TRY_CUDA(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream),
                       static_cast<cudaEvent_t>(event), 0),
        "cudaStreamWaitEvent");
    return COLOC_OK;
}

namespace {
struct host_fn_box
{
    coloc_cuda_host_fn fn;
    void* user;
};

// A stream callback (cudaStreamAddCallback) rather than cudaLaunchHostFunc:
// the runtime passes the status of the preceding work, so a device fault
// before the callback settles the caller's future with an error instead of
// a success (the reference's futures carry the first error,
// detail/bulk.hpp:67-91).  No CUDA call may be made in here.
void CUDART_CB host_fn_trampoline(cudaStream_t, cudaError_t status, void* p)
{
    auto* box = static_cast<host_fn_box*>(p);
    box->fn(box->user, status == cudaSuccess ? COLOC_OK : status_of(status));
    delete box;
}
}    // namespace

int coloc_cuda_launch_host_func(int dev, void* stream, coloc_cuda_host_fn fn,
    void* user)
{
    if (!fn)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "launch_host_func: null fn");
    COLOC_TRY(use_device(dev));
    auto* box = new host_fn_box{fn, user};
    cudaError_t e = cudaStreamAddCallback(static_cast<cudaStream_t>(stream),
        host_fn_trampoline, box, 0);
    if (e != cudaSuccess)
    {
        delete box;
        return fail_cuda(e, "cudaStreamAddCallback");
    }
    return COLOC_OK;
}

}    // extern "C"
