// probe.cu -- measurement probes (not part of the hot path).
//
// They bound the STREAM kernels from the hardware side, with the same
// tile shape and cache hints as ew_pack_kernel:
//   probe_read   reads a buffer once (256-bit evict-first loads) and folds
//                it into a register that is stored only on an impossible
//                value: the HBM read-only ceiling;
//   (write-only) is coloc_cuda_fill, the elementwise kernel with no input;
//   probe_empty  an empty one-CTA kernel: the launch / event-boundary floor
//                of a timed STREAM kernel at small sizes (BASELINE config C5).
#include "common.h"
#include "coloc_b200/kernels/elementwise.cuh"

namespace coloc_cuda {
namespace {

constexpr int kProbeThreads = 1024;
constexpr int kProbeUnroll = 2;

__global__ void __launch_bounds__(kProbeThreads) probe_read_kernel(std::uint64_t const* x,
    std::size_t npacks, unsigned long long* sink)
{
    std::size_t const tile = std::size_t(blockDim.x) * kProbeUnroll;
    std::size_t const p0 = std::size_t(blockIdx.x) * tile + threadIdx.x;
    std::uint64_t acc = 0;
#pragma unroll
    for (int u = 0; u < kProbeUnroll; ++u)
    {
        std::size_t const p = p0 + std::size_t(u) * blockDim.x;
        if (p < npacks)
        {
            std::uint64_t w[4];
            ld_pack<1>(x + p * 4, w);
            acc ^= w[0] ^ w[1] ^ w[2] ^ w[3];
        }
    }
    // A store that (practically) never happens keeps the loads live
    // without the traffic or contention of a real reduction.
    if (acc == 0x5a17c0de5a17c0deULL)
        atomicXor(sink, (unsigned long long) acc);
}

__global__ void probe_empty_kernel() {}

}    // namespace
}    // namespace coloc_cuda

using namespace coloc_cuda;

extern "C" {

int coloc_cuda_probe_read(int dev, void* stream_handle, const void* x, size_t bytes,
    uint64_t* dev_sink)
{
    if (bytes == 0)
        return COLOC_OK;
    if (!x || !dev_sink)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "probe_read: null pointer");
    if (reinterpret_cast<std::uintptr_t>(x) % kPackBytes || bytes % kPackBytes)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "probe_read: buffer must be 32-byte aligned and sized");
    COLOC_TRY(use_device(dev));
    std::size_t const npacks = bytes / kPackBytes;
    std::size_t const tile = std::size_t(kProbeThreads) * kProbeUnroll;
    std::size_t const grid = (npacks + tile - 1) / tile;
    if (grid > 0x7fffffffu)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "probe_read: buffer too large");
    probe_read_kernel<<<unsigned(grid), kProbeThreads, 0, static_cast<cudaStream_t>(stream_handle)>>>(
        static_cast<std::uint64_t const*>(x), npacks, reinterpret_cast<unsigned long long*>(dev_sink));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    COLOC_TRY_CUDA(cudaGetLastError(), "probe_read kernel");
    return COLOC_OK;
}

int coloc_cuda_probe_empty(int dev, void* stream_handle)
{
    COLOC_TRY(use_device(dev));
    probe_empty_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream_handle)>>>();
    g_launches.fetch_add(1, std::memory_order_relaxed);
    COLOC_TRY_CUDA(cudaGetLastError(), "probe_empty kernel");
    return COLOC_OK;
}

}    // extern "C"
