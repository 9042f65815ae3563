// bulk.cuh -- TMA (cp.async.bulk) variant of the STREAM kernels.
//
// Same operations as ew_pack_kernel, different data movement: a persistent
// CTA streams fixed-size chunks global -> shared memory with 1-D bulk copies
// completing on mbarriers (UBLKCP in SASS), computes in shared memory, and
// writes each chunk back with a bulk store (shared -> global).  One thread
// issues all copies, so the SM's issue slots are nearly idle; a STAGES-deep
// ring keeps (STAGES-1) chunk loads in flight while the previous chunk's
// store drains.  Chunks are handed out by an atomic counter so the active
// address window stays compact and the tail stays balanced.
//
// Requirements (checked by the launcher): the body is 32-byte aligned
// (bulk copies need 16-byte alignment and 16-byte multiples), head/tail
// elements are handled like ew_pack_kernel.
#pragma once

#include "coloc_b200/kernels/elementwise.cuh"

#include <cstdint>

namespace coloc_cuda {

constexpr int kBulkThreads = 256;

__device__ __forceinline__ std::uint32_t smem_u32(void const* p)
{
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(std::uint64_t* bar, std::uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* bar, std::uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, std::uint32_t parity)
{
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t"
        "}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_load(void* smem_dst, void const* gmem_src, std::uint32_t bytes,
    std::uint64_t* bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem_dst)),
        "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void bulk_store(void* gmem_dst, void const* smem_src, std::uint32_t bytes)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem_dst),
                 "r"(smem_u32(smem_src)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

template <int N>
__device__ __forceinline__ void bulk_wait_read()
{
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void bulk_wait_all()
{
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Scheduler state in global memory: [0] next chunk, [1] finished CTAs.
// The last CTA to finish resets both, so consecutive launches on the same
// stream reuse it without a memset.
struct bulk_sched
{
    unsigned long long next;
    unsigned long long done;
};

// chunk_bytes per input; smem = STAGES * NIN * chunk_bytes (+ barriers).
template <typename T, typename Op, int STAGES>
__global__ void __launch_bounds__(kBulkThreads, 1) ew_bulk_kernel(Op op, T* dst, T const* s0,
    T const* s1, std::size_t head, std::size_t body_bytes, std::size_t tail,
    std::uint32_t chunk_bytes, bulk_sched* sched)
{
    constexpr int NIN = Op::nin > 0 ? Op::nin : 1;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ std::uint64_t full[STAGES];
    __shared__ unsigned long long chunk_of[STAGES];

    std::size_t const nchunks = (body_bytes + chunk_bytes - 1) / chunk_bytes;
    unsigned char* bd = reinterpret_cast<unsigned char*>(dst + head);
    unsigned char const* b0 = Op::nin >= 1 ? reinterpret_cast<unsigned char const*>(s0 + head) : nullptr;
    unsigned char const* b1 = Op::nin >= 2 ? reinterpret_cast<unsigned char const*>(s1 + head) : nullptr;
    auto buf = [&](int stage, int k) { return smem + (std::size_t(stage) * NIN + k) * chunk_bytes; };
    bool const leader = threadIdx.x == 0;

    // Producer step: claim a chunk and start its loads into `stage`.
    auto issue = [&](int stage) {
        unsigned long long c = atomicAdd(&sched->next, 1ull);
        chunk_of[stage] = c;
        if (c >= nchunks)
        {
            // no work: complete the phase without transactions
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[stage]))
                         : "memory");
            return;
        }
        std::size_t const off = std::size_t(c) * chunk_bytes;
        std::uint32_t const bytes = std::uint32_t(
            body_bytes - off < chunk_bytes ? body_bytes - off : std::size_t(chunk_bytes));
        if constexpr (Op::nin == 0)
        {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[stage]))
                         : "memory");
        }
        else
        {
            mbar_expect_tx(&full[stage], bytes * Op::nin);
            bulk_load(buf(stage, 0), b0 + off, bytes, &full[stage]);
            if constexpr (Op::nin >= 2)
                bulk_load(buf(stage, 1), b1 + off, bytes, &full[stage]);
        }
    };

    if (leader)
    {
        for (int s = 0; s < STAGES; ++s)
            mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (leader)
        for (int s = 0; s < STAGES - 1; ++s)
            issue(s);

    for (std::uint32_t j = 0;; ++j)
    {
        int const stage = int(j % STAGES);
        std::uint32_t const parity = (j / STAGES) & 1u;
        // keep STAGES-1 chunks in flight: refill the stage freed by the
        // store issued in the previous iteration
        if (leader)
        {
            bulk_wait_read<0>();
            issue(int((j + STAGES - 1) % STAGES));
        }
        mbar_wait(&full[stage], parity);
        unsigned long long const c = chunk_of[stage];
        if (c >= nchunks)
            break;
        std::size_t const off = std::size_t(c) * chunk_bytes;
        std::uint32_t const bytes = std::uint32_t(
            body_bytes - off < chunk_bytes ? body_bytes - off : std::size_t(chunk_bytes));
        if constexpr (!Op::identity)
        {
            constexpr int E = kPackBytes / int(sizeof(T));
            std::uint32_t const npk = bytes / kPackBytes;
            for (std::uint32_t p = threadIdx.x; p < npk; p += kBulkThreads)
            {
                pack<T> x, y, o;
                if constexpr (Op::nin >= 1)
                    x = reinterpret_cast<pack<T> const*>(buf(stage, 0))[p];
                if constexpr (Op::nin >= 2)
                    y = reinterpret_cast<pack<T> const*>(buf(stage, 1))[p];
                std::size_t const e0 = head + (off / sizeof(T)) + std::size_t(p) * E;
#pragma unroll
                for (int e = 0; e < E; ++e)
                    o.v[e] = op(e0 + e, Op::nin >= 1 ? x.v[e] : T(), Op::nin >= 2 ? y.v[e] : T());
                reinterpret_cast<pack<T>*>(buf(stage, 0))[p] = o;
            }
            fence_proxy_async_smem();
        }
        // all threads are done with this stage (data and chunk_of[stage])
        // before the leader stores it and later refills it
        __syncthreads();
        if (leader)
            bulk_store(bd + off, buf(stage, 0), bytes);
    }

    if (leader)
    {
        bulk_wait_all();
        __threadfence();
        unsigned long long const d = atomicAdd(&sched->done, 1ull);
        if (d == gridDim.x - 1)
        {
            sched->next = 0;
            sched->done = 0;
            __threadfence();
        }
    }
    // head / tail elements (< 32 B each side), last CTA
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x < head + tail)
    {
        std::size_t const r = threadIdx.x;
        std::size_t const nbody = body_bytes / sizeof(T);
        std::size_t const i = r < head ? r : head + nbody + (r - head);
        dst[i] = op(i, Op::nin >= 1 ? s0[i] : T(), Op::nin >= 2 ? s1[i] : T());
    }
}

}    // namespace coloc_cuda
