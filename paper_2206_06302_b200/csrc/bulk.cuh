// bulk.cuh -- TMA (cp.async.bulk) variant of the STREAM kernels.
//
// Same operations as ew_pack_kernel, different data movement: persistent
// CTAs stream fixed-size chunks global -> shared memory with 1-D bulk
// copies completing on mbarriers (UBLKCP in SASS), compute in shared
// memory, and write each chunk back with a bulk store (shared -> global).
// One producer thread issues every load, so the SM's issue slots stay
// nearly idle; chunks are handed out by an atomic counter so the active
// address window stays compact and the tail stays balanced.
//
// Requirements (checked by the launcher): the body is 32-byte aligned
// (bulk copies need 16-byte alignment and 16-byte multiples); head/tail
// elements are handled like ew_pack_kernel.
#pragma once

#include "coloc_b200/kernels/elementwise.cuh"

#include <cstdint>

namespace coloc_cuda {

constexpr int kTmaConsumerWarps = 4;
constexpr int kTmaThreads = 32 * (1 + kTmaConsumerWarps);    // warp 0 produces
constexpr int kTmaOutStages = 2;

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

// L2 evict-first policy for streamed data (the bulk-copy counterpart of
// the LDG/STG kernels' L2::evict_first).
__device__ __forceinline__ std::uint64_t evict_first_policy()
{
    std::uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ void bulk_load_hint(void* smem_dst, void const* gmem_src,
    std::uint32_t bytes, std::uint64_t* bar, std::uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(smem_dst)),
        "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

__device__ __forceinline__ void bulk_store(void* gmem_dst, void const* smem_src, std::uint32_t bytes)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem_dst),
                 "r"(smem_u32(smem_src)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

__device__ __forceinline__ void bulk_store_hint(void* gmem_dst, void const* smem_src,
    std::uint32_t bytes, std::uint64_t pol)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                     gmem_dst),
                 "r"(smem_u32(smem_src)), "r"(bytes), "l"(pol)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

template <bool Hint>
__device__ __forceinline__ void bulk_load_p(void* smem_dst, void const* gmem_src, std::uint32_t bytes,
    std::uint64_t* bar, std::uint64_t pol)
{
    if constexpr (Hint)
        bulk_load_hint(smem_dst, gmem_src, bytes, bar, pol);
    else
        bulk_load(smem_dst, gmem_src, bytes, bar);
}

template <bool Hint>
__device__ __forceinline__ void bulk_store_p(void* gmem_dst, void const* smem_src, std::uint32_t bytes,
    std::uint64_t pol)
{
    if constexpr (Hint)
        bulk_store_hint(gmem_dst, smem_src, bytes, pol);
    else
        bulk_store(gmem_dst, smem_src, bytes);
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

template <typename T>
union quad
{
    uint4 u;
    T v[16 / sizeof(T)];
};

__device__ __forceinline__ void mbar_arrive(std::uint64_t* bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Barrier among the consumer warps only (the producer warp never joins).
__device__ __forceinline__ void consumer_sync()
{
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kTmaConsumerWarps) : "memory");
}

// Warp-specialised TMA pipeline.
//   warp 0, lane 0 (producer): claims chunks and streams their NIN inputs
//     global -> shared with bulk copies into a `stages`-deep input ring;
//     full[s] completes on the transaction bytes, empty[s] when the slot's
//     consumers are done with it.  Chunks are claimed round robin
//     (chunk = blockIdx.x + j*gridDim.x: no atomics, and all CTAs advance
//     through one compact address window) or from an atomic counter
//     (`dynamic`: balanced tail).
//   warps 1..kTmaConsumerWarps (consumers): compute out = op(in...) from the
//     input slot into a 2-deep output ring, release the input slot, and one
//     consumer thread writes the chunk back with a bulk store (shared ->
//     global), waiting only for the store issued two chunks earlier before
//     its output buffer is reused.
//   Identity ops (copy) skip the compute: the storer writes each chunk back
//     straight from its input slot and releases the slot once the store
//     issued kCopyLag chunks later has been read out of shared memory.
// Smem = stages * NIN * chunk (inputs) + kTmaOutStages * chunk (outputs,
// not used by identity ops).
constexpr int kMaxTmaStages = 8;
constexpr int kCopyLag = 2;    // identity ops: stores in flight per CTA

template <typename Op>
constexpr int tma_out_stages() { return Op::identity ? 0 : kTmaOutStages; }

template <typename T, typename Op, bool Hint>
__global__ void __launch_bounds__(kTmaThreads) ew_bulk_kernel(Op op, T* dst, T const* s0,
    T const* s1, std::size_t head, std::size_t body_bytes, std::size_t tail,
    std::uint32_t chunk_bytes, int stages, int dynamic, bulk_sched* sched)
{
    constexpr int NIN = Op::nin > 0 ? Op::nin : 1;
    constexpr int E16 = 16 / int(sizeof(T));
    constexpr int kConsumers = 32 * kTmaConsumerWarps;
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ std::uint64_t full[kMaxTmaStages], empty[kMaxTmaStages];
    __shared__ unsigned long long chunk_of[kMaxTmaStages];

    std::size_t const nchunks = (body_bytes + chunk_bytes - 1) / chunk_bytes;
    unsigned char* bd = reinterpret_cast<unsigned char*>(dst + head);
    unsigned char const* b0 = Op::nin >= 1 ? reinterpret_cast<unsigned char const*>(s0 + head) : nullptr;
    unsigned char const* b1 = Op::nin >= 2 ? reinterpret_cast<unsigned char const*>(s1 + head) : nullptr;
    auto in_buf = [&](int s, int k) { return smem + (std::size_t(s) * NIN + k) * chunk_bytes; };
    auto out_buf = [&](int o) { return smem + (std::size_t(stages) * NIN + o) * chunk_bytes; };
    auto chunk_len = [&](std::size_t off) {
        return std::uint32_t(body_bytes - off < chunk_bytes ? body_bytes - off : std::size_t(chunk_bytes));
    };
    int const warp = int(threadIdx.x) / 32, lane = int(threadIdx.x) % 32;
    std::uint64_t const pol = Hint ? evict_first_policy() : 0;

    if (threadIdx.x == 0)
    {
        for (int s = 0; s < stages; ++s)
        {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], Op::identity ? 1 : kTmaConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == 0)
    {
        if (lane == 0)
        {
            for (std::uint32_t j = 0;; ++j)
            {
                int const s = int(j % unsigned(stages));
                if (j >= unsigned(stages))    // the slot's previous use has been consumed
                    mbar_wait(&empty[s], ((j / unsigned(stages)) & 1u) ^ 1u);
                unsigned long long const c = dynamic
                    ? atomicAdd(&sched->next, 1ull)
                    : (unsigned long long) blockIdx.x + (unsigned long long) j * gridDim.x;
                chunk_of[s] = c;
                if (c >= nchunks)
                {
                    mbar_arrive(&full[s]);    // end marker, no transactions
                    break;
                }
                std::size_t const off = std::size_t(c) * chunk_bytes;
                std::uint32_t const bytes = chunk_len(off);
                if constexpr (Op::nin == 0)
                    mbar_arrive(&full[s]);
                else
                {
                    mbar_expect_tx(&full[s], bytes * Op::nin);
                    bulk_load_p<Hint>(in_buf(s, 0), b0 + off, bytes, &full[s], pol);
                    if constexpr (Op::nin >= 2)
                        bulk_load_p<Hint>(in_buf(s, 1), b1 + off, bytes, &full[s], pol);
                }
            }
            if (dynamic)
            {
                // every claim of this CTA is done; the last CTA resets the
                // scheduler for the next launch on this stream
                __threadfence();
                if (atomicAdd(&sched->done, 1ull) == gridDim.x - 1)
                {
                    sched->next = 0;
                    sched->done = 0;
                    __threadfence();
                }
            }
        }
    }
    else if constexpr (Op::identity)
    {
        // copy: one thread stores chunks straight from the input ring
        if (threadIdx.x == 32)
        {
            for (std::uint32_t j = 0;; ++j)
            {
                int const s = int(j % unsigned(stages));
                mbar_wait(&full[s], (j / unsigned(stages)) & 1u);
                unsigned long long const c = chunk_of[s];
                if (c >= nchunks)
                    break;
                std::size_t const off = std::size_t(c) * chunk_bytes;
                bulk_store_p<Hint>(bd + off, in_buf(s, 0), chunk_len(off), pol);
                // stores up to chunk j - kCopyLag have left shared memory
                bulk_wait_read<kCopyLag>();
                if (j >= unsigned(kCopyLag))
                    mbar_arrive(&empty[(j - kCopyLag) % unsigned(stages)]);
            }
            bulk_wait_all();
        }
    }
    else
    {
        int const ct = int(threadIdx.x) - 32;
        bool const storer = ct == 0;
        for (std::uint32_t j = 0;; ++j)
        {
            int const s = int(j % unsigned(stages));
            mbar_wait(&full[s], (j / unsigned(stages)) & 1u);
            unsigned long long const c = chunk_of[s];
            if (c >= nchunks)
                break;
            std::size_t const off = std::size_t(c) * chunk_bytes;
            std::uint32_t const bytes = chunk_len(off);
            int const o = int(j % kTmaOutStages);
            if (storer)    // out[o]'s store from kTmaOutStages chunks ago has been read
                bulk_wait_read<kTmaOutStages - 1>();
            consumer_sync();
            // 16-byte units, consecutive threads on consecutive units: each
            // quarter warp touches one 128-byte row, so LDS.128/STS.128 run
            // without bank conflicts
            std::uint32_t const nq = bytes / 16;
            std::size_t const e_base = head + off / sizeof(T);
            for (std::uint32_t q = std::uint32_t(ct); q < nq; q += kConsumers)
            {
                quad<T> x, y, r;
                if constexpr (Op::nin >= 1)
                    x.u = reinterpret_cast<uint4 const*>(in_buf(s, 0))[q];
                if constexpr (Op::nin >= 2)
                    y.u = reinterpret_cast<uint4 const*>(in_buf(s, 1))[q];
#pragma unroll
                for (int e = 0; e < E16; ++e)
                    r.v[e] = op(e_base + std::size_t(q) * E16 + e, Op::nin >= 1 ? x.v[e] : T(),
                        Op::nin >= 2 ? y.v[e] : T());
                reinterpret_cast<uint4*>(out_buf(o))[q] = r.u;
            }
            __syncwarp();
            if (lane == 0)
                mbar_arrive(&empty[s]);    // input slot free for the producer
            fence_proxy_async_smem();          // generic smem writes -> async proxy
            consumer_sync();
            if (storer)
                bulk_store_p<Hint>(bd + off, out_buf(o), bytes, pol);
        }
        if (storer)
            bulk_wait_all();
    }

    // head / tail elements (< 32 B each side), last CTA, consumer threads
    if (warp > 0 && blockIdx.x == gridDim.x - 1)
        for (std::size_t r = threadIdx.x - 32; r < head + tail; r += blockDim.x - 32)
        {
            std::size_t const nbody = body_bytes / sizeof(T);
            std::size_t const i = r < head ? r : head + nbody + (r - head);
            dst[i] = op(i, Op::nin >= 1 ? s0[i] : T(), Op::nin >= 2 ? s1[i] : T());
        }
}


// Hybrid: LDG loads into registers as ew_pack_kernel does (one tile per
// CTA), the tile's results staged in shared memory and written back with
// ONE bulk store per CTA (blockDim * U * 32 bytes contiguous), so the DRAM
// sees long write bursts instead of per-warp 1 KB stores.
template <typename T, typename Op, int U>
__global__ void __launch_bounds__(1024) ew_ldg_bulkst_kernel(Op op, T* dst, T const* s0,
    T const* s1, std::size_t head, std::size_t npacks, std::size_t tail)
{
    constexpr int E = kPackBytes / int(sizeof(T));
    extern __shared__ __align__(1024) unsigned char smem[];
    std::size_t const tile = std::size_t(blockDim.x) * U;
    std::size_t const t0 = std::size_t(blockIdx.x) * tile;
    std::size_t const here = npacks - t0 < tile ? npacks - t0 : tile;    // packs in this tile
    T* bd = dst + head;
    T const* b0 = Op::nin >= 1 ? s0 + head : nullptr;
    T const* b1 = Op::nin >= 2 ? s1 + head : nullptr;
    std::uint64_t const pol = evict_first_policy();

    pack<T> x[U], y[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
    {
        std::size_t const q = threadIdx.x + std::size_t(u) * blockDim.x;
        if (q < here)
        {
            if constexpr (Op::nin >= 1)
                ld_pack<1>(b0 + (t0 + q) * E, x[u].w);
            if constexpr (Op::nin >= 2)
                ld_pack<1>(b1 + (t0 + q) * E, y[u].w);
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
    {
        std::size_t const q = threadIdx.x + std::size_t(u) * blockDim.x;
        if (q < here)
        {
            pack<T> o;
            if constexpr (Op::identity)
                o = x[u];
            else
            {
#pragma unroll
                for (int j = 0; j < E; ++j)
                    o.v[j] = op(head + (t0 + q) * E + std::size_t(j), Op::nin >= 1 ? x[u].v[j] : T(),
                        Op::nin >= 2 ? y[u].v[j] : T());
            }
            // two 16-byte halves: consecutive threads on consecutive 32 B
            auto* d = reinterpret_cast<uint4*>(smem + q * kPackBytes);
            d[0] = make_uint4(unsigned(o.w[0]), unsigned(o.w[0] >> 32), unsigned(o.w[1]), unsigned(o.w[1] >> 32));
            d[1] = make_uint4(unsigned(o.w[2]), unsigned(o.w[2] >> 32), unsigned(o.w[3]), unsigned(o.w[3] >> 32));
        }
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0 && here > 0)
    {
        bulk_store_hint(bd + t0 * E, smem, std::uint32_t(here * kPackBytes), pol);
        bulk_wait_read<0>();
    }
    if (blockIdx.x == gridDim.x - 1)
        for (std::size_t r = threadIdx.x; r < head + tail; r += blockDim.x)
        {
            std::size_t const i = r < head ? r : head + npacks * E + (r - head);
            dst[i] = op(i, Op::nin >= 1 ? s0[i] : T(), Op::nin >= 2 ? s1[i] : T());
        }
}

}    // namespace coloc_cuda
