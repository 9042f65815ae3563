// elementwise.cuh -- the STREAM hot-path kernel template for sm_100a.
//
// One kernel shape serves every elementwise operation of the path
// (copy / scale / add / triad, construction fills and generators): the
// reference runs these as `for i in range: f(i)` on a pinned worker
// (detail/bulk.hpp:36-41, called from algorithms.hpp:384-386, 466-467,
// 505-506); here each CTA streams contiguous tiles of 32-byte packs.
//
// Layout: the range [0, n) is split into an unaligned head (< 32 B), a body
// of 32-byte packs starting at a 32-byte-aligned destination address, and
// a tail (< 32 B).  The body uses 256-bit LDG/STG (LDG.E.256 on sm_100a),
// `U` packs per thread per input issued back to back before any store so
// each thread keeps U*NIN*32 bytes in flight (Little's law at ~7 TB/s
// needs ~40-50 KB in flight per SM).  A tile is blockDim*U packs; CTAs walk
// tiles with a grid stride (persistent grid) or take exactly one tile each.
// Cache hint 1 marks loads L1::no_allocate + L2::evict_first and stores
// L1::no_allocate + L2::evict_first: streamed data is touched once.
#pragma once

#include <cstddef>
#include <cstdint>

namespace coloc_cuda {

constexpr int kPackBytes = 32;

template <typename T>
union pack
{
    std::uint64_t w[4];
    T v[kPackBytes / sizeof(T)];
};

// Hints: 0 plain; 1 streaming (L1 no-allocate, L2 evict-first) loads and
// stores; 2 = 1 + L2 256 B prefetch on loads; 3 streaming loads, stores
// kept in L2 (evict-last: the next kernel of a chain reads them from L2);
// 4 plain loads, evict-last stores; 5 streaming loads, stores evict-last
// for a fraction of the lines (an L2 cache policy, `l2_policy`) and
// evict-first for the rest: the part of an output larger than L2 that
// fits stays there for the next kernel.
template <int Hint>
__device__ __forceinline__ void ld_pack(void const* p, std::uint64_t (&w)[4])
{
    if constexpr (Hint == 1 || Hint == 3 || Hint == 5)
        asm volatile(
            "ld.global.L1::no_allocate.L2::evict_first.v4.u64 {%0,%1,%2,%3}, [%4];"
            : "=l"(w[0]), "=l"(w[1]), "=l"(w[2]), "=l"(w[3])
            : "l"(p));
    else if constexpr (Hint == 2)    // + L2 prefetch of the surrounding 256 B
        asm volatile(
            "ld.global.L1::no_allocate.L2::evict_first.L2::256B.v4.u64 {%0,%1,%2,%3}, [%4];"
            : "=l"(w[0]), "=l"(w[1]), "=l"(w[2]), "=l"(w[3])
            : "l"(p));
    else
        asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(w[0]), "=l"(w[1]), "=l"(w[2]), "=l"(w[3])
                     : "l"(p));
}

__device__ __forceinline__ std::uint64_t l2_policy(float keep)
{
    std::uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.L2::evict_first.b64 %0, %1;"
                 : "=l"(pol)
                 : "f"(keep));
    return pol;
}

template <int Hint>
__device__ __forceinline__ void st_pack(void* p, std::uint64_t const (&w)[4], std::uint64_t pol = 0)
{
    if constexpr (Hint == 5)
        asm volatile(
            "st.global.L1::no_allocate.L2::cache_hint.v4.u64 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p),
            "l"(w[0]), "l"(w[1]), "l"(w[2]), "l"(w[3]), "l"(pol)
            : "memory");
    else if constexpr (Hint >= 3)
        asm volatile(
            "st.global.L1::no_allocate.L2::evict_last.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(p),
            "l"(w[0]), "l"(w[1]), "l"(w[2]), "l"(w[3])
            : "memory");
    else if constexpr (Hint >= 1)
        asm volatile(
            "st.global.L1::no_allocate.L2::evict_first.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(p),
            "l"(w[0]), "l"(w[1]), "l"(w[2]), "l"(w[3])
            : "memory");
    else
        asm volatile("st.global.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(w[0]),
                     "l"(w[1]), "l"(w[2]), "l"(w[3])
                     : "memory");
}

// ---------------------------------------------------------------------
// Operations.  `nin` inputs; idx is the element index within the range
// (used by generators).  Rounding intrinsics (__dmul_rn etc.) are never
// contracted into FMA, which is what makes scale/add/triad bit-exact
// against the reference's uncontracted x86-64 build.
// ---------------------------------------------------------------------

__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
// Integers: two's complement wrap-around (computed unsigned, no signed
// overflow UB), what the reference's x86-64 build does for int vectors.
__device__ __forceinline__ std::int32_t mul_rn(std::int32_t a, std::int32_t b)
{
    return std::int32_t(std::uint32_t(a) * std::uint32_t(b));
}
__device__ __forceinline__ std::int64_t mul_rn(std::int64_t a, std::int64_t b)
{
    return std::int64_t(std::uint64_t(a) * std::uint64_t(b));
}
__device__ __forceinline__ std::int32_t add_rn(std::int32_t a, std::int32_t b)
{
    return std::int32_t(std::uint32_t(a) + std::uint32_t(b));
}
__device__ __forceinline__ std::int64_t add_rn(std::int64_t a, std::int64_t b)
{
    return std::int64_t(std::uint64_t(a) + std::uint64_t(b));
}
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }

struct op_copy
{
    static constexpr int nin = 1;
    static constexpr bool identity = true;
    template <typename T>
    __device__ T operator()(std::size_t, T x, T) const { return x; }
};

template <typename T>
struct op_scale
{
    static constexpr int nin = 1;
    static constexpr bool identity = false;
    T s;
    __device__ T operator()(std::size_t, T c, T) const { return mul_rn(c, s); }
};

template <typename T>
struct op_add
{
    static constexpr int nin = 2;
    static constexpr bool identity = false;
    __device__ T operator()(std::size_t, T a, T b) const { return add_rn(a, b); }
};

// a = b + c*s (Listing 4's Triad: `return b + c*scalar`).
template <typename T, bool Fma>
struct op_triad
{
    static constexpr int nin = 2;
    static constexpr bool identity = false;
    T s;
    __device__ T operator()(std::size_t, T b, T c) const
    {
        if constexpr (Fma)
            return fma_rn(c, s, b);
        else
            return add_rn(b, mul_rn(c, s));
    }
};

struct op_to_upper
{
    static constexpr int nin = 1;
    static constexpr bool identity = false;
    __device__ unsigned char operator()(std::size_t, unsigned char ch, unsigned char) const
    {
        return (ch >= 'a' && ch <= 'z') ? (unsigned char) (ch - 32) : ch;
    }
};

template <typename T>
struct op_fill
{
    static constexpr int nin = 0;
    static constexpr bool identity = false;
    T v;
    __device__ T operator()(std::size_t, T, T) const { return v; }
};

__device__ __forceinline__ std::uint64_t mix64(std::uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

constexpr std::uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
constexpr std::uint64_t kArrayStride = 0xD1B54A32D192ED03ULL;

// Counter-based splitmix64, identical to oracle_random_bits().
template <typename T>
struct op_random
{
    static constexpr int nin = 0;
    static constexpr bool identity = false;
    std::uint64_t base;    // seed + k*STRIDE
    std::uint64_t first;
    __device__ T operator()(std::size_t idx, T, T) const
    {
        std::uint64_t x = mix64(base + (first + idx + 1) * kGolden);
        if constexpr (sizeof(T) == 8)
            return __dsub_rn(__dmul_rn(__dmul_rn(double(x >> 11), 0x1p-53), 2.0), 1.0);
        else
            return __fsub_rn(__fmul_rn(__fmul_rn(float(x >> 40), 0x1p-24f), 2.0f), 1.0f);
    }
};

template <typename T>
struct op_iota
{
    static constexpr int nin = 0;
    static constexpr bool identity = false;
    T first;
    __device__ T operator()(std::size_t idx, T, T) const { return first + T(idx); }
};

// ---------------------------------------------------------------------
// Tile chains: consecutive elementwise kernels on one stream whose tiles
// cover the same index ranges (STREAM's copy -> scale -> add -> triad ->
// copy ...) hand over tile by tile instead of at kernel boundaries.  The
// dependent kernel is launched with programmatic dependent launch, so its
// CTAs are scheduled while the predecessor's last wave drains; each CTA
// then waits only for the predecessor's *same* tile -- every op reads and
// writes index i only, so that tile carries all of its RAW/WAR/WAW
// dependencies, and earlier kernels are covered transitively.
//
// One flag per tile holds the chain position of the last kernel that
// finished it, plus one: kernel p waits (acquire, GPU scope) until its
// tile's flag reaches p, and stores p + 1 after the tile's stores
// (release, GPU scope).  Flags only grow within a chain, so any number of
// chained kernels may be resident at once (PDL lets kernel p+2 start while
// p is still running); the chain's end clears them in stream order
// (kernels.cu: chain state).
// ---------------------------------------------------------------------

constexpr unsigned kSpanLanes = 32;

__device__ __forceinline__ unsigned sm_count()
{
    unsigned n;
    asm volatile("mov.u32 %0, %%nsmid;" : "=r"(n));
    return n;
}

struct chain_args
{
    unsigned int* flags = nullptr;    // per-tile flags (nullptr: unchained)
    unsigned int pos = 0;             // position in the chain (0: head, waits for nothing)
    // In-kernel span (kernels.cu: coloc_cuda_span_begin): earliest CTA
    // start and latest CTA end (after its stores are performed), in
    // %globaltimer ns (32 ns resolution on B200), spread over
    // kSpanLanes slots each (min / max taken on the host); nullptr: not
    // recorded.
    unsigned long long* span_start = nullptr;
    unsigned long long* span_end = nullptr;
};

__device__ __forceinline__ std::uint64_t global_ns()
{
    std::uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Thread 0 waits for the predecessor's flag (acquire, GPU scope); the
// barrier then orders every thread's loads after the producer's stores.
// A flag that never arrives (a broken chain) traps after ~20 s instead of
// hanging the GPU.
__device__ __forceinline__ void chain_acquire(unsigned int const* flag, unsigned int pos)
{
    if (threadIdx.x == 0)
    {
        unsigned int v;
        std::uint64_t const t0 = global_ns();
        for (;;)
        {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
            if (v >= pos)
                break;
            __nanosleep(64);
            if (global_ns() - t0 > 20000000000ull)
                __trap();
        }
    }
    __syncthreads();
}

// Every thread's stores of the tile, then the flag (release, GPU scope:
// cumulative over the writes the barrier ordered before it).
__device__ __forceinline__ void chain_release(unsigned int* flag, unsigned int pos)
{
    __syncthreads();
    if (threadIdx.x == 0)
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(pos + 1) : "memory");
}

// ---------------------------------------------------------------------
// Kernels
// ---------------------------------------------------------------------

// U = 4 packs of two inputs need ~80 registers: those instantiations are
// limited to 512 threads per CTA so they never spill.
template <int U>
inline constexpr int kMaxPackThreads = U >= 4 ? 512 : 1024;

template <typename T, typename Op, int U, int Hint>
__global__ void __launch_bounds__(kMaxPackThreads<U>) ew_pack_kernel(Op op, T* dst,
    T const* s0, T const* s1, std::size_t head, std::size_t npacks,
    std::size_t tail, float l2_keep, chain_args chain)
{
    constexpr int E = kPackBytes / int(sizeof(T));
    // Programmatic dependent launch (launch.cuh, shape.pdl): wait until the
    // previous kernel on the stream has completed and its writes are
    // visible -- unless this kernel is a chained consumer, which waits per
    // tile instead -- then let the next one be scheduled.  Both are no-ops
    // for a normal launch.
    bool const chained = chain.flags != nullptr;
    bool const waits = chained && chain.pos > 0;
    if (!waits)
        asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // Only CTAs that can be first (the first wave) or last (the last
    // wave) stamp, over kSpanLanes addresses: one atomic per CTA on one
    // address slowed a 131072-CTA grid by 3-15% and a few-thousand-CTA
    // grid by microseconds (measured).  CTAs are dispatched in blockIdx
    // order, so the earliest start is among the first nsmid blocks and the
    // latest end among the last nsmid * (2048 / blockDim) blocks.
    if (chain.span_start && threadIdx.x == 0 && blockIdx.x < sm_count())
        atomicMin(chain.span_start + blockIdx.x % kSpanLanes, static_cast<unsigned long long>(global_ns()));
    std::uint64_t const pol = Hint == 5 ? l2_policy(l2_keep) : 0;
    std::size_t const tile = std::size_t(blockDim.x) * U;
    std::size_t const ntiles = (npacks + tile - 1) / tile;
    T* bd = dst + head;
    T const* b0 = Op::nin >= 1 ? s0 + head : nullptr;
    T const* b1 = Op::nin >= 2 ? s1 + head : nullptr;

    for (std::size_t t = blockIdx.x; t < ntiles; t += gridDim.x)
    {
        if (waits)
            chain_acquire(chain.flags + t, chain.pos);
        std::size_t const p0 = t * tile + threadIdx.x;
        bool const full = t * tile + tile <= npacks;
        pack<T> x[U], y[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
        {
            std::size_t const p = p0 + std::size_t(u) * blockDim.x;
            if (full || p < npacks)
            {
                if constexpr (Op::nin >= 1)
                    ld_pack<Hint>(b0 + p * E, x[u].w);
                if constexpr (Op::nin >= 2)
                    ld_pack<Hint>(b1 + p * E, y[u].w);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
        {
            std::size_t const p = p0 + std::size_t(u) * blockDim.x;
            if (full || p < npacks)
            {
                pack<T> o;
                if constexpr (Op::identity)
                {
                    o = x[u];
                }
                else
                {
#pragma unroll
                    for (int j = 0; j < E; ++j)
                        o.v[j] = op(head + p * E + std::size_t(j),
                            Op::nin >= 1 ? x[u].v[j] : T(),
                            Op::nin >= 2 ? y[u].v[j] : T());
                }
                st_pack<Hint>(bd + p * E, o.w, pol);
            }
        }
        if (chained)
            chain_release(chain.flags + t, chain.pos);
    }

    // Unaligned head and sub-pack tail: < 2*E elements, spread over the
    // threads of the last CTA (strided, so any CTA size covers them).
    // In a chain the head and tail are one more flag slot (index ntiles).
    if (blockIdx.x == gridDim.x - 1 && head + tail > 0)
    {
        if (waits)
            chain_acquire(chain.flags + ntiles, chain.pos);
        for (std::size_t r = threadIdx.x; r < head + tail; r += blockDim.x)
        {
            std::size_t const i = r < head ? r : head + npacks * E + (r - head);
            dst[i] = op(i, Op::nin >= 1 ? s0[i] : T(), Op::nin >= 2 ? s1[i] : T());
        }
        if (chained)
            chain_release(chain.flags + ntiles, chain.pos);
    }
    if (chain.span_end && std::size_t(blockIdx.x) + std::size_t(sm_count()) * (2048u / blockDim.x) >= gridDim.x)
    {
        __threadfence();    // this thread's stores are performed
        __syncthreads();
        if (threadIdx.x == 0)
            atomicMax(chain.span_end + blockIdx.x % kSpanLanes, static_cast<unsigned long long>(global_ns()));
    }
}

// Fallback when source and destination disagree on alignment modulo 32 B:
// element-granular, still coalesced.
template <typename T, typename Op>
__global__ void __launch_bounds__(256) ew_scalar_kernel(Op op, T* dst, T const* s0,
    T const* s1, std::size_t n)
{
    std::size_t const stride = std::size_t(gridDim.x) * blockDim.x;
    for (std::size_t i = std::size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += stride)
        dst[i] = op(i, Op::nin >= 1 ? s0[i] : T(), Op::nin >= 2 ? s1[i] : T());
}

}    // namespace coloc_cuda
