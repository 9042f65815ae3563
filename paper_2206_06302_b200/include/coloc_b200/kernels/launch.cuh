// launch.cuh -- host-side launch of the elementwise kernel family.
//
// Header-only so that two kinds of translation units share one launch
// policy: libcoloc_cuda.so (the named STREAM ops behind the C ABI) and user
// code compiled by nvcc that passes its own __device__ lambdas or functors
// to coloc::transform / coloc::for_each (device_lambda.cuh).
//
// A range [0, n) is split into an unaligned head (< 32 B), a body of 32-byte
// packs and a tail; the body runs on ew_pack_kernel when every operand shares
// the destination's alignment modulo 32 B, otherwise the element kernel
// ew_scalar_kernel runs the whole range.
#pragma once

#include "coloc_b200/kernels/elementwise.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstddef>
#include <cstdint>

namespace coloc_cuda {

struct launch_shape
{
    int threads = 0;        // threads per CTA; 0 = automatic
    int unroll = 0;         // packs per thread per input: 1, 2, 4; 0 = automatic
    int hint = -1;          // 0 plain, 1 streaming, 2 = 1 + L2 prefetch, 3/4 evict-last stores; -1 auto
    int exact = -1;         // 1 one tile per CTA, 0 persistent grid stride; -1 auto
    int ctas_per_sm = 0;    // persistent grid: CTAs per SM; 0 = occupancy
    int variant = 0;        // 1 LDG/STG packs, 2 TMA bulk (library ops only); 0 auto
    int chunk_bytes = 0;    // TMA variant chunk per input; 0 auto
    int stages = 0;         // TMA variant input-ring depth; 0 auto
    int schedule = 0;       // TMA variant chunk claiming: 1 round robin, 2 atomic; 0 auto
    int l2_keep_permille = 0;    // hint 5: share of output lines kept in L2; 0 auto
    int pdl = -1;           // programmatic dependent launch: 1 on, 0 off, -1 auto
};

// Measured on B200 (profiles/r01_tune*.jsonl):
//   - one tile per CTA beats a persistent grid-stride grid by ~7% at 8 GiB
//     per array: CTAs retire and get replaced in address order, so the DRAM
//     working set stays compact (profiles/r01_tune_c2_persistent_vs_exact.jsonl);
//   - >= 256 MiB per array: 1024 threads x 1 pack for one-input ops
//     (copy/scale 7.09 TB/s), 1024 x 2 for two-input ops (add/triad
//     7.17 TB/s vs 7.14 at x1); smaller ranges: 256 threads x 2 packs,
//     x 1 at <= 32 MiB.
//   - the TMA variant (bulk.cuh) is never the automatic choice: its best
//     shape (3 CTAs per SM, 2-deep ring of 8 KB chunks per input, atomic
//     chunk claiming, evict-first bulk copies) reached 7.25 TB/s for
//     add/triad on some boxes and 7.06-7.10 on others, while LDG/STG held
//     7.16-7.18 on every box; copy/scale lose 1-30% on TMA.  Over a whole
//     STREAM iteration LDG/STG won every interleaved A/B
//     (profiles/r01_tune_tma_c{2,3}.jsonl, r01_ab_*.jsonl).
//   - cache hint by destination size D against the L2 size L (133 MB on
//     B200), from whole-iteration rates of interleaved A/B rounds
//     (profiles/r01_ab_hints_*.jsonl):
//       3 D <= 0.6 L   plain loads/stores: the three arrays stay in L2
//                      (24 MiB/array: +6-10% over streaming hints);
//       D <= 0.65 L    streaming loads, evict-last stores: a kernel's output
//                      is still in L2 when the next kernel of a chain reads
//                      it (STREAM at 32-80 MiB/array: +4% to +20%; C1's
//                      80 MB arrays: +20%);
//       D <= 0.95 L    streaming loads, evict-last stores for ~0.6 L worth
//                      of the output, evict-first for the rest (96 MiB:
//                      +11%, 112 MiB: +5-8%; evict-last for all of it
//                      loses 3% at 112 MiB);
//       larger         streaming loads and stores (evict-last loses 4-6%
//                      at 128 MiB and ~0.5% at 1-8 GiB; any share kept
//                      through a cache policy loses 0-6% from 128 MiB to
//                      8 GiB).
inline int auto_hint(std::size_t range_bytes, std::size_t l2_bytes)
{
    if (l2_bytes == 0)
        return 1;
    if (10 * 3 * range_bytes <= 6 * l2_bytes)
        return 0;
    if (20 * range_bytes <= 13 * l2_bytes)
        return 3;
    if (20 * range_bytes <= 19 * l2_bytes)
        return 5;
    return 1;
}

inline launch_shape resolve_shape(launch_shape s, int nin, std::size_t range_bytes,
    std::size_t l2_bytes = 0)
{
    bool const large = range_bytes >= (std::size_t(256) << 20);
    if (s.exact < 0)
        s.exact = 1;
    if (s.threads <= 0)
        s.threads = large ? 1024 : 256;
    // <= 32 MiB: 8 KB tiles (256 x 1) so even a one-wave range spreads
    // evenly over the SMs (16 MiB add/triad: +20% over 16 KB tiles,
    // profiles/r01_ab_small_tiles_c2.jsonl)
    bool const small = range_bytes <= (std::size_t(32) << 20);
    if (s.unroll <= 0)
        s.unroll = (large && nin < 2) || small ? 1 : 2;
    if (s.hint < 0)
        s.hint = auto_hint(range_bytes, l2_bytes);
    if (s.l2_keep_permille <= 0)
    {
        // keep ~60% of L2 worth of the output (the measured sweet spot of
        // hint 3 is an output of 0.6-0.8 L2)
        double const keep = range_bytes ? 0.6 * double(l2_bytes) / double(range_bytes) : 1.0;
        s.l2_keep_permille = int(std::clamp(keep, 1.0 / 16, 1.0) * 1000.0);
    }
    s.l2_keep_permille = std::min(s.l2_keep_permille, 1000);
    if (s.variant <= 0)
        s.variant = 1;
    if (s.unroll >= 4)
        s.threads = std::min(s.threads, kMaxPackThreads<4>);
    if (s.variant == 2)
    {
        if (s.chunk_bytes <= 0)
            s.chunk_bytes = 8192;
        if (s.stages <= 0)
            s.stages = 2;
        if (s.ctas_per_sm <= 0)
            s.ctas_per_sm = 3;
    }
    if (s.schedule <= 0)
        s.schedule = 2;
    if (s.pdl < 0)
        s.pdl = 0;
    return s;
}

// Resident CTAs per SM of one kernel instantiation at a block size.
template <typename Kernel>
int occupancy_of(Kernel fn, int threads)
{
    static std::atomic<int> cache[33];    // indexed by threads / 32
    int const slot = std::clamp(threads / 32, 0, 32);
    int v = cache[slot].load(std::memory_order_relaxed);
    if (v > 0)
        return v;
    int blocks = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, threads, 0) != cudaSuccess)
    {
        (void) cudaGetLastError();
        blocks = 1;
    }
    blocks = std::max(blocks, 1);
    cache[slot].store(blocks, std::memory_order_relaxed);
    return blocks;
}

template <typename T, typename Op, int U, int Hint>
cudaError_t launch_pack(cudaStream_t stream, int sm_count, Op const& op, T* dst, T const* s0,
    T const* s1, std::size_t head, std::size_t npacks, std::size_t tail, launch_shape const& shape,
    chain_args chain)
{
    auto fn = ew_pack_kernel<T, Op, U, Hint>;
    std::size_t const tile = std::size_t(shape.threads) * U;
    std::size_t const ntiles = std::max<std::size_t>((npacks + tile - 1) / tile, 1);
    std::size_t grid = ntiles;
    if (!shape.exact)
    {
        int const per_sm = shape.ctas_per_sm > 0 ? shape.ctas_per_sm : occupancy_of(fn, shape.threads);
        grid = std::min<std::size_t>(ntiles, std::size_t(per_sm) * std::size_t(sm_count));
    }
    grid = std::min<std::size_t>(grid, 0x7fffffffu);
    float const keep = float(shape.l2_keep_permille) / 1000.0f;
    if (shape.pdl > 0 || (chain.flags && chain.pos > 0))
    {
        // Programmatic dependent launch: this grid may be scheduled while
        // its predecessor on the stream drains its last wave (the
        // predecessor's CTAs signal griddepcontrol.launch_dependents on
        // entry); every CTA waits in griddepcontrol.wait until the
        // predecessor has completed and its writes are visible, so only
        // the launch latency overlaps, never the data.
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(unsigned(grid));
        cfg.blockDim = dim3(unsigned(shape.threads));
        cfg.dynamicSmemBytes = 0;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, fn, op, dst, s0, s1, head, npacks, tail, keep, chain);
    }
    fn<<<dim3(unsigned(grid)), dim3(unsigned(shape.threads)), 0, stream>>>(
        op, dst, s0, s1, head, npacks, tail, keep, chain);
    return cudaGetLastError();
}

template <typename T, typename Op, int U>
cudaError_t launch_pack_hint(cudaStream_t stream, int sm_count, Op const& op, T* dst, T const* s0,
    T const* s1, std::size_t head, std::size_t npacks, std::size_t tail, launch_shape const& shape,
    chain_args chain)
{
    switch (shape.hint)
    {
    case 1:
        return launch_pack<T, Op, U, 1>(stream, sm_count, op, dst, s0, s1, head, npacks, tail, shape, chain);
    case 2:
        return launch_pack<T, Op, U, 2>(stream, sm_count, op, dst, s0, s1, head, npacks, tail, shape, chain);
    case 3:
        return launch_pack<T, Op, U, 3>(stream, sm_count, op, dst, s0, s1, head, npacks, tail, shape, chain);
    case 4:
        return launch_pack<T, Op, U, 4>(stream, sm_count, op, dst, s0, s1, head, npacks, tail, shape, chain);
    case 5:
        return launch_pack<T, Op, U, 5>(stream, sm_count, op, dst, s0, s1, head, npacks, tail, shape, chain);
    default:
        return launch_pack<T, Op, U, 0>(stream, sm_count, op, dst, s0, s1, head, npacks, tail, shape, chain);
    }
}

// Pack decomposition of [0, n) for the operands of an op with `nin` inputs.
struct pack_split
{
    bool aligned;
    std::size_t head, npacks, tail;
};

template <typename T>
pack_split split_range(int nin, T const* dst, T const* s0, T const* s1, std::size_t n)
{
    auto mis = [](void const* q) { return reinterpret_cast<std::uintptr_t>(q) % kPackBytes; };
    std::uintptr_t const md = mis(dst);
    bool aligned = md % sizeof(T) == 0;
    if (nin >= 1)
        aligned = aligned && mis(s0) == md;
    if (nin >= 2)
        aligned = aligned && mis(s1) == md;
    pack_split p{aligned, 0, 0, 0};
    if (!aligned)
        return p;
    constexpr std::size_t E = kPackBytes / sizeof(T);
    p.head = std::min<std::size_t>(md == 0 ? 0 : (kPackBytes - md) / sizeof(T), n);
    p.npacks = (n - p.head) / E;
    p.tail = n - p.head - p.npacks * E;
    return p;
}

// op over [0, n) with the LDG/STG kernel family.  `shape` must be resolved.
// Returns the launch status; n == 0 launches nothing.
// `chain` (kernels.cu) links this launch into a tile chain; only valid
// for aligned ranges (the caller checks split_range first).
template <typename T, typename Op>
cudaError_t launch_elementwise(cudaStream_t stream, int sm_count, Op const& op, T* dst,
    T const* s0, T const* s1, std::size_t n, launch_shape const& shape, chain_args chain = {})
{
    if (n == 0)
        return cudaSuccess;
    pack_split const p = split_range<T>(Op::nin, dst, s0, s1, n);
    if (!p.aligned)
    {
        std::size_t const grid = std::min<std::size_t>((n + 255) / 256, std::size_t(sm_count) * 8);
        ew_scalar_kernel<T, Op><<<unsigned(grid), 256, 0, stream>>>(op, dst, s0, s1, n);
        return cudaGetLastError();
    }
    switch (shape.unroll)
    {
    case 1:
        return launch_pack_hint<T, Op, 1>(stream, sm_count, op, dst, s0, s1, p.head, p.npacks, p.tail, shape, chain);
    case 2:
        return launch_pack_hint<T, Op, 2>(stream, sm_count, op, dst, s0, s1, p.head, p.npacks, p.tail, shape, chain);
    case 4:
        return launch_pack_hint<T, Op, 4>(stream, sm_count, op, dst, s0, s1, p.head, p.npacks, p.tail, shape, chain);
    default:
        return cudaErrorInvalidValue;
    }
}

}    // namespace coloc_cuda
