// kernels.cu -- C-ABI entry points for the elementwise hot path and the
// on-device construction kernels.  See include/coloc_cuda.h for the
// reference operation each entry point replaces.
#include "common.h"
#include "bulk.cuh"
#include "pipe.cuh"
#include "coloc_b200/kernels/launch.cuh"

#include <algorithm>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>

namespace coloc_cuda {

namespace {

// Process-wide tuning (coloc_cuda_set_tuning); 0 / -1 fields are automatic.
std::atomic<int> g_threads{0}, g_unroll{0}, g_ctas_per_sm{0}, g_hint{-1},
    g_exact{-1}, g_variant{0}, g_chunk{0}, g_stages{0}, g_schedule{0}, g_keep{0}, g_pdl{-1};

launch_shape current_shape(int nin, std::size_t range_bytes, std::size_t l2_bytes)
{
    launch_shape s;
    s.threads = g_threads.load(std::memory_order_relaxed);
    s.unroll = g_unroll.load(std::memory_order_relaxed);
    s.hint = g_hint.load(std::memory_order_relaxed);
    s.exact = g_exact.load(std::memory_order_relaxed);
    s.ctas_per_sm = g_ctas_per_sm.load(std::memory_order_relaxed);
    s.variant = g_variant.load(std::memory_order_relaxed);
    s.chunk_bytes = g_chunk.load(std::memory_order_relaxed);
    s.stages = g_stages.load(std::memory_order_relaxed);
    s.schedule = g_schedule.load(std::memory_order_relaxed);
    s.l2_keep_permille = g_keep.load(std::memory_order_relaxed);
    s.pdl = g_pdl.load(std::memory_order_relaxed);
    return resolve_shape(s, nin, range_bytes, l2_bytes);
}

// Lets one-time setup calls (cudaMalloc, cudaFuncSetAttribute) run while
// the calling thread is capturing a CUDA graph: they are not stream work
// and must not be captured, only permitted.
struct relaxed_capture_mode
{
    cudaStreamCaptureMode saved = cudaStreamCaptureModeRelaxed;
    relaxed_capture_mode() { (void) cudaThreadExchangeStreamCaptureMode(&saved); }
    ~relaxed_capture_mode() { (void) cudaThreadExchangeStreamCaptureMode(&saved); }
};

// Per-(device, stream) scheduler words of the TMA variant (zeroed once;
// the kernel's last CTA re-zeroes them for the next launch).
bulk_sched* sched_for(int dev, cudaStream_t stream)
{
    relaxed_capture_mode relaxed;
    static std::mutex mu;
    static std::unordered_map<std::uint64_t, bulk_sched*> slots;
    std::uint64_t const key = (std::uint64_t(dev) << 56) ^ reinterpret_cast<std::uintptr_t>(stream);
    std::lock_guard<std::mutex> lock(mu);
    auto it = slots.find(key);
    if (it != slots.end())
        return it->second;
    void* p = nullptr;
    if (cudaMalloc(&p, sizeof(bulk_sched)) != cudaSuccess ||
        cudaMemset(p, 0, sizeof(bulk_sched)) != cudaSuccess)
    {
        (void) cudaGetLastError();
        return nullptr;
    }
    slots[key] = static_cast<bulk_sched*>(p);
    return static_cast<bulk_sched*>(p);
}

template <typename T, typename Op>
int launch_bulk(int dev, cudaStream_t stream, Op op, T* dst, T const* s0, T const* s1,
    pack_split const& ps, launch_shape const& shape)
{
    auto fn = shape.hint >= 1 ? ew_bulk_kernel<T, Op, true> : ew_bulk_kernel<T, Op, false>;
    device_props const* p = props(dev);
    if (!p)
        return fail(COLOC_ERR_INVALID_TARGET, "cuda device " + std::to_string(dev));
    constexpr int nin = Op::nin > 0 ? Op::nin : 1;
    int const stages = std::clamp(shape.stages, Op::identity ? kCopyLag + 1 : 2, kMaxTmaStages);
    // both rings must fit in shared memory: clamp the chunk to 200 KB / buffers
    int const buffers = stages * nin + tma_out_stages<Op>();
    std::uint32_t const cap = std::uint32_t(200 * 1024 / buffers);
    std::uint32_t const chunk = std::min(std::uint32_t(shape.chunk_bytes), cap) & ~31u;
    std::size_t const smem = std::size_t(buffers) * chunk;
    if (chunk == 0)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "tuning.chunk_bytes out of range for the TMA variant");
    {
        relaxed_capture_mode relaxed;
        COLOC_TRY_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)),
            "cudaFuncSetAttribute");
    }
    bool const dynamic = shape.schedule == 2;
    bulk_sched* sched = nullptr;
    if (dynamic && !(sched = sched_for(dev, stream)))
        return fail(COLOC_ERR_ALLOCATION, "TMA scheduler words");
    // persistent grid: never more CTAs than fit at once (round-robin chunks
    // assume every CTA is resident)
    int occ = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kTmaThreads, smem) != cudaSuccess)
    {
        (void) cudaGetLastError();
        occ = 1;
    }
    occ = std::max(occ, 1);
    int const per_sm = shape.ctas_per_sm > 0 ? std::min(shape.ctas_per_sm, occ) : occ;
    std::size_t const body = ps.npacks * kPackBytes;
    std::size_t const nchunks = std::max<std::size_t>((body + chunk - 1) / chunk, 1);
    std::size_t const grid = std::min<std::size_t>(nchunks, std::size_t(per_sm) * p->sm_count);
    fn<<<unsigned(grid), kTmaThreads, smem, stream>>>(op, dst, s0, s1, ps.head, body, ps.tail,
        chunk, stages, dynamic ? 1 : 0, sched);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    COLOC_TRY_CUDA(cudaGetLastError(), "bulk kernel launch");
    return COLOC_OK;
}

template <typename T, typename Op, int U>
int launch_ldg_bulkst_u(cudaStream_t stream, Op op, T* dst, T const* s0, T const* s1,
    pack_split const& ps, int threads)
{
    auto fn = ew_ldg_bulkst_kernel<T, Op, U>;
    std::size_t const tile = std::size_t(threads) * U;
    std::size_t const smem = tile * kPackBytes;
    {
        relaxed_capture_mode relaxed;
        COLOC_TRY_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)),
            "cudaFuncSetAttribute");
    }
    std::size_t const grid = std::max<std::size_t>((ps.npacks + tile - 1) / tile, 1);
    if (grid > 0x7fffffffu)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "range too large for the hybrid variant");
    fn<<<unsigned(grid), threads, smem, stream>>>(op, dst, s0, s1, ps.head, ps.npacks, ps.tail);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    COLOC_TRY_CUDA(cudaGetLastError(), "hybrid kernel launch");
    return COLOC_OK;
}

template <typename T, typename Op>
int launch_ldg_bulkst(cudaStream_t stream, Op op, T* dst, T const* s0, T const* s1,
    pack_split const& ps, launch_shape const& shape)
{
    int const threads = std::min(shape.threads, 1024);
    if (shape.unroll >= 2)
        return launch_ldg_bulkst_u<T, Op, 2>(stream, op, dst, s0, s1, ps, threads);
    return launch_ldg_bulkst_u<T, Op, 1>(stream, op, dst, s0, s1, ps, threads);
}

template <typename T, typename Op, int U, bool Blocked>
int launch_pipe_u(cudaStream_t stream, int sm_count, Op op, T* dst, T const* s0, T const* s1,
    pack_split const& ps, launch_shape const& shape)
{
    auto fn = ew_pipe_kernel<T, Op, U, Blocked>;
    int const threads = std::min(shape.threads, 512);
    int occ = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, 0) != cudaSuccess)
    {
        (void) cudaGetLastError();
        occ = 1;
    }
    occ = std::max(occ, 1);
    int const per_sm = shape.ctas_per_sm > 0 ? std::min(shape.ctas_per_sm, occ) : occ;
    std::size_t const tile = std::size_t(threads) * U;
    std::size_t const ntiles = std::max<std::size_t>((ps.npacks + tile - 1) / tile, 1);
    std::size_t const grid = std::min<std::size_t>(ntiles, std::size_t(per_sm) * sm_count);
    fn<<<unsigned(grid), threads, 0, stream>>>(op, dst, s0, s1, ps.head, ps.npacks, ps.tail);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    COLOC_TRY_CUDA(cudaGetLastError(), "pipelined kernel launch");
    return COLOC_OK;
}

template <typename T, typename Op>
int launch_pipe(cudaStream_t stream, int sm_count, Op op, T* dst, T const* s0, T const* s1,
    pack_split const& ps, launch_shape const& shape)
{
    // shape.exact selects the tile order here: 1 blocked, 0 interleaved
    bool const blocked = shape.exact != 0;
    if (shape.unroll >= 2)
        return blocked ? launch_pipe_u<T, Op, 2, true>(stream, sm_count, op, dst, s0, s1, ps, shape)
                       : launch_pipe_u<T, Op, 2, false>(stream, sm_count, op, dst, s0, s1, ps, shape);
    return blocked ? launch_pipe_u<T, Op, 1, true>(stream, sm_count, op, dst, s0, s1, ps, shape)
                   : launch_pipe_u<T, Op, 1, false>(stream, sm_count, op, dst, s0, s1, ps, shape);
}

// ---------------------------------------------------------------------
// Tile chains (coloc_cuda_chain_begin/end; elementwise.cuh chain_args).
// Between begin and end, the elementwise launches on a stream form a
// chain: launch k > 0 is a programmatic dependent launch that waits per
// tile for launch k-1 (flag == k, set by launch k-1 as its position + 1).  All chained launches must split their ranges the
// same way (same byte geometry); a launch that cannot join (misaligned
// operands, a different geometry) breaks the chain: the flags are cleared
// in stream order and the next chainable launch starts a new chain.
// ---------------------------------------------------------------------

struct chain_geometry
{
    std::size_t head_bytes = 0, npacks = 0, tail_bytes = 0, tile = 0;
    bool operator==(chain_geometry const& o) const
    {
        return head_bytes == o.head_bytes && npacks == o.npacks && tail_bytes == o.tail_bytes &&
            tile == o.tile;
    }
};

struct chain_state
{
    bool active = false;
    std::size_t pos = 0;          // launches chained since the last (re)start
    chain_geometry geo;
    unsigned int* flags = nullptr;    // `cap` per-tile slots
    std::size_t cap = 0;
    std::size_t used = 0;         // slots that may be non-zero
};

std::mutex g_chain_mu;
std::atomic<int> g_open_chains{0};    // lets launches skip the chain lookup when none is open
std::unordered_map<std::uint64_t, chain_state>& chains()
{
    static std::unordered_map<std::uint64_t, chain_state> m;
    return m;
}

std::uint64_t chain_key(int dev, cudaStream_t stream)
{
    return (std::uint64_t(dev) << 56) ^ reinterpret_cast<std::uintptr_t>(stream);
}

// In-kernel spans (coloc_cuda_span_begin/read/end): per (device, stream)
// a device buffer of 2 u64 per launch, filled by the elementwise kernels.
struct span_state
{
    bool active = false;
    unsigned long long* slots = nullptr;    // starts[capacity], then ends[capacity]
    int capacity = 0;
    int used = 0;
};

std::mutex g_span_mu;
std::atomic<int> g_open_spans{0};
std::unordered_map<std::uint64_t, span_state>& spans()
{
    static std::unordered_map<std::uint64_t, span_state> m;
    return m;
}

}    // namespace

void chain_forget(int dev, void* stream)
{
    {
        std::lock_guard<std::mutex> lock(g_span_mu);
        auto it = spans().find(chain_key(dev, static_cast<cudaStream_t>(stream)));
        if (it != spans().end())
        {
            if (it->second.active)
                g_open_spans.fetch_sub(1, std::memory_order_release);
            // slots are not freed: a graph captured on the stream may outlive it
            spans().erase(it);
        }
    }
    std::lock_guard<std::mutex> lock(g_chain_mu);
    auto it = chains().find(chain_key(dev, static_cast<cudaStream_t>(stream)));
    if (it == chains().end())
        return;
    if (it->second.active)
        g_open_chains.fetch_sub(1, std::memory_order_release);
    chains().erase(it);
}

namespace {

// Clears the flags the chain may have set, ordered on the stream.
int chain_clear(chain_state& c, cudaStream_t stream)
{
    if (c.flags && c.used)
    {
        COLOC_TRY_CUDA(cudaMemsetAsync(c.flags, 0, c.used * sizeof(unsigned int), stream),
            "chain: cudaMemsetAsync");
    }
    c.pos = 0;
    c.used = 0;
    return COLOC_OK;
}

int chain_reserve(chain_state& c, std::size_t slots)
{
    if (slots <= c.cap)
        return COLOC_OK;
    // The old buffer may still be referenced by launches in flight: it is
    // kept (process lifetime) rather than freed.
    std::size_t const cap = std::max<std::size_t>(slots, 2 * c.cap);
    relaxed_capture_mode relaxed;
    void* p = nullptr;
    COLOC_TRY_CUDA(cudaMalloc(&p, cap * sizeof(unsigned int)), "chain: flag allocation");
    COLOC_TRY_CUDA(cudaMemset(p, 0, cap * sizeof(unsigned int)), "chain: flag init");
    c.flags = static_cast<unsigned int*>(p);
    c.cap = cap;
    c.pos = 0;
    c.used = 0;
    return COLOC_OK;
}

void span_slot(int dev, cudaStream_t stream, chain_args* args)
{
    if (g_open_spans.load(std::memory_order_acquire) == 0)
        return;
    std::lock_guard<std::mutex> lock(g_span_mu);
    auto it = spans().find(chain_key(dev, stream));
    if (it == spans().end() || !it->second.active || it->second.used >= it->second.capacity)
        return;
    span_state& st = it->second;
    args->span_start = st.slots + std::size_t(st.used) * kSpanLanes;
    args->span_end = st.slots + (std::size_t(st.capacity) + st.used) * kSpanLanes;
    ++st.used;
}

// Decides how a launch joins its stream's chain (if any): fills *args,
// or leaves them empty for a normal launch (breaking the chain first when
// one is running).  *shape is replaced by the chain's uniform tile shape.
template <typename T, typename Op>
int chain_join(int dev, cudaStream_t stream, T* dst, T const* s0, T const* s1, std::size_t n,
    std::size_t l2_bytes, launch_shape* shape, chain_args* args)
{
    if (g_open_chains.load(std::memory_order_acquire) == 0)
        return COLOC_OK;
    std::lock_guard<std::mutex> lock(g_chain_mu);
    auto it = chains().find(chain_key(dev, stream));
    if (it == chains().end() || !it->second.active)
        return COLOC_OK;
    chain_state& c = it->second;
    // One tile shape for every op of the chain.  Unless tuned, 256 x 2
    // packs: the per-tile flag wait costs one L2 round trip per CTA, which
    // several resident CTAs per SM hide (1024-thread CTAs, one per SM,
    // lose 6-9% to it at 256 MiB - 8 GiB; 256 x 2 chains run at or above
    // plain launches from 128 MiB up, profiles/r02_probe_chain_shapes.jsonl).
    launch_shape sh = current_shape(2, n * sizeof(T), l2_bytes);
    if (g_threads.load(std::memory_order_relaxed) <= 0)
        sh.threads = 256;
    if (g_unroll.load(std::memory_order_relaxed) <= 0 && n * sizeof(T) > (std::size_t(32) << 20))
        sh.unroll = 2;
    sh.variant = 1;
    pack_split const ps = split_range<T>(Op::nin, dst, s0, s1, n);
    if (!ps.aligned)
        return chain_clear(c, stream);    // runs unchained; the next launch starts over
    chain_geometry const g{ps.head * sizeof(T), ps.npacks, ps.tail * sizeof(T),
        std::size_t(sh.threads) * std::size_t(sh.unroll)};
    std::size_t const slots = (g.npacks + g.tile - 1) / g.tile + 1;
    if (c.pos > 0 && !(g == c.geo))
        COLOC_TRY(chain_clear(c, stream));
    COLOC_TRY(chain_reserve(c, slots));
    if (c.pos == 0)
        c.geo = g;
    args->flags = c.flags;
    args->pos = unsigned(c.pos);
    c.used = std::max(c.used, slots);
    ++c.pos;
    *shape = sh;
    return COLOC_OK;
}

// Runs op over [0, n) on `dev`/`stream` with the process tuning: the TMA
// variant when selected and the operands are pack-aligned, else the
// LDG/STG family (launch.cuh).
template <typename T, typename Op>
int run_elementwise(char const* what, int dev, void* stream_handle, Op op,
    T* dst, T const* s0, T const* s1, std::size_t n)
{
    if (n == 0)
        return COLOC_OK;
    if (!dst || (Op::nin >= 1 && !s0) || (Op::nin >= 2 && !s1))
        return fail(COLOC_ERR_INVALID_ARGUMENT, std::string(what) + ": null pointer");
    COLOC_TRY(use_device(dev));
    device_props const* p = props(dev);
    if (!p)
        return fail(COLOC_ERR_INVALID_TARGET, "cuda device " + std::to_string(dev));
    cudaStream_t stream = static_cast<cudaStream_t>(stream_handle);
    launch_shape shape = current_shape(Op::nin, n * sizeof(T), p->l2_bytes);
    chain_args chain;
    COLOC_TRY((chain_join<T, Op>(dev, stream, dst, s0, s1, n, p->l2_bytes, &shape, &chain)));
    span_slot(dev, stream, &chain);
    if (chain.span_start && !chain.flags)
    {
        // spans are recorded by the LDG/STG kernel family only
        shape.variant = 1;
    }
    if (chain.flags || chain.span_start)
    {
        cudaError_t const e = launch_elementwise<T, Op>(stream, p->sm_count, op, dst, s0, s1, n, shape, chain);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        COLOC_TRY_CUDA(e, what);
        return COLOC_OK;
    }
    if (shape.variant >= 2)
    {
        pack_split const ps = split_range<T>(Op::nin, dst, s0, s1, n);
        if (ps.aligned && shape.variant == 2)
            return launch_bulk<T, Op>(dev, stream, op, dst, s0, s1, ps, shape);
        if (ps.aligned && shape.variant == 3)
            return launch_ldg_bulkst<T, Op>(stream, op, dst, s0, s1, ps, shape);
        if (ps.aligned)
            return launch_pipe<T, Op>(stream, p->sm_count, op, dst, s0, s1, ps, shape);
    }
    cudaError_t const e = launch_elementwise<T, Op>(stream, p->sm_count, op, dst, s0, s1, n, shape);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    COLOC_TRY_CUDA(e, what);
    return COLOC_OK;
}

bool overlaps_partially(void const* a, void const* b, std::size_t bytes)
{
    auto pa = reinterpret_cast<std::uintptr_t>(a);
    auto pb = reinterpret_cast<std::uintptr_t>(b);
    return pa != pb && pa < pb + bytes && pb < pa + bytes;
}

template <typename T>
int check_overlap(char const* what, T const* dst, T const* src, std::size_t n)
{
    // algorithms.hpp:380-383 rejects overlapping copies; exact aliasing of
    // an elementwise transform (dst == src) is well defined and allowed.
    if (src && overlaps_partially(dst, src, n * sizeof(T)))
        return fail(COLOC_ERR_INVALID_ARGUMENT, std::string(what) + ": overlapping ranges");
    return COLOC_OK;
}

}    // namespace
}    // namespace coloc_cuda

using namespace coloc_cuda;

extern "C" {

int coloc_cuda_set_tuning(const coloc_cuda_tuning* t)
{
    if (!t)
    {
        g_threads = 0;
        g_unroll = 0;
        g_ctas_per_sm = 0;
        g_hint = -1;
        g_exact = -1;
        g_variant = 0;
        g_chunk = 0;
        g_stages = 0;
        g_schedule = 0;
        g_keep = 0;
        g_pdl = -1;
        return COLOC_OK;
    }
    if (t->threads != 0 &&
        (t->threads < 32 || t->threads > 1024 || t->threads % 32 != 0))
        return fail(COLOC_ERR_INVALID_ARGUMENT, "tuning.threads must be a multiple of 32 in [32,1024]");
    if (t->unroll != 0 && t->unroll != 1 && t->unroll != 2 && t->unroll != 4)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "tuning.unroll must be 0, 1, 2 or 4");
    if (t->cache_hint < -1 || t->cache_hint > 5)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "tuning.cache_hint must be in [-1, 5]");
    if (t->l2_keep_permille < 0 || t->l2_keep_permille > 1000)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "tuning.l2_keep_permille must be in [0, 1000]");
    if (t->variant < 0 || t->variant > 4)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "tuning.variant must be in [0, 4]");
    if (t->stages < 0 || t->stages > kMaxTmaStages)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "tuning.stages must be in [0, 8]");
    if (t->schedule < 0 || t->schedule > 2)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "tuning.schedule must be 0, 1 or 2");
    if (t->pdl < -1 || t->pdl > 1)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "tuning.pdl must be -1, 0 or 1");
    g_threads = t->threads;
    g_unroll = t->unroll;
    g_ctas_per_sm = t->ctas_per_sm;
    g_hint = t->cache_hint;
    g_exact = t->exact_grid;
    g_variant = t->variant;
    g_chunk = t->chunk_bytes;
    g_stages = t->stages;
    g_schedule = t->schedule;
    g_keep = t->l2_keep_permille;
    g_pdl = t->pdl;
    return COLOC_OK;
}

int coloc_cuda_get_tuning(coloc_cuda_tuning* t)
{
    if (!t)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "get_tuning: null out");
    t->threads = g_threads;
    t->unroll = g_unroll;
    t->ctas_per_sm = g_ctas_per_sm;
    t->cache_hint = g_hint;
    t->exact_grid = g_exact;
    t->variant = g_variant;
    t->chunk_bytes = g_chunk;
    t->stages = g_stages;
    t->schedule = g_schedule;
    t->l2_keep_permille = g_keep;
    t->pdl = g_pdl;
    return COLOC_OK;
}

int coloc_cuda_chain_begin(int dev, void* stream)
{
    COLOC_TRY(use_device(dev));
    auto* s = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lock(g_chain_mu);
    chain_state& c = chains()[chain_key(dev, s)];
    if (c.active)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "chain_begin: a chain is already open on this stream");
    c.active = true;
    c.pos = 0;
    g_open_chains.fetch_add(1, std::memory_order_release);
    return COLOC_OK;
}

int coloc_cuda_chain_end(int dev, void* stream)
{
    COLOC_TRY(use_device(dev));
    auto* s = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lock(g_chain_mu);
    auto it = chains().find(chain_key(dev, s));
    if (it == chains().end() || !it->second.active)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "chain_end: no chain open on this stream");
    it->second.active = false;
    g_open_chains.fetch_sub(1, std::memory_order_release);
    // the last launch's signals are cleared behind it, so the next chain
    // (or the next replay of a captured graph) starts from zero flags
    return chain_clear(it->second, s);
}

int coloc_cuda_span_begin(int dev, void* stream, int capacity)
{
    if (capacity <= 0)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "span_begin: capacity must be positive");
    COLOC_TRY(use_device(dev));
    auto* s = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lock(g_span_mu);
    span_state& st = spans()[chain_key(dev, s)];
    if (st.active)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "span_begin: already recording on this stream");
    if (st.capacity < capacity)
    {
        // a smaller buffer may still be referenced by launches in flight or
        // by captured graphs: it is kept (process lifetime), not freed
        relaxed_capture_mode relaxed;
        st.slots = nullptr;
        st.capacity = 0;
        void* p = nullptr;
        COLOC_TRY_CUDA(cudaMalloc(&p, 2 * kSpanLanes * sizeof(unsigned long long) * std::size_t(capacity)),
            "span: slot allocation");    // starts, then ends, kSpanLanes each
        st.slots = static_cast<unsigned long long*>(p);
        st.capacity = capacity;
    }
    // earliest starts = all ones, latest ends = 0, in stream order
    std::size_t const lanes = kSpanLanes * std::size_t(capacity);
    COLOC_TRY_CUDA(cudaMemsetAsync(st.slots, 0xff, sizeof(unsigned long long) * lanes, s), "span: init");
    COLOC_TRY_CUDA(cudaMemsetAsync(st.slots + std::size_t(st.capacity) * kSpanLanes, 0,
                       sizeof(unsigned long long) * lanes, s),
        "span: init");
    st.active = true;
    st.used = 0;
    g_open_spans.fetch_add(1, std::memory_order_release);
    return COLOC_OK;
}

int coloc_cuda_span_end(int dev, void* stream, int* count)
{
    COLOC_TRY(use_device(dev));
    auto* s = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lock(g_span_mu);
    auto it = spans().find(chain_key(dev, s));
    if (it == spans().end() || !it->second.active)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "span_end: not recording on this stream");
    it->second.active = false;
    g_open_spans.fetch_sub(1, std::memory_order_release);
    if (count)
        *count = it->second.used;
    return COLOC_OK;
}

int coloc_cuda_span_read(int dev, void* stream, double* ms, int count)
{
    if (count < 0 || (count > 0 && !ms))
        return fail(COLOC_ERR_INVALID_ARGUMENT, "span_read: bad arguments");
    COLOC_TRY(use_device(dev));
    auto* s = static_cast<cudaStream_t>(stream);
    unsigned long long* slots = nullptr;
    int cap = 0;
    {
        std::lock_guard<std::mutex> lock(g_span_mu);
        auto it = spans().find(chain_key(dev, s));
        if (it == spans().end() || it->second.active || count > it->second.used)
            return fail(COLOC_ERR_INVALID_ARGUMENT, "span_read: end the recording first; count <= recorded");
        slots = it->second.slots;
        cap = it->second.capacity;
    }
    std::size_t const lanes = kSpanLanes * static_cast<std::size_t>(count);
    std::vector<unsigned long long> a(lanes), b(lanes);
    if (count)
    {
        COLOC_TRY_CUDA(cudaMemcpyAsync(a.data(), slots, lanes * sizeof(a[0]), cudaMemcpyDeviceToHost, s),
            "span_read: copy");
        COLOC_TRY_CUDA(cudaMemcpyAsync(b.data(), slots + std::size_t(cap) * kSpanLanes, lanes * sizeof(b[0]),
                           cudaMemcpyDeviceToHost, s),
            "span_read: copy");
        COLOC_TRY_CUDA(cudaStreamSynchronize(s), "span_read: sync");
    }
    for (int i = 0; i < count; ++i)
    {
        auto const lo = a.begin() + std::ptrdiff_t(i) * kSpanLanes;
        auto const hi = b.begin() + std::ptrdiff_t(i) * kSpanLanes;
        unsigned long long const start = *std::min_element(lo, lo + kSpanLanes);
        unsigned long long const end = *std::max_element(hi, hi + kSpanLanes);
        ms[i] = end >= start ? double(end - start) * 1e-6 : 0.0;
    }
    return COLOC_OK;
}

int coloc_cuda_chain_break(int dev, void* stream)
{
    if (g_open_chains.load(std::memory_order_acquire) == 0)
        return COLOC_OK;
    COLOC_TRY(use_device(dev));
    auto* s = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lock(g_chain_mu);
    auto it = chains().find(chain_key(dev, s));
    if (it == chains().end() || !it->second.active || it->second.pos == 0)
        return COLOC_OK;
    return chain_clear(it->second, s);
}

int coloc_cuda_copy_bytes(int dev, void* stream, void* dst, const void* src,
    size_t bytes)
{
    if (bytes == 0)
        return COLOC_OK;
    COLOC_TRY(check_overlap("copy", static_cast<unsigned char const*>(dst),
        static_cast<unsigned char const*>(src), bytes));
    if (dst == src)
        return COLOC_OK;
    auto* d = static_cast<unsigned char*>(dst);
    auto const* s = static_cast<unsigned char const*>(src);
    // Wider element granularity on the misaligned fallback when possible.
    auto mis = [](void const* q) { return reinterpret_cast<std::uintptr_t>(q) % kPackBytes; };
    if (mis(d) != mis(s) && reinterpret_cast<std::uintptr_t>(d) % 8 == 0 &&
        reinterpret_cast<std::uintptr_t>(s) % 8 == 0 && bytes % 8 == 0)
        return run_elementwise<std::uint64_t>("copy", dev, stream, op_copy{},
            reinterpret_cast<std::uint64_t*>(d), reinterpret_cast<std::uint64_t const*>(s),
            nullptr, bytes / 8);
    return run_elementwise<unsigned char>("copy", dev, stream, op_copy{}, d, s, nullptr, bytes);
}

int coloc_cuda_copy_f64(int dev, void* stream, double* dst, const double* src,
    size_t n)
{
    return coloc_cuda_copy_bytes(dev, stream, dst, src, n * sizeof(double));
}

int coloc_cuda_copy_f32(int dev, void* stream, float* dst, const float* src,
    size_t n)
{
    return coloc_cuda_copy_bytes(dev, stream, dst, src, n * sizeof(float));
}

int coloc_cuda_scale_f64(int dev, void* stream, double* dst, const double* src,
    double s, size_t n)
{
    COLOC_TRY(check_overlap("scale", dst, src, n));
    return run_elementwise<double>("scale", dev, stream, op_scale<double>{s}, dst, src, nullptr, n);
}

int coloc_cuda_scale_f32(int dev, void* stream, float* dst, const float* src,
    float s, size_t n)
{
    COLOC_TRY(check_overlap("scale", dst, src, n));
    return run_elementwise<float>("scale", dev, stream, op_scale<float>{s}, dst, src, nullptr, n);
}

int coloc_cuda_add_f64(int dev, void* stream, double* dst, const double* a,
    const double* b, size_t n)
{
    COLOC_TRY(check_overlap("add", dst, a, n));
    COLOC_TRY(check_overlap("add", dst, b, n));
    return run_elementwise<double>("add", dev, stream, op_add<double>{}, dst, a, b, n);
}

int coloc_cuda_add_f32(int dev, void* stream, float* dst, const float* a,
    const float* b, size_t n)
{
    COLOC_TRY(check_overlap("add", dst, a, n));
    COLOC_TRY(check_overlap("add", dst, b, n));
    return run_elementwise<float>("add", dev, stream, op_add<float>{}, dst, a, b, n);
}

int coloc_cuda_triad_f64(int dev, void* stream, double* dst, const double* b,
    const double* c, double s, size_t n, int fma)
{
    COLOC_TRY(check_overlap("triad", dst, b, n));
    COLOC_TRY(check_overlap("triad", dst, c, n));
    if (fma)
        return run_elementwise<double>("triad", dev, stream, op_triad<double, true>{s}, dst, b, c, n);
    return run_elementwise<double>("triad", dev, stream, op_triad<double, false>{s}, dst, b, c, n);
}

int coloc_cuda_triad_f32(int dev, void* stream, float* dst, const float* b,
    const float* c, float s, size_t n, int fma)
{
    COLOC_TRY(check_overlap("triad", dst, b, n));
    COLOC_TRY(check_overlap("triad", dst, c, n));
    if (fma)
        return run_elementwise<float>("triad", dev, stream, op_triad<float, true>{s}, dst, b, c, n);
    return run_elementwise<float>("triad", dev, stream, op_triad<float, false>{s}, dst, b, c, n);
}

int coloc_cuda_scale_i32(int dev, void* stream, int32_t* dst, const int32_t* src,
    int32_t s, size_t n)
{
    COLOC_TRY(check_overlap("scale", dst, src, n));
    return run_elementwise<std::int32_t>("scale", dev, stream, op_scale<std::int32_t>{s}, dst, src, nullptr, n);
}

int coloc_cuda_scale_i64(int dev, void* stream, int64_t* dst, const int64_t* src,
    int64_t s, size_t n)
{
    COLOC_TRY(check_overlap("scale", dst, src, n));
    return run_elementwise<std::int64_t>("scale", dev, stream, op_scale<std::int64_t>{s}, dst, src, nullptr, n);
}

int coloc_cuda_add_i32(int dev, void* stream, int32_t* dst, const int32_t* a,
    const int32_t* b, size_t n)
{
    COLOC_TRY(check_overlap("add", dst, a, n));
    COLOC_TRY(check_overlap("add", dst, b, n));
    return run_elementwise<std::int32_t>("add", dev, stream, op_add<std::int32_t>{}, dst, a, b, n);
}

int coloc_cuda_add_i64(int dev, void* stream, int64_t* dst, const int64_t* a,
    const int64_t* b, size_t n)
{
    COLOC_TRY(check_overlap("add", dst, a, n));
    COLOC_TRY(check_overlap("add", dst, b, n));
    return run_elementwise<std::int64_t>("add", dev, stream, op_add<std::int64_t>{}, dst, a, b, n);
}

int coloc_cuda_triad_i32(int dev, void* stream, int32_t* dst, const int32_t* b,
    const int32_t* c, int32_t s, size_t n)
{
    COLOC_TRY(check_overlap("triad", dst, b, n));
    COLOC_TRY(check_overlap("triad", dst, c, n));
    return run_elementwise<std::int32_t>("triad", dev, stream, op_triad<std::int32_t, false>{s}, dst, b, c, n);
}

int coloc_cuda_triad_i64(int dev, void* stream, int64_t* dst, const int64_t* b,
    const int64_t* c, int64_t s, size_t n)
{
    COLOC_TRY(check_overlap("triad", dst, b, n));
    COLOC_TRY(check_overlap("triad", dst, c, n));
    return run_elementwise<std::int64_t>("triad", dev, stream, op_triad<std::int64_t, false>{s}, dst, b, c, n);
}

int coloc_cuda_to_upper_u8(int dev, void* stream, unsigned char* dst,
    const unsigned char* src, size_t n)
{
    COLOC_TRY(check_overlap("to_upper", dst, src, n));
    return run_elementwise<unsigned char>("to_upper", dev, stream, op_to_upper{}, dst, src, nullptr, n);
}

int coloc_cuda_fill(int dev, void* stream, void* dst, size_t n,
    const void* value, size_t elem_size)
{
    if (n == 0)
        return COLOC_OK;
    if (!value)
        return fail(COLOC_ERR_INVALID_ARGUMENT, "fill: null value");
    switch (elem_size)
    {
    case 1: {
        unsigned char v;
        std::memcpy(&v, value, 1);
        return run_elementwise<unsigned char>("fill", dev, stream, op_fill<unsigned char>{v},
            static_cast<unsigned char*>(dst), nullptr, nullptr, n);
    }
    case 2: {
        std::uint16_t v;
        std::memcpy(&v, value, 2);
        return run_elementwise<std::uint16_t>("fill", dev, stream, op_fill<std::uint16_t>{v},
            static_cast<std::uint16_t*>(dst), nullptr, nullptr, n);
    }
    case 4: {
        std::uint32_t v;
        std::memcpy(&v, value, 4);
        return run_elementwise<std::uint32_t>("fill", dev, stream, op_fill<std::uint32_t>{v},
            static_cast<std::uint32_t*>(dst), nullptr, nullptr, n);
    }
    case 8: {
        std::uint64_t v;
        std::memcpy(&v, value, 8);
        return run_elementwise<std::uint64_t>("fill", dev, stream, op_fill<std::uint64_t>{v},
            static_cast<std::uint64_t*>(dst), nullptr, nullptr, n);
    }
    case 16:
    case 32: {
        // Wider patterns: fill 8-byte lanes with the pattern repeating.
        // Only valid when the pattern is uniform across its 8-byte words.
        std::uint64_t w[4];
        std::memcpy(w, value, elem_size);
        for (std::size_t j = 1; j < elem_size / 8; ++j)
            if (w[j] != w[0])
                return fail(COLOC_ERR_UNSUPPORTED, "fill: non-uniform wide pattern");
        return run_elementwise<std::uint64_t>("fill", dev, stream, op_fill<std::uint64_t>{w[0]},
            static_cast<std::uint64_t*>(dst), nullptr, nullptr, n * (elem_size / 8));
    }
    default:
        return fail(COLOC_ERR_INVALID_ARGUMENT,
            "fill: unsupported element size " + std::to_string(elem_size));
    }
}

int coloc_cuda_fill_f64(int dev, void* stream, double* dst, size_t n, double v)
{
    return run_elementwise<double>("fill", dev, stream, op_fill<double>{v}, dst, nullptr, nullptr, n);
}

int coloc_cuda_fill_f32(int dev, void* stream, float* dst, size_t n, float v)
{
    return run_elementwise<float>("fill", dev, stream, op_fill<float>{v}, dst, nullptr, nullptr, n);
}

int coloc_cuda_generate_random_f64(int dev, void* stream, double* dst,
    size_t n, uint64_t seed, uint32_t k, uint64_t first)
{
    op_random<double> op{seed + std::uint64_t(k) * kArrayStride, first};
    return run_elementwise<double>("generate_random", dev, stream, op, dst, nullptr, nullptr, n);
}

int coloc_cuda_generate_random_f32(int dev, void* stream, float* dst,
    size_t n, uint64_t seed, uint32_t k, uint64_t first)
{
    op_random<float> op{seed + std::uint64_t(k) * kArrayStride, first};
    return run_elementwise<float>("generate_random", dev, stream, op, dst, nullptr, nullptr, n);
}

int coloc_cuda_iota_f64(int dev, void* stream, double* dst, size_t n,
    double first)
{
    return run_elementwise<double>("iota", dev, stream, op_iota<double>{first}, dst, nullptr, nullptr, n);
}

}    // extern "C"
