// SPDX-License-Identifier: Apache-2.0
// Restates the public interface of the reference coloc library's algorithms.hpp
// (arXiv 2206.06302; /root/reference/proj/include/coloc, Apache-2.0): the
// names, signatures and semantics are kept for drop-in compatibility.
// parallel.hpp -- execution policies and the parallel algorithms (copy,
// transform, for_each) over GPU-resident coloc::vectors.
//
// Mirrors include/coloc/algorithms.hpp:
//   seq / par / .on(exec)              33-86
//   policy_info, iter_info             90-149
//   algorithm_shape                    210-234  (one range per destination block
//                                                here: a GPU block is one launch,
//                                                not 4 x workers host chunks)
//   with_default_executor              257-280  (the vexing parse at 277 does not
//                                                exist here)
//   copy                               359-444
//   transform (unary / binary)         452-526
// for_each is the north star's third algorithm; the reference has none.
//
// Dispatch is decided at compile time from the iterators' memory space:
//   device -> device : kernel launches through the policy's CUDA executor,
//                      one per (destination block x source segment piece)
//   host  <-> device : staged copies (cudaMemcpyAsync) per destination/source
//                      block, completed before returning (the caller owns the
//                      host buffer), algorithms.hpp:388-407
//   device -> other device : cudaMemcpyPeerAsync over NVLink instead of the
//                      reference's host bounce buffer (algorithms.hpp:420-436)
// Anything involving only host memory is not this library's business and
// does not compile; there is no CPU fallback.
#pragma once

#include "coloc_b200/container.hpp"
#include "coloc_b200/executors.hpp"
#include "coloc_b200/memory.hpp"
#include "coloc_b200/ops.hpp"
#include "coloc_b200/schedule_log.hpp"

#include <algorithm>
#include <array>
#include <cstddef>
#include <iterator>
#include <memory>
#include <mutex>
#include <set>
#include <stdexcept>
#include <type_traits>
#include <utility>
#include <vector>

#if defined(__CUDACC__)
// loops over the NSrc sources are empty for NSrc == 0 (for_each)
#pragma nv_diag_suppress 186
#endif

namespace coloc {

// ---------------------------------------------------------------------
// Execution policies (algorithms.hpp:33-86)
// ---------------------------------------------------------------------

template <typename Executor>
struct parallel_executor_policy;
template <typename Executor>
struct sequenced_executor_policy;

struct sequenced_policy
{
    template <typename Executor>
    sequenced_executor_policy<Executor> on(Executor& exec) const noexcept
    {
        return {&exec};
    }
};

struct parallel_policy
{
    template <typename Executor>
    parallel_executor_policy<Executor> on(Executor& exec) const noexcept
    {
        return {&exec};
    }
};

template <typename Executor>
struct parallel_executor_policy
{
    Executor* exec;
    template <typename E2>
    parallel_executor_policy<E2> on(E2& next) const noexcept
    {
        return {&next};
    }
    Executor& executor() const noexcept { return *exec; }
};

template <typename Executor>
struct sequenced_executor_policy
{
    Executor* exec;
    template <typename E2>
    sequenced_executor_policy<E2> on(E2& next) const noexcept
    {
        return {&next};
    }
    Executor& executor() const noexcept { return *exec; }
};

inline constexpr sequenced_policy seq{};
inline constexpr parallel_policy par{};

namespace detail {

template <typename Policy>
struct policy_info
{
    static constexpr bool has_executor = false;
    static constexpr bool sequenced = std::is_same_v<Policy, sequenced_policy>;
    using executor_type = void;
};
template <typename E>
struct policy_info<parallel_executor_policy<E>>
{
    static constexpr bool has_executor = true;
    static constexpr bool sequenced = false;
    using executor_type = E;
};
template <typename E>
struct policy_info<sequenced_executor_policy<E>>
{
    static constexpr bool has_executor = true;
    static constexpr bool sequenced = true;
    using executor_type = E;
};

// ---------------------------------------------------------------------
// Iterator classification (algorithms.hpp:118-149)
// ---------------------------------------------------------------------

template <typename A, typename = void>
struct space_of
{
    using type = void;
};
template <typename A>
struct space_of<A, std::void_t<typename A::memory_space>>
{
    using type = typename A::memory_space;
};

template <typename It>
struct iter_info
{
    static constexpr bool device = false;
    static constexpr bool host_contiguous =
        std::is_pointer_v<It> || std::contiguous_iterator<It>;
};

template <typename V>
struct iter_info<vector_iterator<V>>
{
    using vector_type = std::remove_const_t<V>;
    using space = typename space_of<typename vector_type::allocator_type>::type;
    static constexpr bool device = std::is_same_v<space, cuda::cuda_memory_space>;
    static constexpr bool host_contiguous = false;
};

template <typename It>
auto device_base(It it)
{
    return it.container()->data_handle() + std::ptrdiff_t(it.position());
}

template <typename It>
auto host_base(It it)
{
    return std::to_address(it);
}

template <typename It>
using iter_value_t = typename std::iterator_traits<It>::value_type;

// ---------------------------------------------------------------------
// Cross-stream ordering for pieces whose data lives on another target
// ---------------------------------------------------------------------

inline void ensure_peer(int dev, int peer)
{
    if (dev == peer)
        return;
    static std::mutex mu;
    static std::set<std::pair<int, int>> done;
    std::lock_guard<std::mutex> lock(mu);
    if (done.count({dev, peer}))
        return;
    check(coloc_cuda_enable_peer_access(dev, peer), "coloc: enable peer access");
    done.insert({dev, peer});
}

/// Makes `to`'s stream wait for the work already queued on `from`.
inline void order_after(cuda::target const& from, cuda::target const& to)
{
    if (from == to)
        return;
    void* ev = nullptr;
    check(coloc_cuda_event_create(from.device(), &ev), "coloc: event_create");
    int st = coloc_cuda_event_record(from.device(), ev, from.stream());
    if (st == COLOC_OK)
        st = coloc_cuda_stream_wait_event(to.device(), to.stream(), ev);
    (void) coloc_cuda_event_destroy(from.device(), ev);
    check(st, "coloc: cross-stream ordering");
}

// Splits relative range r at every source segment boundary and calls
// fn(rel_begin, len, src_segments...) per piece.
template <typename T, std::size_t NSrc, typename Fn>
void for_each_piece(index_range const& r, cuda::segmented_ptr<T> const* srcs, Fn&& fn)
{
    std::size_t at = r.begin;
    while (at < r.end)
    {
        std::size_t len = r.end - at;
        cuda::segment<T> const* segs[NSrc > 0 ? NSrc : 1] = {};
        for (std::size_t k = 0; k < NSrc; ++k)
        {
            auto const& all = srcs[k].segments();
            std::size_t const abs = srcs[k].index() + at;
            auto const& s = all[srcs[k].segment_of(at)];
            len = std::min(len, s.end() - abs);
            segs[k] = &s;
        }
        fn(at, len, segs);
        at += len;
    }
}

// Range kernel for an elementwise op: dst[i] = op(src_0[i], ..., src_{N-1}[i])
// with i relative to the algorithm's first element.  launch() enqueues on
// the executing target's stream; data on other targets is ordered in with
// events and reached through peer access.
template <typename T, std::size_t NSrc, typename Launch>
struct elementwise_kernel
{
    cuda::segmented_ptr<T> dst;
    cuda::segmented_ptr<T> src[NSrc > 0 ? NSrc : 1];
    Launch run;    // int(int dev, void* stream, T* dst, T const* const* src, size_t n)

    void launch(cuda::target const& t, index_range const& r) const
    {
        for_each_piece<T, NSrc>(r, src, [&](std::size_t at, std::size_t len, auto const& segs) {
            // the destination piece may itself straddle destination
            // segments when the executor's blocks differ from the data's
            std::size_t done = 0;
            while (done < len)
            {
                std::size_t const rel = at + done;
                auto const& dseg = dst.segments()[dst.segment_of(rel)];
                std::size_t const abs = dst.index() + rel;
                std::size_t const n = std::min(len - done, dseg.end() - abs);
                T* d = dseg.base + (abs - dseg.offset);
                T const* s[NSrc > 0 ? NSrc : 1] = {};
                ensure_peer(t.device(), dseg.where.device());
                order_after(dseg.where, t);
                for (std::size_t k = 0; k < NSrc; ++k)
                {
                    auto const& ss = *segs[k];
                    s[k] = ss.base + (src[k].index() + rel - ss.offset);
                    ensure_peer(t.device(), ss.where.device());
                    order_after(ss.where, t);
                }
                check(run(t.device(), t.stream(), d, s, n), "coloc: kernel launch");
                if (schedule_log::global().enabled())
                    schedule_log::global().record({rel, rel + n, r.block, t.device(), t.stream(),
                        dseg.where.device(), dseg.where.stream(), "kernel"});
                // writers/readers on other streams must not overtake us
                order_after(t, dseg.where);
                for (std::size_t k = 0; k < NSrc; ++k)
                    order_after(t, segs[k]->where);
                done += n;
            }
        });
    }
};

template <typename T, std::size_t NSrc, typename Launch>
elementwise_kernel<T, NSrc, Launch> make_kernel(cuda::segmented_ptr<T> dst,
    std::array<cuda::segmented_ptr<T>, NSrc> const& src, Launch run)
{
    elementwise_kernel<T, NSrc, Launch> k{std::move(dst), {}, std::move(run)};
    for (std::size_t i = 0; i < NSrc; ++i)
        k.src[i] = src[i];
    return k;
}

/// One range per destination block overlapping [d0, d0+n), relative to
/// d0 and tagged with the block (algorithm_shape, algorithms.hpp:210-234).
template <typename OutIt>
shape block_shape(OutIt d_first, std::size_t n)
{
    shape s;
    auto const& part = d_first.container()->distribution();
    std::size_t const d0 = d_first.position();
    for (std::size_t b = 0; b < part.blocks.size(); ++b)
    {
        std::size_t const lo = std::max(part.blocks[b].offset, d0);
        std::size_t const hi = std::min(part.blocks[b].end(), d0 + n);
        if (lo < hi)
            s.push_back({lo - d0, hi - d0, b});
    }
    return s;
}

template <typename Exec, typename K>
void execute_shape(Exec& exec, shape const& s, K const& k, bool sequenced)
{
    static_assert(is_cuda_executor<std::remove_cv_t<Exec>>::value,
        "device data can only be processed by cuda_executor / cuda_block_executor");
    if (!sequenced)
    {
        executor_traits<std::remove_cv_t<Exec>>::bulk_execute(exec, k, s);
        return;
    }
    // seq: ranges one at a time in index order, each finished before the
    // next starts (algorithms.hpp:245-251).
    shape ordered = s;
    std::sort(ordered.begin(), ordered.end(),
        [](index_range const& a, index_range const& b) { return a.begin < b.begin; });
    for (index_range const& r : ordered)
    {
        executor_traits<std::remove_cv_t<Exec>>::bulk_execute(exec, k, shape{r});
        exec.drain();
    }
}

/// Default executor: the destination's own targets (so the streams that
/// built the data also process it).
template <typename OutIt, typename Fn>
void with_default_executor(OutIt d_first, Fn&& fn)
{
    auto const& part = d_first.container()->distribution();
    std::vector<cuda::target> targets;
    targets.reserve(part.blocks.size());
    for (auto const& b : part.blocks)
        targets.push_back(b.target);
    cuda_block_executor exec(std::move(targets));
    fn(exec);
}

template <typename Policy, typename OutIt, typename K>
void run_blocks(Policy const& policy, OutIt d_first, std::size_t n, K const& k)
{
    using info = policy_info<Policy>;
    shape const s = block_shape(d_first, n);
    if constexpr (info::has_executor)
        execute_shape(policy.executor(), s, k, info::sequenced);
    else
        with_default_executor(d_first,
            [&](auto& exec) { execute_shape(exec, s, k, info::sequenced); });
}

// Whether a host<->device copy must finish before copy() returns: always
// for the reference's blocking semantics; with a stream-ordered executor
// (executor_options::synchronous == false) the transfer is only enqueued on
// each block's stream -- the host buffer must then stay valid until the
// executor is drained, as with cudaMemcpyAsync -- so transfers of one block
// overlap kernels and transfers of the others.
template <typename Policy>
bool host_copy_blocks(Policy const& policy)
{
    if constexpr (policy_info<Policy>::has_executor)
        return policy.executor().options().synchronous;
    else
        return true;
}

// Host <-> device copies on each device block's own stream.  Every
// segment's copy is enqueued stream-ordered first (pageable host memory
// goes through the library's staging workers, so the segments of several
// GPUs/streams move concurrently); with `wait` the streams are then
// synchronized, which gives the reference's blocking semantics.
template <typename T>
void stage(cuda::segmented_ptr<T> const& dev, std::size_t n, T* host, bool to_device,
    bool wait = true)
{
    std::size_t const lo = dev.index(), hi = lo + n;
    std::vector<cuda::target const*> used;
    for (auto const& s : dev.segments())
    {
        std::size_t const b = std::max(lo, s.offset), e = std::min(hi, s.end());
        if (b >= e)
            continue;
        T* d = s.base + (b - s.offset);
        T* h = host + (b - lo);
        int st = to_device ?
            coloc_cuda_memcpy_stream_ordered(s.where.device(), s.where.stream(), d, h, (e - b) * sizeof(T)) :
            coloc_cuda_memcpy_stream_ordered(s.where.device(), s.where.stream(), h, d, (e - b) * sizeof(T));
        check(st, to_device ? "coloc::copy host->device" : "coloc::copy device->host");
        used.push_back(&s.where);
    }
    if (wait)
        for (auto const* t : used)
            t->synchronize();
}

}    // namespace detail

// ---------------------------------------------------------------------
// copy (algorithms.hpp:359-444)
// ---------------------------------------------------------------------

template <typename Policy, typename InIt, typename OutIt>
OutIt copy(Policy const& policy, InIt first, InIt last, OutIt d_first)
{
    using in = detail::iter_info<InIt>;
    using out = detail::iter_info<OutIt>;
    using T = detail::iter_value_t<InIt>;
    static_assert(std::is_same_v<T, detail::iter_value_t<OutIt>>,
        "coloc::copy requires identical element types");
    static_assert(std::is_trivially_copyable_v<T>, "device copies are bytewise");
    static_assert(in::device || out::device,
        "coloc_b200 algorithms operate on GPU-resident vectors; host-only ranges "
        "belong to the host library");

    std::size_t const n = std::size_t(last - first);
    if (n == 0)
        return d_first;

    if constexpr (in::host_contiguous && out::device)
    {
        detail::stage(detail::device_base(d_first), n,
            const_cast<T*>(detail::host_base(first)), true, detail::host_copy_blocks(policy));
    }
    else if constexpr (in::device && out::host_contiguous)
    {
        detail::stage(detail::device_base(first), n, detail::host_base(d_first), false,
            detail::host_copy_blocks(policy));
    }
    else
    {
        static_assert(in::device && out::device, "unsupported iterator combination");
        auto dst = detail::device_base(d_first);
        auto src = detail::device_base(first);
        if (&dst.storage() == &src.storage())
        {
            std::size_t const a = dst.index(), b = src.index();
            if (a != b && a < b + n && b < a + n)
                throw std::invalid_argument("coloc::copy: overlapping ranges");
        }
        auto run = [](int dev, void* stream, T* d, T const* const* s, std::size_t len) {
            return coloc_cuda_copy_bytes(dev, stream, d, s[0], len * sizeof(T));
        };
        auto k = detail::make_kernel<T, 1>(dst, {src}, run);
        detail::run_blocks(policy, d_first, n, k);
    }
    return d_first + std::ptrdiff_t(n);
}

// ---------------------------------------------------------------------
// transform (algorithms.hpp:452-526)
// ---------------------------------------------------------------------

template <typename Policy, typename InIt, typename OutIt, typename F>
OutIt transform(Policy const& policy, InIt first, InIt last, OutIt d_first, F f)
{
    using T = detail::iter_value_t<OutIt>;
    static_assert(detail::iter_info<InIt>::device && detail::iter_info<OutIt>::device,
        "coloc_b200 transform runs on GPU-resident vectors");
    static_assert(std::is_same_v<T, detail::iter_value_t<InIt>>,
        "device transform keeps the element type");
    using dispatch = detail::device_unary<F, T>;
    static_assert(dispatch::supported,
        "no sm_100a kernel for this operation: use a named op from coloc::ops "
        "(identity, scale, to_upper)");

    std::size_t const n = std::size_t(last - first);
    if (n == 0)
        return d_first;
    auto run = [f](int dev, void* stream, T* d, T const* const* s, std::size_t len) {
        return dispatch::launch(f, dev, stream, d, s[0], len);
    };
    auto k = detail::make_kernel<T, 1>(detail::device_base(d_first),
        {detail::device_base(first)}, run);
    detail::run_blocks(policy, d_first, n, k);
    return d_first + std::ptrdiff_t(n);
}

template <typename Policy, typename InIt1, typename InIt2, typename OutIt, typename F>
OutIt transform(Policy const& policy, InIt1 first1, InIt1 last1, InIt2 first2,
    OutIt d_first, F f)
{
    using T = detail::iter_value_t<OutIt>;
    static_assert(detail::iter_info<InIt1>::device && detail::iter_info<InIt2>::device &&
            detail::iter_info<OutIt>::device,
        "coloc_b200 transform runs on GPU-resident vectors");
    static_assert(std::is_same_v<T, detail::iter_value_t<InIt1>> &&
            std::is_same_v<T, detail::iter_value_t<InIt2>>,
        "device transform keeps the element type");
    using dispatch = detail::device_binary<F, T>;
    static_assert(dispatch::supported,
        "no sm_100a kernel for this operation: use a named op from coloc::ops "
        "(plus, triad, triad_fma)");

    std::size_t const n = std::size_t(last1 - first1);
    if (n == 0)
        return d_first;
    auto run = [f](int dev, void* stream, T* d, T const* const* s, std::size_t len) {
        return dispatch::launch(f, dev, stream, d, s[0], s[1], len);
    };
    auto k = detail::make_kernel<T, 2>(detail::device_base(d_first),
        {detail::device_base(first1), detail::device_base(first2)}, run);
    detail::run_blocks(policy, d_first, n, k);
    return d_first + std::ptrdiff_t(n);
}

// ---------------------------------------------------------------------
// for_each (named in BASELINE.json's north star; absent from the reference)
// ---------------------------------------------------------------------

template <typename Policy, typename It, typename F>
void for_each(Policy const& policy, It first, It last, F f)
{
    using T = detail::iter_value_t<It>;
    static_assert(detail::iter_info<It>::device, "coloc_b200 for_each runs on GPU-resident vectors");
    using dispatch = detail::device_in_place<F, T>;
    static_assert(dispatch::supported,
        "no sm_100a kernel for this operation: use a named op from coloc::ops "
        "(assign, multiply_by, make_upper)");
    std::size_t const n = std::size_t(last - first);
    if (n == 0)
        return;
    auto run = [f](int dev, void* stream, T* d, T const* const*, std::size_t len) {
        return dispatch::launch(f, dev, stream, d, len);
    };
    auto k = detail::make_kernel<T, 0>(detail::device_base(first), {}, run);
    detail::run_blocks(policy, first, n, k);
}

}    // namespace coloc
