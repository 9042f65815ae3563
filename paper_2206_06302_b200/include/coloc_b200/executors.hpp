// SPDX-License-Identifier: Apache-2.0
// Restates the public interface of the reference coloc library's executor_traits.hpp and detail/bulk.hpp
// (arXiv 2206.06302; /root/reference/proj/include/coloc, Apache-2.0): the
// names, signatures and semantics are kept for drop-in compatibility.
// executors.hpp -- executors whose bulk work items are kernel launches.
//
//   reference                                           here
//   executor_traits (executor_traits.hpp:81-240)        executor_traits (same derivation)
//   device_executor (device_executor.hpp:24-150):       cuda_executor: one cuda::target;
//     FIFO worker thread, one task per range              one kernel launch per range on
//                                                         the target's stream
//   block_executor (host_executor.hpp:171-290):         cuda_block_executor: range tagged
//     range tagged block b -> executor(b)                 block b -> launch on targets[b]
//   bulk_state (detail/bulk.hpp:131-198): first          same semantics at launch
//     error wins, not-yet-started ranges cancelled,       granularity; completion signalled
//     last range settles the promise                      by a stream host callback
//
// A bulk function for the CUDA executors is a *range kernel*: an object
// with `void launch(cuda::target const&, index_range const&) const` that
// enqueues the work for one range.  The algorithms (parallel.hpp) build
// these from named operations; host callables cannot run on a GPU and are
// rejected at compile time for bulk submission.
#pragma once

#include "coloc_b200/errors.hpp"
#include "coloc_b200/index_space.hpp"
#include "coloc_b200/targets.hpp"

#include <algorithm>
#include <array>
#include <atomic>
#include <cstdio>
#include <exception>
#include <functional>
#include <future>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <type_traits>
#include <utility>
#include <vector>

namespace coloc {

template <typename T>
using future = std::future<T>;

/// Sink for exceptions escaping fire-and-forget work (src/execution.cpp:12-67).
using apply_error_hook = std::function<void(std::exception_ptr)>;

namespace detail {

struct apply_hook_state
{
    std::mutex mu;
    apply_error_hook hook;
};

inline apply_hook_state& apply_hook()
{
    static apply_hook_state s;
    return s;
}

inline void report_apply_error(std::exception_ptr e) noexcept
{
    apply_error_hook hook;
    {
        std::lock_guard<std::mutex> lock(apply_hook().mu);
        hook = apply_hook().hook;
    }
    if (hook)
    {
        try
        {
            hook(e);
            return;
        }
        catch (...)
        {
        }
    }
    try
    {
        std::rethrow_exception(e);
    }
    catch (std::exception const& ex)
    {
        std::fprintf(stderr, "coloc: error in fire-and-forget task: %s\n", ex.what());
    }
    catch (...)
    {
        std::fprintf(stderr, "coloc: unknown error in fire-and-forget task\n");
    }
}

}    // namespace detail

inline void set_apply_error_hook(apply_error_hook hook)
{
    std::lock_guard<std::mutex> lock(detail::apply_hook().mu);
    detail::apply_hook().hook = std::move(hook);
}

/// Knobs shared by the CUDA executors.
struct executor_options
{
    /// true: bulk_execute returns only after the GPU work finished (the
    /// reference algorithms block on .get(), algorithms.hpp:236-252).
    /// false: it returns once the work is enqueued; stream order keeps every
    /// later operation on the same targets correct.
    bool synchronous = true;
};

namespace cuda {

template <typename K>
concept range_kernel = requires(K const& k, target const& t, index_range const& r) {
    k.launch(t, r);
};

}    // namespace cuda

namespace detail {

// Completion of one bulk submission (bulk.hpp:131-198, void case).
class bulk_completion
{
public:
    void store_error(std::exception_ptr e) noexcept
    {
        std::lock_guard<std::mutex> lock(mu_);
        if (!error_)
            error_ = std::move(e);
    }
    bool failed() const noexcept
    {
        std::lock_guard<std::mutex> lock(mu_);
        return error_ != nullptr;
    }
    void expect(std::size_t n) noexcept { remaining_.fetch_add(n, std::memory_order_relaxed); }
    void complete_one() noexcept
    {
        if (remaining_.fetch_sub(1, std::memory_order_acq_rel) == 1)
            settle();
    }
    std::future<void> get_future() { return promise_.get_future(); }

private:
    void settle() noexcept
    {
        std::lock_guard<std::mutex> lock(mu_);
        if (error_)
            promise_.set_exception(error_);
        else
            promise_.set_value();
    }

    mutable std::mutex mu_;
    std::exception_ptr error_;
    std::atomic<std::size_t> remaining_{1};    // the submitter's own token
    std::promise<void> promise_;
};

// First error of a blocking bulk submission: the bulk_completion
// contract without a promise (no shared-state allocation per call on the
// synchronous path).
struct error_slot
{
    std::exception_ptr error;
    void store_error(std::exception_ptr e) noexcept
    {
        if (!error)
            error = std::move(e);
    }
};

// The executors a bulk submission launched on: a few inline slots (one
// per partition block of a vector, usually 1-8), the heap beyond.
template <typename E>
class used_set
{
public:
    void insert(E* e)
    {
        for (std::size_t i = 0; i < n_; ++i)
            if (inline_[i] == e)
                return;
        if (std::find(more_.begin(), more_.end(), e) != more_.end())
            return;
        if (n_ < inline_.size())
            inline_[n_++] = e;
        else
            more_.push_back(e);
    }
    template <typename F>
    void for_each(F&& f) const
    {
        for (std::size_t i = 0; i < n_; ++i)
            f(inline_[i]);
        for (E* e : more_)
            f(e);
    }

private:
    std::array<E*, 8> inline_{};
    std::size_t n_ = 0;
    std::vector<E*> more_;
};

inline void host_fn_complete(void* user, int status)
{
    auto* holder = static_cast<std::shared_ptr<bulk_completion>*>(user);
    if (status != COLOC_OK)
        (*holder)->store_error(std::make_exception_ptr(
            error("coloc::cuda: device work before this completion failed (status " +
                std::to_string(status) + ")")));
    (*holder)->complete_one();
    delete holder;
}

// Arrange for `state->complete_one()` once `t`'s stream drains.
inline void complete_after(cuda::target const& t, std::shared_ptr<bulk_completion> const& state)
{
    state->expect(1);
    auto* holder = new std::shared_ptr<bulk_completion>(state);
    int st = coloc_cuda_launch_host_func(t.device(), t.stream(), &host_fn_complete, holder);
    if (st != COLOC_OK)
    {
        delete holder;
        try
        {
            throw_status(st, "coloc::cuda completion callback");
        }
        catch (...)
        {
            state->store_error(std::current_exception());
        }
        state->complete_one();
    }
}

template <typename F, typename... Ts>
using async_result_t = std::invoke_result_t<std::decay_t<F>&, std::decay_t<Ts>&...>;

// Host task run in stream order from a CUDA host callback: the device
// counterpart of fifo_queue::enqueue (device.hpp:63-71).  The callable must
// not call CUDA itself (CUDA forbids API calls inside host callbacks).
struct host_task
{
    std::function<void()> fn;
    static void run(void* user, int)
    {
        std::unique_ptr<host_task> self(static_cast<host_task*>(user));
        self->fn();
    }
};

template <typename R>
future<R> rejected_future(std::exception_ptr e)
{
    std::promise<R> p;
    p.set_exception(std::move(e));
    return p.get_future();
}

}    // namespace detail

/// Executor bound to one cuda::target (device + stream).
class cuda_executor
{
public:
    explicit cuda_executor(cuda::target t, executor_options options = {})
      : target_(std::move(t))
      , options_(options)
    {
        if (!target_.valid())
            throw invalid_target_error("cuda_executor: default-constructed target");
    }

    cuda::target const& target() const noexcept { return target_; }
    executor_options const& options() const noexcept { return options_; }
    /// One in-order stream: a single "worker" (algorithms.hpp:186-204 uses
    /// this to size shapes; GPU shapes use one range per block).
    std::size_t worker_count() const noexcept { return 1; }

    /// Runs f(ts...) after all previously submitted work on the stream.
    template <typename F, typename... Ts>
    auto async_execute(F&& f, Ts&&... ts) -> future<detail::async_result_t<F, Ts...>>
    {
        using R = detail::async_result_t<F, Ts...>;
        auto task = std::make_shared<std::packaged_task<R()>>(
            [f = std::decay_t<F>(std::forward<F>(f)),
                args = std::make_tuple(std::forward<Ts>(ts)...)]() mutable {
                return std::apply(f, args);
            });
        future<R> result = task->get_future();
        auto* box = new detail::host_task{[task] { (*task)(); }};
        int st = coloc_cuda_launch_host_func(target_.device(), target_.stream(),
            &detail::host_task::run, box);
        if (st != COLOC_OK)
        {
            delete box;
            try
            {
                detail::throw_status(st == COLOC_ERR_INVALID_ARGUMENT ? COLOC_ERR_SUBMISSION : st,
                    target_.description() + " rejected work");
            }
            catch (...)
            {
                return detail::rejected_future<R>(std::current_exception());
            }
        }
        return result;
    }

    /// Synchronous form: waits for the stream, then runs f on the caller
    /// (cheaper than a host callback round trip).
    template <typename F, typename... Ts>
    decltype(auto) execute(F&& f, Ts&&... ts)
    {
        target_.synchronize();
        return std::invoke(std::forward<F>(f), std::forward<Ts>(ts)...);
    }

    template <typename F, typename... Ts>
    void apply_execute(F&& f, Ts&&... ts)
    {
        auto* box = new detail::host_task{
            [f = std::decay_t<F>(std::forward<F>(f)),
                args = std::make_tuple(std::forward<Ts>(ts)...)]() mutable {
                try
                {
                    std::apply(f, args);
                }
                catch (...)
                {
                    detail::report_apply_error(std::current_exception());
                }
            }};
        int st = coloc_cuda_launch_host_func(target_.device(), target_.stream(),
            &detail::host_task::run, box);
        if (st != COLOC_OK)
        {
            delete box;
            detail::report_apply_error(std::make_exception_ptr(
                submission_error(target_.description() + " rejected work")));
        }
    }

    /// One launch per range, in shape order; the future settles when the
    /// stream has executed all of them.  A failing launch cancels the
    /// ranges after it and becomes the future's exception.
    template <cuda::range_kernel K>
    future<void> bulk_async_execute(K const& k, shape const& s)
    {
        auto state = std::make_shared<detail::bulk_completion>();
        auto result = state->get_future();
        launch_all(k, s, *state);
        detail::complete_after(target_, state);
        state->complete_one();
        return result;
    }

    template <cuda::range_kernel K>
    void bulk_execute(K const& k, shape const& s)
    {
        detail::error_slot sink;
        launch_all(k, s, sink);
        if (sink.error)
        {
            // Let the ranges that did launch finish, then rethrow the
            // first error.
            target_.synchronize();
            std::rethrow_exception(sink.error);
        }
        if (options_.synchronous)
            target_.synchronize();
    }

    /// Waits for everything submitted so far (device_executor::drain).
    void drain() { target_.synchronize(); }

private:
    template <cuda::range_kernel K, typename Sink>
    void launch_all(K const& k, shape const& s, Sink& state)
    {
        for (index_range const& r : s)
        {
            if (r.size() == 0)
                continue;
            try
            {
                k.launch(target_, r);
            }
            catch (...)
            {
                state.store_error(std::current_exception());
                return;
            }
        }
    }

    cuda::target target_;
    executor_options options_;
};

/// Executor over an ordered target list: work tagged with block b runs on
/// targets[b] (host_executor.hpp:171-290), so each block of a partitioned
/// vector is processed by the GPU that holds it.
class cuda_block_executor
{
public:
    explicit cuda_block_executor(std::vector<cuda::target> targets, executor_options options = {})
      : options_(options)
    {
        if (targets.empty())
            throw invalid_target_error("cuda block executor requires at least one target");
        executors_.reserve(targets.size());
        for (auto& t : targets)
            executors_.push_back(std::make_unique<cuda_executor>(std::move(t), options));
    }

    std::size_t block_count() const noexcept { return executors_.size(); }
    cuda_executor& executor(std::size_t block) noexcept
    {
        return *executors_[block % executors_.size()];
    }
    std::vector<cuda::target> targets() const
    {
        std::vector<cuda::target> out;
        out.reserve(executors_.size());
        for (auto const& e : executors_)
            out.push_back(e->target());
        return out;
    }
    std::size_t worker_count() const noexcept { return executors_.size(); }
    executor_options const& options() const noexcept { return options_; }

    template <typename F, typename... Ts>
    auto async_execute(F&& f, Ts&&... ts)
    {
        return next().async_execute(std::forward<F>(f), std::forward<Ts>(ts)...);
    }

    template <typename F, typename... Ts>
    decltype(auto) execute(F&& f, Ts&&... ts)
    {
        return next().execute(std::forward<F>(f), std::forward<Ts>(ts)...);
    }

    template <typename F, typename... Ts>
    void apply_execute(F&& f, Ts&&... ts)
    {
        next().apply_execute(std::forward<F>(f), std::forward<Ts>(ts)...);
    }

    /// Launches every range on its block's target (untagged ranges round
    /// robin); settles once all involved streams have drained.
    template <cuda::range_kernel K>
    future<void> bulk_async_execute(K const& k, shape const& s)
    {
        auto state = std::make_shared<detail::bulk_completion>();
        auto result = state->get_future();
        detail::used_set<cuda_executor> used;
        launch_all(k, s, *state, used);
        used.for_each([&](cuda_executor* e) { detail::complete_after(e->target(), state); });
        state->complete_one();
        return result;
    }

    template <cuda::range_kernel K>
    void bulk_execute(K const& k, shape const& s)
    {
        detail::error_slot sink;
        detail::used_set<cuda_executor> used;
        launch_all(k, s, sink, used);
        // The reference's caller blocks until the last block's range
        // settles (bulk.hpp:175-179): wait on every stream that got work,
        // also when a later launch failed, so no launch is left running.
        if (options_.synchronous || sink.error)
            used.for_each([](cuda_executor* e) { e->drain(); });
        if (sink.error)
            std::rethrow_exception(sink.error);
    }

    void drain()
    {
        for (auto const& e : executors_)
            e->drain();
    }

private:
    cuda_executor& next() noexcept
    {
        return *executors_[rr_.fetch_add(1, std::memory_order_relaxed) % executors_.size()];
    }

    template <cuda::range_kernel K, typename Sink>
    void launch_all(K const& k, shape const& s, Sink& state, detail::used_set<cuda_executor>& used)
    {
        for (index_range const& r : s)
        {
            if (r.size() == 0)
                continue;
            cuda_executor& e = r.block == no_block ? next() : executor(r.block);
            try
            {
                k.launch(e.target(), r);
            }
            catch (...)
            {
                state.store_error(std::current_exception());
                break;
            }
            used.insert(&e);
        }
    }

    executor_options options_;
    std::vector<std::unique_ptr<cuda_executor>> executors_;
    std::atomic<std::size_t> rr_{0};
};

namespace detail {

template <typename E>
struct is_cuda_executor : std::false_type
{
};
template <>
struct is_cuda_executor<cuda_executor> : std::true_type
{
};
template <>
struct is_cuda_executor<cuda_block_executor> : std::true_type
{
};

template <typename E, typename F, typename... Ts>
concept has_async_execute = requires(E& e, F&& f, Ts&&... ts) {
    e.async_execute(std::forward<F>(f), std::forward<Ts>(ts)...);
};
template <typename E, typename F, typename... Ts>
concept has_execute = requires(E& e, F&& f, Ts&&... ts) {
    e.execute(std::forward<F>(f), std::forward<Ts>(ts)...);
};
template <typename E, typename F, typename... Ts>
concept has_apply_execute = requires(E& e, F&& f, Ts&&... ts) {
    e.apply_execute(std::forward<F>(f), std::forward<Ts>(ts)...);
};
template <typename E, typename F>
concept has_bulk_async_execute = requires(E& e, F const& f, shape const& s) {
    e.bulk_async_execute(f, s);
};
template <typename E, typename F>
concept has_bulk_execute = requires(E& e, F const& f, shape const& s) {
    e.bulk_execute(f, s);
};

}    // namespace detail

/// Uniform executor access (executor_traits.hpp:81-240): an executor must
/// provide async_execute; the other forms are derived when missing.  Bulk
/// derivation (one async task per range plus a final join, executor_traits.hpp:
/// 185-239) applies to executors whose bulk function is a host callable f(i).
template <typename Executor>
struct executor_traits
{
    using executor_type = Executor;

    template <typename F, typename... Ts>
    static auto async_execute(Executor& e, F&& f, Ts&&... ts)
    {
        static_assert(detail::has_async_execute<Executor, F, Ts...>,
            "an executor must implement async_execute");
        return e.async_execute(std::forward<F>(f), std::forward<Ts>(ts)...);
    }

    template <typename F, typename... Ts>
    static decltype(auto) execute(Executor& e, F&& f, Ts&&... ts)
    {
        if constexpr (detail::has_execute<Executor, F, Ts...>)
            return e.execute(std::forward<F>(f), std::forward<Ts>(ts)...);
        else
            return async_execute(e, std::forward<F>(f), std::forward<Ts>(ts)...).get();
    }

    template <typename F, typename... Ts>
    static void apply_execute(Executor& e, F&& f, Ts&&... ts)
    {
        if constexpr (detail::has_apply_execute<Executor, F, Ts...>)
            e.apply_execute(std::forward<F>(f), std::forward<Ts>(ts)...);
        else
        {
            auto wrapped = [f = std::decay_t<F>(std::forward<F>(f)),
                               args = std::make_tuple(std::forward<Ts>(ts)...)]() mutable {
                try
                {
                    std::apply(f, args);
                }
                catch (...)
                {
                    detail::report_apply_error(std::current_exception());
                }
            };
            (void) e.async_execute(std::move(wrapped));
        }
    }

    template <typename F>
    static future<void> bulk_async_execute(Executor& e, F const& f, shape const& s)
    {
        if constexpr (detail::has_bulk_async_execute<Executor, F>)
            return e.bulk_async_execute(f, s);
        else
            return bulk_via_async(e, f, s);
    }

    template <typename F>
    static void bulk_execute(Executor& e, F const& f, shape const& s)
    {
        if constexpr (detail::has_bulk_execute<Executor, F>)
            e.bulk_execute(f, s);
        else
            bulk_async_execute(e, f, s).get();
    }

private:
    // One async task per range calling f(i) for each index, joined by a
    // final task; first error wins and cancels ranges not yet started.
    template <typename F>
    static future<void> bulk_via_async(Executor& e, F const& f, shape const& s)
    {
        static_assert(std::is_invocable_v<F const&, std::size_t>,
            "derived bulk execution needs a callable f(index)");
        struct state
        {
            std::atomic<bool> cancelled{false};
            std::mutex mu;
            std::exception_ptr first;
        };
        auto st = std::make_shared<state>();
        auto fn = std::make_shared<F>(f);
        using range_future = decltype(e.async_execute([] {}));
        auto pending = std::make_shared<std::vector<range_future>>();
        pending->reserve(s.size());
        for (index_range const& r : s)
        {
            auto body = [st, fn, r] {
                if (st->cancelled.load(std::memory_order_relaxed))
                    return;
                try
                {
                    for (std::size_t i = r.begin; i != r.end; ++i)
                        (*fn)(i);
                }
                catch (...)
                {
                    st->cancelled = true;
                    std::lock_guard<std::mutex> lock(st->mu);
                    if (!st->first)
                        st->first = std::current_exception();
                }
            };
            try
            {
                pending->push_back(e.async_execute(std::move(body)));
            }
            catch (...)
            {
                st->cancelled = true;
                std::lock_guard<std::mutex> lock(st->mu);
                if (!st->first)
                    st->first = std::current_exception();
            }
        }
        return e.async_execute([st, pending] {
            for (auto& p : *pending)
            {
                try
                {
                    p.get();
                }
                catch (...)
                {
                    std::lock_guard<std::mutex> lock(st->mu);
                    if (!st->first)
                        st->first = std::current_exception();
                }
            }
            if (st->first)
                std::rethrow_exception(st->first);
        });
    }
};

}    // namespace coloc
