// stream_driver.cpp -- the STREAM benchmark on the C++ drop-in API,
// exported through include/coloc_stream.h.
//
// The benchmark body is Listing 4 with the lambdas
// replaced by the named operations of coloc::ops, run with par.on(exec)
// over vectors whose allocator and executor share the same targets (the
// co-location rule of PAPER.md:366-367 / SPEC.md:531).  Timing follows
// SPEC.md:516-520 and BASELINE.md section 3: CUDA events around each
// kernel on every target, per-kernel time = max over targets, bytes by the
// 2/2/3/3 rule.  Validation is SPEC.md:539-547.
#include "coloc_stream.h"

#include "coloc_b200/coloc.hpp"

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <map>
#include <memory>
#include <new>
#include <string>
#include <utility>
#include <vector>

namespace {

thread_local std::string t_error;

int report(std::exception_ptr e)
{
    try
    {
        std::rethrow_exception(e);
    }
    catch (coloc::allocation_error const& x)
    {
        t_error = x.what();
        return COLOC_ERR_ALLOCATION;
    }
    catch (coloc::invalid_target_error const& x)
    {
        t_error = x.what();
        return COLOC_ERR_INVALID_TARGET;
    }
    catch (coloc::submission_error const& x)
    {
        t_error = x.what();
        return COLOC_ERR_SUBMISSION;
    }
    catch (std::invalid_argument const& x)
    {
        t_error = x.what();
        return COLOC_ERR_INVALID_ARGUMENT;
    }
    catch (std::bad_alloc const&)
    {
        t_error = "host allocation failed";
        return COLOC_ERR_ALLOCATION;
    }
    catch (std::exception const& x)
    {
        t_error = x.what();
        return COLOC_ERR_CUDA;
    }
    catch (...)
    {
        t_error = "unknown error";
        return COLOC_ERR_CUDA;
    }
}

template <typename F>
int guarded(F&& f)
{
    try
    {
        f();
        return COLOC_OK;
    }
    catch (...)
    {
        return report(std::current_exception());
    }
}

// Events owned per target for one timed region.
struct event_pair
{
    int dev;
    void* start = nullptr;
    void* stop = nullptr;
};

class run_base
{
public:
    virtual ~run_base() = default;
    virtual void iterate(int record) = 0;
    virtual void iterate_many(int k, int record, bool graph) = 0;
    virtual void sync() = 0;
    virtual int recorded() = 0;
    virtual std::array<double, 4> kernel_ms(int i) = 0;
    virtual double iteration_ms(int i) = 0;
    virtual void clear_records() = 0;
    virtual int iterations() const = 0;
    virtual double e2e_step(int ntimes) = 0;
    virtual void err_sums(double expected[3], double sums[3], double* dev_out) = 0;
    virtual void checksums(std::uint64_t out[3]) = 0;
    virtual void read(int k, std::uint64_t first, std::uint64_t n, void* out) = 0;
    virtual void set_comm(void* comm) = 0;
    virtual char const* reduction() const = 0;
};

template <typename T>
class stream_run final : public run_base
{
    using alloc_t = coloc::cuda::block_allocator<T>;
    using vec_t = coloc::vector<T, alloc_t>;

public:
    explicit stream_run(coloc_stream_config const& cfg)
      : cfg_(cfg)
      , targets_(make_targets(cfg))
      , alloc_(targets_)
      , exec_(targets_, coloc::executor_options{cfg.synchronous != 0})
      , a_(make(0))
      , b_(make(1))
      , c_(make(2))
    {
        if (cfg.host_buffers)
        {
            bool const pinned = cfg.host_buffers != 2;
            for (int k = 0; k < 3; ++k)
            {
                host_in_[k] = host_array(std::size_t(cfg.count), pinned);
                host_out_[k] = host_array(std::size_t(cfg.count), pinned);
                // the same initial contents the device vectors got
                read(k, 0, cfg.count, host_in_[k].get());
            }
        }
    }

    ~stream_run() override
    {
        try
        {
            sync();
        }
        catch (...)
        {
        }
        release_graphs();
        clear_records();
        for (std::size_t t = 0; t < side_.size(); ++t)
            if (side_[t])
                (void) coloc_cuda_stream_destroy(targets_[t].device(), side_[t]);
        if (!comms_.empty())
            (void) coloc_cuda_nccl_destroy(int(comms_.size()), comms_.data());
    }

    // record: 0 none, 1 events around every kernel, 2 events around the
    // whole iteration only (nothing between the kernels, so programmatic
    // dependent launch can overlap each kernel's launch with its
    // predecessor's tail), 3 every kernel timed by completion stamps on a
    // side stream (no event node between the kernels on their own stream:
    // kernel k spans the completion of kernel k-1 to its own completion).
    // (4, in-kernel spans, runs through iterate_many/iterate_spans.)
    void iterate(int record) override
    {
        auto policy = coloc::par.on(exec_);
        T const s = T(cfg_.scalar);
        T const ts = T(cfg_.triad_scalar);
        side_stamps_ = record == 3;
        std::vector<event_pair>* ev = record == 1 || record == 3 ? &records_.emplace_back() : nullptr;
        std::vector<event_pair>* whole = record == 2 ? &records_.emplace_back() : nullptr;
        if (whole)
            for (auto const& t : targets_)
            {
                whole->push_back(new_pair(t));
                coloc::detail::check(coloc_cuda_event_record(t.device(), whole->back().start, t.stream()),
                    "coloc_stream: event record");
            }

        // Listing 4, kernel by kernel.
        mark(ev, 0, true);
        coloc::copy(policy, a_.begin(), a_.end(), c_.begin());
        mark(ev, 0, false);
        mark(ev, 1, true);
        coloc::transform(policy, c_.begin(), c_.end(), b_.begin(), coloc::ops::scale<T>{s});
        mark(ev, 1, false);
        mark(ev, 2, true);
        coloc::transform(policy, a_.begin(), a_.end(), b_.begin(), c_.begin(),
            coloc::ops::plus<T>{});
        mark(ev, 2, false);
        mark(ev, 3, true);
        if (cfg_.fma)
            coloc::transform(policy, b_.begin(), b_.end(), c_.begin(), a_.begin(),
                coloc::ops::triad_fma<T>{ts});
        else
            coloc::transform(policy, b_.begin(), b_.end(), c_.begin(), a_.begin(),
                coloc::ops::triad<T>{ts});
        mark(ev, 3, false);
        if (whole)
            for (std::size_t t = 0; t < targets_.size(); ++t)
                coloc::detail::check(coloc_cuda_event_record(targets_[t].device(), (*whole)[t].stop,
                                         targets_[t].stream()),
                    "coloc_stream: event record");
        ++iterations_;
    }

    // k iterations; with `graph` (stream-ordered executor) every target's
    // stream is captured into its own CUDA graph -- its kernels and the
    // event records between them -- and each graph is replayed with one
    // launch, so host launch overhead stays out of the device timeline for
    // any number of targets and GPUs (the STREAM loop has no cross-target
    // dependency, so per-target graphs lose no ordering).
    void iterate_many(int k, int record, bool graph) override
    {
        if (k <= 0)
            return;
        if (record == 4)
        {
            iterate_spans(k, graph);
            return;
        }
        // chain: each target's kernels hand over tile by tile (kernels.cu)
        bool const chain = !cfg_.synchronous &&
            (cfg_.chain == 1 || (cfg_.chain == 2 && record != 1 && record != 3 && chain_pays()));
        auto body = [&] {
            std::size_t opened = 0;
            try
            {
                if (chain)
                    for (; opened < targets_.size(); ++opened)
                        coloc::detail::check(coloc_cuda_chain_begin(targets_[opened].device(),
                                                 targets_[opened].stream()),
                            "chain_begin");
                for (int i = 0; i < k; ++i)
                    iterate(record);
                join_sides();
            }
            catch (...)
            {
                // never leave a chain open on a target's stream
                for (std::size_t t = 0; t < opened; ++t)
                    (void) coloc_cuda_chain_end(targets_[t].device(), targets_[t].stream());
                throw;
            }
            int st = COLOC_OK;
            for (std::size_t t = 0; t < opened; ++t)
            {
                int const e = coloc_cuda_chain_end(targets_[t].device(), targets_[t].stream());
                st = st == COLOC_OK ? e : st;
            }
            coloc::detail::check(st, "chain_end");
        };
        if (!graph || cfg_.synchronous)
            body();
        else
            capture(body);
    }

    void sync() override
    {
        join_sides();
        exec_.drain();
        for (std::size_t t = 0; t < side_.size(); ++t)
            if (side_[t])
                coloc::detail::check(coloc_cuda_stream_sync(targets_[t].device(), side_[t]), "side sync");
        release_graphs();
    }

    int recorded() override { return int(records_.size()); }

    std::array<double, 4> kernel_ms(int i) override
    {
        if (i < 0 || std::size_t(i) >= records_.size())
            throw std::invalid_argument("kernel_ms: no such recorded iteration");
        sync();
        if (auto it = span_rows_.find(std::size_t(i)); it != span_rows_.end())
            return it->second;
        std::array<double, 4> out{0, 0, 0, 0};
        auto const& r = records_[std::size_t(i)];
        std::size_t const nt = targets_.size();
        if (r.size() != 4 * nt)
            throw std::invalid_argument("kernel_ms: iteration-level record (use coloc_stream_iteration_ms)");
        for (int k = 0; k < 4; ++k)
            for (std::size_t t = 0; t < nt; ++t)
            {
                auto const& e = r[std::size_t(k) * nt + t];
                float ms = 0;
                coloc::detail::check(coloc_cuda_event_elapsed_ms(e.start, e.stop, &ms),
                    "coloc_stream: elapsed");
                out[std::size_t(k)] = std::max(out[std::size_t(k)], double(ms));
            }
        return out;
    }

    // Span of recorded iteration i (first kernel's start to last kernel's
    // stop), max over this process's targets.
    double iteration_ms(int i) override
    {
        if (i < 0 || std::size_t(i) >= records_.size())
            throw std::invalid_argument("iteration_ms: no such recorded iteration");
        sync();
        if (auto it = span_rows_.find(std::size_t(i)); it != span_rows_.end())
            return it->second[0] + it->second[1] + it->second[2] + it->second[3];
        auto const& r = records_[std::size_t(i)];
        std::size_t const nt = targets_.size();
        double out = 0;
        for (std::size_t t = 0; t < nt; ++t)
        {
            void* stop = r.size() == nt ? r[t].stop : r[3 * nt + t].stop;
            float ms = 0;
            coloc::detail::check(coloc_cuda_event_elapsed_ms(r[t].start, stop, &ms), "coloc_stream: elapsed");
            out = std::max(out, double(ms));
        }
        return out;
    }

    void clear_records() override
    {
        // kernel k's start event is kernel k-1's stop event (see mark()), so
        // only the first kernel's starts and every stop are owned
        std::size_t const nt = targets_.size();
        for (auto& r : records_)
            for (std::size_t s = 0; s < r.size(); ++s)
            {
                if (s < nt)
                    (void) coloc_cuda_event_destroy(r[s].dev, r[s].start);
                (void) coloc_cuda_event_destroy(r[s].dev, r[s].stop);
            }
        records_.clear();
        span_rows_.clear();
    }

    int iterations() const override { return iterations_; }

    double e2e_step(int ntimes) override
    {
        if (!host_in_[0])
            throw std::invalid_argument("e2e_step: created without host_buffers");
        auto policy = coloc::par.on(exec_);
        std::size_t const n = std::size_t(cfg_.count);
        // One start event per device, recorded on that device's first target;
        // the device's other targets wait for it, so every block's work lies
        // inside [start, stop_t] and the step's span on a device is
        // max_t elapsed(start, stop_t).  With several targets per GPU and a
        // stream-ordered executor, block b's transfers overlap block b-1's
        // kernels (the block partition doubling as a copy/compute pipeline).
        std::vector<event_pair> ev;
        std::vector<std::size_t> first_on_dev(targets_.size());
        for (std::size_t i = 0; i < targets_.size(); ++i)
        {
            ev.push_back(new_pair(targets_[i]));
            first_on_dev[i] = i;
            for (std::size_t j = 0; j < i; ++j)
                if (targets_[j].device() == targets_[i].device())
                {
                    first_on_dev[i] = j;
                    break;
                }
        }
        // Host->device block by block (a, b, c of block 0 first), so the copy
        // engine delivers whole blocks in order and each block's kernels can
        // start while later blocks are still in flight.
        vec_t* vs[3] = {&a_, &b_, &c_};
        auto const& part = a_.distribution();
        auto body = [&] {
            for (auto const& blk : part.blocks)
                for (int k = 0; k < 3; ++k)
                {
                    T* h = host_in_[k].get() + blk.offset;
                    coloc::copy(policy, h, h + blk.length, vs[k]->begin() + std::ptrdiff_t(blk.offset));
                }
            for (int k = 0; k < ntimes; ++k)
                iterate(0);
            for (auto const& blk : part.blocks)
                for (int k = 0; k < 3; ++k)
                {
                    auto first = vs[k]->begin() + std::ptrdiff_t(blk.offset);
                    coloc::copy(policy, first, first + std::ptrdiff_t(blk.length),
                        host_out_[k].get() + blk.offset);
                }
        };
        // Pinned buffers with a stream-ordered executor: the whole step is
        // captured first (one graph per target: copy nodes and kernels),
        // so the timed region holds no host launches.  Pageable buffers
        // need the staging workers, which a graph cannot hold.
        bool const graph = cfg_.host_buffers == 1 && !cfg_.synchronous;
        std::vector<void*> graphs;
        if (graph)
            graphs = capture_graphs(body);
        for (std::size_t i = 0; i < targets_.size(); ++i)
        {
            auto const& t = targets_[i];
            if (first_on_dev[i] == i)
                coloc::detail::check(coloc_cuda_event_record(t.device(), ev[i].start, t.stream()),
                    "coloc_stream: event record");
            else
                coloc::detail::check(coloc_cuda_stream_wait_event(t.device(), t.stream(),
                                         ev[first_on_dev[i]].start),
                    "coloc_stream: stream wait");
        }
        if (graph)
            launch_graphs(graphs);
        else
            body();
        (void) n;
        for (std::size_t i = 0; i < targets_.size(); ++i)
            coloc::detail::check(coloc_cuda_event_record(targets_[i].device(), ev[i].stop,
                                     targets_[i].stream()),
                "coloc_stream: event record");
        sync();
        double worst = 0;
        for (std::size_t i = 0; i < ev.size(); ++i)
        {
            float ms = 0;
            coloc::detail::check(
                coloc_cuda_event_elapsed_ms(ev[first_on_dev[i]].start, ev[i].stop, &ms),
                "coloc_stream: elapsed");
            worst = std::max(worst, double(ms));
        }
        for (auto& e : ev)
        {
            (void) coloc_cuda_event_destroy(e.dev, e.start);
            (void) coloc_cuda_event_destroy(e.dev, e.stop);
        }
        // The device arrays now hold the state after this step's
        // iterations starting from the initial contents; the iteration
        // count restarts so validation refers to this step.
        iterations_ = ntimes;
        return worst;
    }

    void err_sums(double expected[3], double sums[3], double* dev_out) override
    {
        expected_values(expected);
        std::size_t const nt = targets_.size();
        auto const& sa = a_.data_handle().segments();
        auto const& sb = b_.data_handle().segments();
        auto const& sc = c_.data_handle().segments();

        // Fused per-block error sums into 3 doubles of device memory per block.
        struct dev_buf
        {
            int dev;
            void* p = nullptr;
            ~dev_buf() { (void) coloc_cuda_free(dev, p); }
        };
        std::vector<std::unique_ptr<dev_buf>> bufs;
        for (std::size_t t = 0; t < nt; ++t)
        {
            auto const& tg = sa[t].where;
            auto b = std::make_unique<dev_buf>();
            b->dev = tg.device();
            coloc::detail::check(coloc_cuda_malloc(tg.device(), 3 * sizeof(double), &b->p),
                "coloc_stream: err buffer");
            double const zero[3] = {0.0, 0.0, 0.0};
            int st = coloc_cuda_memcpy_async(tg.device(), tg.stream(), b->p, zero, sizeof zero);
            if (st == COLOC_OK)
                st = coloc_cuda_stream_sync(tg.device(), tg.stream());
            if (st == COLOC_OK && sa[t].length != 0)
            {
                if constexpr (std::is_same_v<T, double>)
                    st = coloc_cuda_stream_err_sums_f64(tg.device(), tg.stream(), sa[t].base,
                        sb[t].base, sc[t].base, sa[t].length, expected, static_cast<double*>(b->p));
                else
                    st = coloc_cuda_stream_err_sums_f32(tg.device(), tg.stream(), sa[t].base,
                        sb[t].base, sc[t].base, sa[t].length, expected, static_cast<double*>(b->p));
            }
            coloc::detail::check(st, "coloc_stream: err sums");
            bufs.push_back(std::move(b));
        }

        // One block per GPU on several GPUs: the sums are combined by an NCCL
        // allreduce over NVLink that follows the kernels on the same streams
        // (SURVEY.md section 8e).  Otherwise the host adds them in block order.
        bool const want_nccl = cfg_.reduction == COLOC_STREAM_REDUCE_NCCL ||
            (cfg_.reduction == COLOC_STREAM_REDUCE_AUTO && distinct_devices() && nt > 1);
        if (want_nccl && !distinct_devices())
            throw std::invalid_argument("coloc_stream: the NCCL reduction needs one target per GPU "
                                        "(NCCL allows one rank per device)");
        if (want_nccl)
        {
            if (comms_.empty())
            {
                std::vector<int> devs;
                for (auto const& t : targets_)
                    devs.push_back(t.device());
                comms_.assign(nt, nullptr);
                coloc::detail::check(coloc_cuda_nccl_init_all(int(nt), devs.data(), comms_.data()),
                    "coloc_stream: ncclCommInitAll");
            }
            std::vector<double*> ptrs;
            std::vector<void*> streams;
            for (std::size_t t = 0; t < nt; ++t)
            {
                ptrs.push_back(static_cast<double*>(bufs[t]->p));
                streams.push_back(targets_[t].stream());
            }
            coloc::detail::check(coloc_cuda_nccl_allreduce_sum_f64(int(nt), comms_.data(),
                                     ptrs.data(), 3, streams.data()),
                "coloc_stream: ncclAllReduce");
            auto const& t0 = targets_.front();
            coloc::detail::check(coloc_cuda_memcpy_async(t0.device(), t0.stream(), sums,
                                     bufs[0]->p, 3 * sizeof(double)),
                "coloc_stream: err sums");
            sync();
            last_reduction_ = "nccl";
        }
        else
        {
            std::vector<double> per(nt * 3, 0.0);
            for (std::size_t t = 0; t < nt; ++t)
            {
                auto const& tg = targets_[t];
                coloc::detail::check(coloc_cuda_memcpy_async(tg.device(), tg.stream(), &per[3 * t],
                                         bufs[t]->p, 3 * sizeof(double)),
                    "coloc_stream: err sums");
            }
            sync();
            for (int j = 0; j < 3; ++j)
            {
                sums[j] = 0.0;
                for (std::size_t t = 0; t < nt; ++t)
                    sums[j] += per[3 * t + std::size_t(j)];
            }
            last_reduction_ = "host";
        }
        // One process per GPU: the per-process sums are summed over the
        // ranks by NCCL on the first target's stream (the library's own
        // communicator; coloc_stream_set_comm).
        if (rank_comm_)
        {
            auto const& t0 = targets_.front();
            auto* d = static_cast<double*>(bufs[0]->p);
            int st = coloc_cuda_memcpy_async(t0.device(), t0.stream(), d, sums, 3 * sizeof(double));
            if (st == COLOC_OK)
                st = coloc_cuda_nccl_allreduce_f64(rank_comm_, t0.device(), t0.stream(), d, d, 3,
                    COLOC_REDUCE_SUM);
            if (st == COLOC_OK)
                st = coloc_cuda_memcpy_async(t0.device(), t0.stream(), sums, d, 3 * sizeof(double));
            if (st == COLOC_OK)
                st = coloc_cuda_stream_sync(t0.device(), t0.stream());
            coloc::detail::check(st, "coloc_stream: cross-rank ncclAllReduce");
            last_reduction_ = last_reduction_[0] == 'n' ? "nccl+ranks" : "host+ranks";
        }
        if (dev_out)
        {
            auto const& t0 = targets_.front();
            coloc::detail::check(coloc_cuda_memcpy_async(t0.device(), t0.stream(), dev_out,
                                     sums, 3 * sizeof(double)),
                "coloc_stream: err sums out");
            t0.synchronize();
        }
    }

    void checksums(std::uint64_t out[3]) override
    {
        vec_t const* v[3] = {&a_, &b_, &c_};
        for (int k = 0; k < 3; ++k)
        {
            std::uint64_t total = 0;
            for (auto const& s : v[k]->data_handle().segments())
            {
                if (s.length == 0)
                    continue;
                void* buf = nullptr;
                coloc::detail::check(coloc_cuda_malloc(s.where.device(), 8, &buf),
                    "coloc_stream: checksum buffer");
                std::uint64_t zero = 0, got = 0;
                int st = coloc_cuda_memcpy_async(s.where.device(), s.where.stream(), buf, &zero, 8);
                if (st == COLOC_OK)
                    st = coloc_cuda_checksum(s.where.device(), s.where.stream(), s.base, s.length,
                        sizeof(T), cfg_.first + s.offset, static_cast<std::uint64_t*>(buf));
                if (st == COLOC_OK)
                    st = coloc_cuda_memcpy_async(s.where.device(), s.where.stream(), &got, buf, 8);
                if (st == COLOC_OK)
                    st = coloc_cuda_stream_sync(s.where.device(), s.where.stream());
                (void) coloc_cuda_free(s.where.device(), buf);
                coloc::detail::check(st, "coloc_stream: checksum");
                total += got;
            }
            out[k] = total;
        }
    }

    void read(int k, std::uint64_t first, std::uint64_t n, void* out) override
    {
        vec_t& v = k == 0 ? a_ : k == 1 ? b_ : c_;
        if (k < 0 || k > 2 || first + n > v.size())
            throw std::invalid_argument("coloc_stream_read: range out of bounds");
        auto it = v.begin() + std::ptrdiff_t(first);
        coloc::copy(coloc::par.on(exec_), it, it + std::ptrdiff_t(n), static_cast<T*>(out));
        // with a stream-ordered executor the copy is only enqueued: the
        // header promises the elements are in `out` on return
        exec_.drain();
    }

    void set_comm(void* comm) override { rank_comm_ = comm; }
    char const* reduction() const override { return last_reduction_; }

private:
    // Host arrays of the e2e step: pinned (coloc_cuda_host_alloc) or, with
    // host_buffers == 2, ordinary pageable memory as a reference user's
    // std::vector would be (copies then go through the staging ring).
    struct host_free
    {
        bool pinned = true;
        void operator()(T* p) const noexcept
        {
            if (pinned)
                (void) coloc_cuda_host_free(p);
            else
                delete[] p;
        }
    };
    using pinned_ptr = std::unique_ptr<T, host_free>;

    static pinned_ptr host_array(std::size_t n, bool pinned)
    {
        if (!pinned)
            return pinned_ptr(new T[n], host_free{false});
        void* p = nullptr;
        coloc::detail::check(coloc_cuda_host_alloc(n * sizeof(T), &p), "coloc_stream: pinned host buffer");
        return pinned_ptr(static_cast<T*>(p), host_free{true});
    }

    static std::vector<coloc::cuda::target> make_targets(coloc_stream_config const& cfg)
    {
        if (cfg.ntargets <= 0 || !cfg.devices)
            throw std::invalid_argument("coloc_stream: need at least one target");
        return coloc::cuda::make_targets(std::vector<int>(cfg.devices, cfg.devices + cfg.ntargets));
    }

    vec_t make(unsigned k)
    {
        std::size_t const n = std::size_t(cfg_.count);
        if (cfg_.init == COLOC_STREAM_INIT_RANDOM)
            return vec_t::generate(n, coloc::ops::uniform_random<T>{cfg_.seed, k, cfg_.first},
                alloc_);
        T const init[3] = {T(1.0), T(2.0), T(0.0)};
        return vec_t(n, init[k], alloc_);
    }

    static event_pair new_pair(coloc::cuda::target const& t)
    {
        event_pair e{t.device()};
        coloc::detail::check(coloc_cuda_event_create(t.device(), &e.start), "event_create");
        coloc::detail::check(coloc_cuda_event_create(t.device(), &e.stop), "event_create");
        return e;
    }

    // Events on every target, slot (kernel k, target t) = k*nt + t.
    // Kernel k of an iteration is bracketed by boundary events k and k+1 on
    // every target; consecutive kernels share the boundary between them, so
    // an iteration records 5 events per target instead of 8 (fewer event
    // nodes between dependent kernels).
    void mark(std::vector<event_pair>* ev, int k, bool start)
    {
        if (!ev)
            return;
        std::size_t const nt = targets_.size();
        if (start)
        {
            for (std::size_t t = 0; t < nt; ++t)
            {
                event_pair e{targets_[t].device()};
                if (k == 0)
                {
                    coloc::detail::check(coloc_cuda_event_create(e.dev, &e.start), "event_create");
                    stamp(t, e.start);
                }
                else
                    e.start = (*ev)[std::size_t(k - 1) * nt + t].stop;
                coloc::detail::check(coloc_cuda_event_create(e.dev, &e.stop), "event_create");
                ev->push_back(e);
            }
            return;
        }
        for (std::size_t t = 0; t < nt; ++t)
            stamp(t, (*ev)[std::size_t(k) * nt + t].stop);
    }

    // record mode 4: k iterations with every kernel's in-kernel span
    // (earliest CTA start to latest CTA end, %globaltimer; kernels.cu
    // coloc_cuda_span_*), no event anywhere in the chain.  Per iteration and
    // kernel the max over targets is kept; an empty records_ entry keeps
    // the iteration numbering shared with the event modes.
    void iterate_spans(int k, bool graph)
    {
        std::size_t const nt = targets_.size();
        auto body = [&] {
            std::size_t opened = 0;
            try
            {
                for (; opened < nt; ++opened)
                    coloc::detail::check(coloc_cuda_span_begin(targets_[opened].device(),
                                             targets_[opened].stream(), 4 * k),
                        "span_begin");
                for (int i = 0; i < k; ++i)
                    iterate(0);
            }
            catch (...)
            {
                for (std::size_t t = 0; t < opened; ++t)
                    (void) coloc_cuda_span_end(targets_[t].device(), targets_[t].stream(), nullptr);
                throw;
            }
            for (std::size_t t = 0; t < nt; ++t)
            {
                int used = 0;
                coloc::detail::check(coloc_cuda_span_end(targets_[t].device(), targets_[t].stream(), &used),
                    "span_end");
                if (used != 4 * k)
                    throw std::invalid_argument("coloc_stream: in-kernel spans need the LDG/STG kernels "
                                                "(one elementwise launch per kernel and target)");
            }
        };
        if (graph && !cfg_.synchronous)
            capture(body);
        else
            body();
        sync();
        std::vector<std::array<double, 4>> rows(std::size_t(k), {0, 0, 0, 0});
        std::vector<double> ms(4 * std::size_t(k));
        for (std::size_t t = 0; t < nt; ++t)
        {
            coloc::detail::check(coloc_cuda_span_read(targets_[t].device(), targets_[t].stream(), ms.data(),
                                     4 * k),
                "span_read");
            for (int i = 0; i < k; ++i)
                for (int j = 0; j < 4; ++j)
                    rows[std::size_t(i)][std::size_t(j)] =
                        std::max(rows[std::size_t(i)][std::size_t(j)], ms[4 * std::size_t(i) + std::size_t(j)]);
        }
        for (auto const& r : rows)
        {
            span_rows_[records_.size()] = r;
            records_.emplace_back();
        }
    }

    // Records a timing event after the work queued on target t: on the
    // target's stream, or (record mode 3) on its side stream.
    void stamp(std::size_t t, void* event)
    {
        auto const& tg = targets_[t];
        if (!side_stamps_)
        {
            coloc::detail::check(coloc_cuda_event_record(tg.device(), event, tg.stream()),
                "coloc_stream: event record");
            return;
        }
        if (side_.size() < targets_.size())
            side_.resize(targets_.size(), nullptr);
        if (!side_[t])
            coloc::detail::check(coloc_cuda_stream_create(tg.device(), &side_[t]), "side stream");
        coloc::detail::check(coloc_cuda_stream_fork_timestamp(tg.device(), tg.stream(), side_[t], event),
            "coloc_stream: side timestamp");
        side_used_ = true;
    }

    // Side streams rejoin their targets' streams (before a capture ends,
    // and so that sync() covers the timing records).
    void join_sides()
    {
        if (!side_used_)
            return;
        for (std::size_t t = 0; t < side_.size(); ++t)
            if (side_[t])
                coloc::detail::check(coloc_cuda_stream_join(targets_[t].device(), targets_[t].stream(),
                                         side_[t]),
                    "coloc_stream: side join");
        side_used_ = false;
    }

    // iterate c=a; b=s*c; c=a+b; a=b+s*c from (1,2,0) in T.
    void expected_values(double out[3]) const
    {
        T a = 1, b = 2, c = 0;
        T const s = T(cfg_.scalar);
        for (int k = 0; k < iterations_; ++k)
        {
            c = a;
            b = s * c;
            c = a + b;
            T volatile t = s * c;
            a = b + t;
        }
        out[0] = double(a);
        out[1] = double(b);
        out[2] = double(c);
    }

    // Automatic chains (cfg.chain == 2): only where they were measured to
    // win -- per-target arrays from ~1 to 16 L2 sizes (128 MiB - 1 GiB on
    // B200: +0.5-4.6% per iteration; below, in the L2 regime, they lose;
    // above, neutral; profiles/r02_sweep_c5_1gpu_chain.jsonl).
    bool chain_pays() const
    {
        coloc_cuda_device_info info{};
        if (coloc_cuda_device_info_get(targets_.front().device(), &info) != COLOC_OK || !info.l2_bytes)
            return false;
        double const block = double(cfg_.count) / double(targets_.size()) * double(sizeof(T));
        double const l2 = double(info.l2_bytes);
        return block >= 0.95 * l2 && block <= 16.0 * l2;
    }

    bool distinct_devices() const
    {
        for (std::size_t i = 0; i < targets_.size(); ++i)
            for (std::size_t j = 0; j < i; ++j)
                if (targets_[i].device() == targets_[j].device())
                    return false;
        return true;
    }

    // Captures what fn() enqueues on every target's stream into one graph
    // per target, then launches the graphs (graphs_ keeps them until the
    // next sync).
    template <typename F>
    void capture(F&& fn)
    {
        launch_graphs(capture_graphs(std::forward<F>(fn)));
    }

    void launch_graphs(std::vector<void*> const& made)
    {
        for (std::size_t i = 0; i < made.size(); ++i)
            coloc::detail::check(coloc_cuda_graph_launch(targets_[i].device(), made[i],
                                     targets_[i].stream()),
                "coloc_stream: graph launch");
    }

    template <typename F>
    std::vector<void*> capture_graphs(F&& fn)
    {
        std::size_t begun = 0;
        auto abort = [&] {
            std::vector<int> devs;
            std::vector<void*> streams, broken(begun, nullptr);
            for (std::size_t i = 0; i < begun; ++i)
            {
                devs.push_back(targets_[i].device());
                streams.push_back(targets_[i].stream());
            }
            (void) coloc_cuda_graph_capture_end_many(int(begun), devs.data(), streams.data(),
                broken.data());
            for (std::size_t i = 0; i < begun; ++i)
                (void) coloc_cuda_graph_destroy(targets_[i].device(), broken[i]);
        };
        try
        {
            for (; begun < targets_.size(); ++begun)
                coloc::detail::check(coloc_cuda_graph_capture_begin(targets_[begun].device(),
                                         targets_[begun].stream()),
                    "coloc_stream: graph capture");
            fn();
        }
        catch (...)
        {
            abort();
            throw;
        }
        std::vector<int> devs;
        std::vector<void*> streams, made(targets_.size(), nullptr);
        for (auto const& t : targets_)
        {
            devs.push_back(t.device());
            streams.push_back(t.stream());
        }
        coloc::detail::check(coloc_cuda_graph_capture_end_many(int(targets_.size()), devs.data(),
                                 streams.data(), made.data()),
            "coloc_stream: graph instantiate");
        for (std::size_t i = 0; i < made.size(); ++i)
            graphs_.push_back({targets_[i].device(), made[i]});
        return made;
    }

    void release_graphs() noexcept
    {
        for (auto const& g : graphs_)
            (void) coloc_cuda_graph_destroy(g.first, g.second);
        graphs_.clear();
    }

    coloc_stream_config cfg_;
    std::vector<coloc::cuda::target> targets_;
    alloc_t alloc_;
    coloc::cuda_block_executor exec_;
    vec_t a_, b_, c_;
    pinned_ptr host_in_[3], host_out_[3];
    std::vector<std::vector<event_pair>> records_;
    std::vector<std::pair<int, void*>> graphs_;    // (device, graph) replayed, destroyed after the next sync
    std::vector<void*> comms_;     // NCCL communicators (one per GPU), lazily created
    char const* last_reduction_ = "none";
    void* rank_comm_ = nullptr;    // cross-process communicator (not owned)
    std::vector<void*> side_;      // per-target side streams of record mode 3
    std::map<std::size_t, std::array<double, 4>> span_rows_;    // record mode 4 rows by index
    bool side_stamps_ = false;
    bool side_used_ = false;
    int iterations_ = 0;
};

// ---------------------------------------------------------------------
// Abstraction vs native: blocking calls timed with the host clock
// (the paper's own timing of its CUDA port).
// ---------------------------------------------------------------------

template <typename T>
void summarize(std::vector<double> const (&times)[4], coloc_stream_timing* out)
{
    for (int k = 0; k < 4; ++k)
    {
        auto const& t = times[k];
        std::size_t const skip = t.size() > 1 ? 1 : 0;    // first iteration excluded
        double mn = 1e300, mx = 0, sum = 0;
        for (std::size_t i = skip; i < t.size(); ++i)
        {
            mn = std::min(mn, t[i]);
            mx = std::max(mx, t[i]);
            sum += t[i];
        }
        out->min_s[k] = mn;
        out->max_s[k] = mx;
        out->avg_s[k] = sum / double(t.size() - skip);
    }
}

template <typename T>
void validate_host(T const* const (&arrays)[3], std::size_t n, int iterations, coloc_stream_timing* out)
{
    T ea = 1, eb = 2, ec = 0;
    T const s = T(3.0);
    for (int k = 0; k < iterations; ++k)
    {
        ec = ea;
        eb = s * ec;
        ec = ea + eb;
        T volatile t = s * ec;
        ea = eb + t;
    }
    T const want[3] = {ea, eb, ec};
    double worst = 0;
    for (int j = 0; j < 3; ++j)
        for (std::size_t i = 0; i < n; ++i)
            if (arrays[j][i] != want[j])
                worst = std::max(worst,
                    std::fabs(double(arrays[j][i]) - double(want[j])) / std::fabs(double(want[j])));
    out->max_rel_err = worst;
    out->validated = worst <= (sizeof(T) == 8 ? 1e-8 : 1e-6) ? 1 : 0;
}

template <typename T>
void blocking_run(int arm, int dev, std::size_t n, int iterations, coloc_stream_timing* out)
{
    using clock = std::chrono::steady_clock;
    std::vector<double> times[4];
    T const s = T(3.0);
    std::vector<T> host[3];
    for (auto& h : host)
        h.resize(n);
    auto tick = [&](int k, auto&& call) {
        auto t0 = clock::now();
        call();
        times[k].push_back(std::chrono::duration<double>(clock::now() - t0).count());
    };
    if (arm == COLOC_STREAM_ARM_DROPIN)
    {
        // Listing 4 exactly as a reference user writes it, with the
        // reference's blocking executor semantics.
        auto targets = coloc::cuda::make_targets(std::vector<int>{dev});
        coloc::cuda::block_allocator<T> alloc(targets);
        coloc::cuda_block_executor exec(targets, coloc::executor_options{true});
        using vec = coloc::vector<T, coloc::cuda::block_allocator<T>>;
        vec a(n, T(1.0), alloc), b(n, T(2.0), alloc), c(n, T(0.0), alloc);
        auto policy = coloc::par.on(exec);
        for (int it = 0; it < iterations; ++it)
        {
            tick(0, [&] { coloc::copy(policy, a.begin(), a.end(), c.begin()); });
            tick(1, [&] { coloc::transform(policy, c.begin(), c.end(), b.begin(), coloc::ops::scale<T>{s}); });
            tick(2, [&] { coloc::transform(policy, a.begin(), a.end(), b.begin(), c.begin(), coloc::ops::plus<T>{}); });
            tick(3, [&] {
                coloc::transform(policy, b.begin(), b.end(), c.begin(), a.begin(), coloc::ops::triad<T>{s});
            });
        }
        coloc::copy(policy, a.begin(), a.end(), host[0].data());
        coloc::copy(policy, b.begin(), b.end(), host[1].data());
        coloc::copy(policy, c.begin(), c.end(), host[2].data());
    }
    else if (arm == COLOC_STREAM_ARM_CABI)
    {
        using coloc::detail::check;
        void* stream = nullptr;
        check(coloc_cuda_stream_create(dev, &stream), "stream_create");
        void* p[3] = {nullptr, nullptr, nullptr};
        auto cleanup = [&] {
            for (void* q : p)
                (void) coloc_cuda_free(dev, q);
            (void) coloc_cuda_stream_destroy(dev, stream);
        };
        try
        {
            T const init[3] = {T(1.0), T(2.0), T(0.0)};
            for (int j = 0; j < 3; ++j)
            {
                check(coloc_cuda_malloc(dev, n * sizeof(T), &p[j]), "malloc");
                check(coloc_cuda_fill(dev, stream, p[j], n, &init[j], sizeof(T)), "fill");
            }
            check(coloc_cuda_stream_sync(dev, stream), "sync");
            auto* a = static_cast<T*>(p[0]);
            auto* b = static_cast<T*>(p[1]);
            auto* c = static_cast<T*>(p[2]);
            auto done = [&](int st) {
                check(st, "kernel");
                check(coloc_cuda_stream_sync(dev, stream), "sync");
            };
            for (int it = 0; it < iterations; ++it)
            {
                if constexpr (std::is_same_v<T, double>)
                {
                    tick(0, [&] { done(coloc_cuda_copy_f64(dev, stream, c, a, n)); });
                    tick(1, [&] { done(coloc_cuda_scale_f64(dev, stream, b, c, s, n)); });
                    tick(2, [&] { done(coloc_cuda_add_f64(dev, stream, c, a, b, n)); });
                    tick(3, [&] { done(coloc_cuda_triad_f64(dev, stream, a, b, c, s, n, 0)); });
                }
                else
                {
                    tick(0, [&] { done(coloc_cuda_copy_f32(dev, stream, c, a, n)); });
                    tick(1, [&] { done(coloc_cuda_scale_f32(dev, stream, b, c, s, n)); });
                    tick(2, [&] { done(coloc_cuda_add_f32(dev, stream, c, a, b, n)); });
                    tick(3, [&] { done(coloc_cuda_triad_f32(dev, stream, a, b, c, s, n, 0)); });
                }
            }
            for (int j = 0; j < 3; ++j)
                check(coloc_cuda_memcpy_async(dev, stream, host[j].data(), p[j], n * sizeof(T)), "read back");
            check(coloc_cuda_stream_sync(dev, stream), "sync");
        }
        catch (...)
        {
            cleanup();
            throw;
        }
        cleanup();
    }
    else
        throw std::invalid_argument("coloc_stream_blocking_run: unknown arm");
    summarize<T>(times, out);
    T const* arrays[3] = {host[0].data(), host[1].data(), host[2].data()};
    validate_host<T>(arrays, n, iterations, out);
}

run_base* as_run(void* h)
{
    if (!h)
        throw std::invalid_argument("coloc_stream: null handle");
    return static_cast<run_base*>(h);
}

}    // namespace

extern "C" {

const char* coloc_stream_last_error(void)
{
    return t_error.c_str();
}

int coloc_stream_create(const coloc_stream_config* cfg, void** handle)
{
    return guarded([&] {
        if (!cfg || !handle)
            throw std::invalid_argument("coloc_stream_create: null argument");
        *handle = nullptr;
        if (cfg->dtype == COLOC_STREAM_F64)
            *handle = static_cast<run_base*>(new stream_run<double>(*cfg));
        else if (cfg->dtype == COLOC_STREAM_F32)
            *handle = static_cast<run_base*>(new stream_run<float>(*cfg));
        else
            throw std::invalid_argument("coloc_stream_create: unknown dtype");
    });
}

int coloc_stream_destroy(void* handle)
{
    return guarded([&] { delete static_cast<run_base*>(handle); });
}

int coloc_stream_iterate(void* handle, int record)
{
    return guarded([&] {
        if (record < 0 || record > 4)
            throw std::invalid_argument("coloc_stream_iterate: record must be 0..4");
        if (record == 4)
            as_run(handle)->iterate_many(1, 4, false);
        else
            as_run(handle)->iterate(record);
    });
}

int coloc_stream_iterate_many(void* handle, int iterations, int record, int graph)
{
    return guarded([&] {
        if (record < 0 || record > 4)
            throw std::invalid_argument("coloc_stream_iterate_many: record must be 0..4");
        as_run(handle)->iterate_many(iterations, record, graph != 0);
    });
}

int coloc_stream_sync(void* handle)
{
    return guarded([&] { as_run(handle)->sync(); });
}

int coloc_stream_recorded(void* handle, int* count)
{
    return guarded([&] { *count = as_run(handle)->recorded(); });
}

int coloc_stream_kernel_ms(void* handle, int i, double ms[4])
{
    return guarded([&] {
        auto r = as_run(handle)->kernel_ms(i);
        std::memcpy(ms, r.data(), sizeof(double) * 4);
    });
}

int coloc_stream_iteration_ms(void* handle, int i, double* ms)
{
    return guarded([&] { *ms = as_run(handle)->iteration_ms(i); });
}

void coloc_stream_clear_records(void* handle)
{
    (void) guarded([&] { as_run(handle)->clear_records(); });
}

int coloc_stream_iterations(void* handle, int* count)
{
    return guarded([&] { *count = as_run(handle)->iterations(); });
}

int coloc_stream_e2e_step(void* handle, int ntimes, double* ms)
{
    return guarded([&] { *ms = as_run(handle)->e2e_step(ntimes); });
}

int coloc_stream_err_sums(void* handle, double expected[3], double sums[3], double* dev_out)
{
    return guarded([&] { as_run(handle)->err_sums(expected, sums, dev_out); });
}

int coloc_stream_checksums(void* handle, uint64_t out[3])
{
    return guarded([&] { as_run(handle)->checksums(out); });
}

int coloc_stream_read(void* handle, int k, uint64_t first, uint64_t n, void* out)
{
    return guarded([&] { as_run(handle)->read(k, first, n, out); });
}

int coloc_stream_set_comm(void* handle, void* comm)
{
    return guarded([&] { as_run(handle)->set_comm(comm); });
}

const char* coloc_stream_reduction(void* handle)
{
    try
    {
        return as_run(handle)->reduction();
    }
    catch (...)
    {
        return "";
    }
}

int coloc_stream_blocking_run(int arm, int dtype, int dev, uint64_t n, int iterations,
    coloc_stream_timing* out)
{
    return guarded([&] {
        if (!out || iterations < 1)
            throw std::invalid_argument("coloc_stream_blocking_run: bad arguments");
        if (dtype == COLOC_STREAM_F64)
            blocking_run<double>(arm, dev, std::size_t(n), iterations, out);
        else if (dtype == COLOC_STREAM_F32)
            blocking_run<float>(arm, dev, std::size_t(n), iterations, out);
        else
            throw std::invalid_argument("coloc_stream_blocking_run: unknown dtype");
    });
}

uint64_t coloc_stream_launch_count(void)
{
    return coloc_cuda_launch_count();
}

}    // extern "C"
