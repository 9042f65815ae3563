// test_api.cpp -- tests of the C++ drop-in API, written the way a user of
// the reference would write them (SPEC.md acceptance criteria 4, 5, 7, 8).
//
//   test_api --cpu   host-side logic only (partition, shapes, policies,
//                    executor_traits derivation, error mapping without a GPU)
//   test_api --gpu   the same API on real device data (needs a GPU)
//
// Exit code 0 when every selected test passes.
#include "coloc_b200/coloc.hpp"

#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <numeric>
#include <random>
#include <string>
#include <thread>
#include <vector>

namespace {

int g_failed = 0;
int g_run = 0;

#define EXPECT(cond)                                                              \
    do                                                                            \
    {                                                                             \
        if (!(cond))                                                              \
        {                                                                         \
            std::fprintf(stderr, "  FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            throw std::runtime_error("expectation failed");                       \
        }                                                                         \
    } while (0)

void run(char const* name, std::function<void()> const& fn)
{
    ++g_run;
    try
    {
        fn();
        std::printf("ok   %s\n", name);
    }
    catch (std::exception const& e)
    {
        ++g_failed;
        std::printf("FAIL %s: %s\n", name, e.what());
    }
}

template <typename E, typename F>
bool throws(F&& f)
{
    try
    {
        f();
    }
    catch (E const&)
    {
        return true;
    }
    catch (...)
    {
        return false;
    }
    return false;
}

// A minimal executor implementing only async_execute (SPEC criterion 5).
struct inline_executor
{
    template <typename F, typename... Ts>
    auto async_execute(F&& f, Ts&&... ts)
    {
        using R = std::invoke_result_t<F&, Ts&...>;
        std::packaged_task<R()> task([&] { return std::invoke(f, ts...); });
        auto fut = task.get_future();
        task();
        return fut;
    }
};

// ---------------------------------------------------------------- CPU tests

void cpu_tests()
{
    run("partition_block matches SPEC examples", [] {
        auto p = coloc::partition_block(10, std::vector<int>{0, 1, 2});
        EXPECT(p.blocks.size() == 3);
        EXPECT(p.blocks[0].offset == 0 && p.blocks[0].length == 4);
        EXPECT(p.blocks[1].offset == 4 && p.blocks[1].length == 3);
        EXPECT(p.blocks[2].offset == 7 && p.blocks[2].length == 3);
        auto q = coloc::partition_block(2, std::vector<int>{0, 1, 2});
        EXPECT(q.blocks[2].length == 0 && q.blocks[2].offset == 2);
        EXPECT(throws<std::invalid_argument>([] { coloc::partition_block(1, std::vector<int>{}); }));
    });

    run("partition exhaustive n<=10^4 (sampled) k<=16", [] {
        for (std::size_t k = 1; k <= 16; ++k)
        {
            std::vector<int> t(k);
            for (std::size_t n = 0; n <= 10000; n += (n < 500 ? 1 : 37))
            {
                auto p = coloc::partition_block(n, t);
                std::size_t at = 0, mn = ~std::size_t(0), mx = 0;
                for (auto const& b : p.blocks)
                {
                    EXPECT(b.offset == at);
                    at += b.length;
                    mn = std::min(mn, b.length);
                    mx = std::max(mx, b.length);
                }
                EXPECT(at == n && p.total() == n && mx - mn <= 1);
                for (std::size_t i = 0; i < n; i += 1 + n / 50)
                {
                    std::size_t b = p.block_of(i);
                    EXPECT(b != coloc::no_block);
                    EXPECT(p.blocks[b].offset <= i && i < p.blocks[b].end());
                }
                EXPECT(p.block_of(n) == coloc::no_block);
            }
        }
    });

    run("chunk_range ceil-first", [] {
        coloc::shape s;
        coloc::chunk_range(s, 0, 10, 3, 7);
        EXPECT(s.size() == 3 && s[0].size() == 4 && s[1].size() == 3 && s[2].end == 10);
        EXPECT(s[0].block == 7 && coloc::shape_size(s) == 10);
        coloc::shape t;
        coloc::chunk_range(t, 5, 7, 100);
        EXPECT(t.size() == 2);
        EXPECT(coloc::single_range(0).empty() && coloc::single_range(5).size() == 1);
    });

    run("executor_traits derives everything from async_execute", [] {
        inline_executor ex;
        using traits = coloc::executor_traits<inline_executor>;
        EXPECT(traits::execute(ex, [] { return 41 + 1; }) == 42);
        std::vector<int> hits(1000, 0);
        std::mt19937 rng(7);
        for (int trial = 0; trial < 200; ++trial)
        {
            std::fill(hits.begin(), hits.end(), 0);
            coloc::shape s;
            std::size_t at = 0;
            while (at < hits.size())
            {
                std::size_t len = 1 + rng() % 97;
                len = std::min(len, hits.size() - at);
                s.push_back({at, at + len});
                at += len;
            }
            std::shuffle(s.begin(), s.end(), rng);
            traits::bulk_execute(ex, [&](std::size_t i) { hits[i] += 1; }, s);
            EXPECT(std::all_of(hits.begin(), hits.end(), [](int h) { return h == 1; }));
        }
        // first error wins and propagates
        bool threw = throws<std::runtime_error>([&] {
            traits::bulk_execute(ex,
                [](std::size_t i) {
                    if (i == 3)
                        throw std::runtime_error("boom");
                },
                coloc::shape{{0, 5}, {5, 9}});
        });
        EXPECT(threw);
        int applied = 0;
        traits::apply_execute(ex, [&] { ++applied; });
        EXPECT(applied == 1);
    });

    run("apply error hook receives fire-and-forget errors", [] {
        inline_executor ex;
        int seen = 0;
        coloc::set_apply_error_hook([&](std::exception_ptr) { ++seen; });
        coloc::executor_traits<inline_executor>::apply_execute(ex, [] { throw std::runtime_error("x"); });
        coloc::set_apply_error_hook({});
        EXPECT(seen == 1);
    });

    run("named ops have the reference's host arithmetic", [] {
        EXPECT(coloc::ops::scale<double>{3.0}(2.0) == 6.0);
        EXPECT(coloc::ops::plus<double>{}(1.0, 2.0) == 3.0);
        EXPECT(coloc::ops::triad<double>{3.0}(2.0, 1.0) == 5.0);
        EXPECT(coloc::ops::to_upper{}('h') == 'H' && coloc::ops::to_upper{}('!') == '!');
        double x = 2.0;
        coloc::ops::multiply_by<double>{3.0}(x);
        EXPECT(x == 6.0);
        // generator restates the oracle's first value for seed 0x220606302
        coloc::ops::uniform_random<double> g{0x220606302ULL, 0, 0};
        double v = g(0);
        EXPECT(v >= -1.0 && v < 1.0);
    });

    run("no GPU: targets fail loudly with invalid_target_error", [] {
        if (coloc::cuda::device_count() > 0)
            return;
        EXPECT(coloc::cuda::get_targets().empty());
        EXPECT(throws<coloc::invalid_target_error>([] { coloc::cuda::target t(0); }));
        EXPECT(throws<coloc::invalid_target_error>(
            [] { coloc::cuda::block_allocator<double> a(std::vector<coloc::cuda::target>{}); }));
        EXPECT(throws<coloc::invalid_target_error>(
            [] { coloc::cuda_block_executor e(std::vector<coloc::cuda::target>{}); }));
    });
}

// ---------------------------------------------------------------- GPU tests

template <typename T>
using dvec = coloc::vector<T, coloc::cuda::block_allocator<T>>;

template <typename T>
std::vector<T> to_host(dvec<T> const& v)
{
    std::vector<T> h(v.size());
    coloc::copy(coloc::par, v.begin(), v.end(), h.data());
    return h;
}

void gpu_tests()
{
    using namespace coloc;
    int const ngpu = cuda::device_count();
    std::printf("# %d GPU(s): %s\n", ngpu, ngpu ? cuda::device_info(0).name : "");
    EXPECT(ngpu >= 1);

    // Several targets on GPU 0 (own streams) exercise the block logic on a
    // one-GPU box; on bigger boxes the GPUs themselves are used.
    std::vector<int> devs = ngpu >= 2 ? std::vector<int>{0, 1} : std::vector<int>{0, 0, 0};
    auto targets = cuda::make_targets(devs);

    run("listing 4 on a block-partitioned vector", [&] {
        cuda::block_allocator<double> alloc(targets);
        cuda_block_executor exec(targets);
        std::size_t const n = 1'000'003;
        dvec<double> as(n, 1.0, alloc), bs(n, 2.0, alloc), cs(n, 0.0, alloc);
        EXPECT(as.distribution().size() == targets.size());
        double const scalar = 3.0;
        for (int k = 0; k < 10; ++k)
        {
            copy(par.on(exec), as.begin(), as.end(), cs.begin());
            transform(par.on(exec), cs.begin(), cs.end(), bs.begin(), ops::scale<double>{scalar});
            transform(par.on(exec), as.begin(), as.end(), bs.begin(), cs.begin(), ops::plus<double>{});
            transform(par.on(exec), bs.begin(), bs.end(), cs.begin(), as.begin(), ops::triad<double>{scalar});
        }
        auto a = to_host(as), b = to_host(bs), c = to_host(cs);
        for (std::size_t i = 0; i < n; i += 997)
            EXPECT(a[i] == 576650390625.0 && b[i] == 115330078125.0 && c[i] == 153773437500.0);
        EXPECT(a[n - 1] == 576650390625.0);
    });

    run("transform/copy equal a sequential loop (random inputs, 1-3 targets)", [&] {
        std::mt19937_64 rng(11);
        for (std::size_t nt = 1; nt <= 3; ++nt)
            for (std::size_t n : {std::size_t(0), std::size_t(1), std::size_t(7), std::size_t(1000),
                     std::size_t(100000)})
            {
                std::vector<cuda::target> ts(targets.begin(), targets.begin() + std::min(nt, targets.size()));
                cuda::block_allocator<double> alloc(ts);
                std::vector<double> hb(n), hc(n);
                std::uniform_real_distribution<double> u(-1, 1);
                for (auto& x : hb)
                    x = u(rng);
                for (auto& x : hc)
                    x = u(rng);
                dvec<double> b(n, 0.0, alloc), c(n, 0.0, alloc), out(n, 0.0, alloc);
                copy(par, hb.begin(), hb.end(), b.begin());
                copy(par, hc.begin(), hc.end(), c.begin());
                transform(par, b.begin(), b.end(), c.begin(), out.begin(), ops::triad<double>{3.0});
                auto got = to_host(out);
                for (std::size_t i = 0; i < n; ++i)
                {
                    double volatile t = hc[i] * 3.0;
                    EXPECT(got[i] == hb[i] + t);
                }
                transform(seq, c.begin(), c.end(), out.begin(), ops::scale<double>{3.0});
                got = to_host(out);
                for (std::size_t i = 0; i < n; ++i)
                    EXPECT(got[i] == hc[i] * 3.0);
            }
    });

    run("host->device->host round trip of 10^5 doubles is bitwise", [&] {
        cuda::block_allocator<double> alloc(targets);
        std::vector<double> src(100000);
        std::mt19937_64 rng(5);
        for (auto& x : src)
        {
            std::uint64_t bits = rng();
            std::memcpy(&x, &bits, 8);
        }
        dvec<double> d(src.size(), 0.0, alloc);
        auto end = copy(par, src.begin(), src.end(), d.begin());
        EXPECT(end == d.end());
        std::vector<double> back(src.size());
        copy(par, d.begin(), d.end(), back.data());
        EXPECT(std::memcmp(src.data(), back.data(), src.size() * 8) == 0);
    });

    run("H2D -> scale -> add -> D2H gives 0 4 8 ... 28 (SURVEY section 4 probe)", [&] {
        // the survey's mock-device probe on the real device path: iota on
        // the host, scale by 2 on the device, add the vector to itself
        cuda::block_allocator<double> alloc(targets);
        cuda_block_executor exec(targets);
        std::vector<double> h(8);
        std::iota(h.begin(), h.end(), 0.0);
        dvec<double> d(8, alloc), t(8, alloc);
        copy(par.on(exec), h.begin(), h.end(), d.begin());
        transform(par.on(exec), d.begin(), d.end(), t.begin(), ops::scale<double>{2.0});
        transform(par.on(exec), t.begin(), t.end(), t.begin(), d.begin(), ops::plus<double>{});
        std::vector<double> back(8);
        copy(par.on(exec), d.begin(), d.end(), back.data());
        for (int i = 0; i < 8; ++i)
            EXPECT(back[std::size_t(i)] == 4.0 * i);
    });

    run("std::vector round trip of 2^24+5 doubles (pinned staging path) is bitwise", [&] {
        // > 4 MiB per block: host copies of pageable memory are staged
        cuda::block_allocator<double> alloc(targets);
        std::vector<double> src((std::size_t(1) << 24) + 5);
        std::mt19937_64 rng(6);
        for (auto& x : src)
        {
            std::uint64_t bits = rng();
            std::memcpy(&x, &bits, 8);
        }
        dvec<double> d(src.size(), 0.0, alloc);
        copy(par, src.begin(), src.end(), d.begin());
        std::vector<double> back(src.size());
        copy(par, d.begin(), d.end(), back.data());
        EXPECT(std::memcmp(src.data(), back.data(), src.size() * 8) == 0);
        // sub-range at an odd offset
        std::vector<double> part(src.size() - 3);
        copy(par, d.begin() + 3, d.end(), part.data());
        EXPECT(std::memcmp(src.data() + 3, part.data(), part.size() * 8) == 0);
    });

    run("std::vector with cuda::pinned_allocator: stream-ordered round trip is bitwise", [&] {
        cuda::block_allocator<double> alloc(targets);
        cuda_block_executor exec(targets, executor_options{false});
        std::size_t const n = (std::size_t(1) << 23) + 3;
        std::vector<double, cuda::pinned_allocator<double>> h(n), back(n);
        for (std::size_t i = 0; i < n; ++i)
            h[i] = double(i) * 0.5 - 7.0;
        dvec<double> v(n, alloc);
        copy(par.on(exec), h.begin(), h.end(), v.begin());
        transform(par.on(exec), v.begin(), v.end(), v.begin(), ops::scale<double>{2.0});
        copy(par.on(exec), v.begin(), v.end(), back.data());
        exec.drain();
        for (std::size_t i = 0; i < n; ++i)
            EXPECT(back[i] == h[i] * 2.0);
    });

    run("integer vectors: int and uint64_t transforms equal a sequential loop", [&] {
        // the reference's transform is generic over T; the drop-in runs
        // int / long / unsigned vectors on the i32/i64 kernels (wrap-around)
        std::mt19937_64 rng(17);
        std::size_t const n = 100'003;
        {
            cuda::block_allocator<int> alloc(targets);
            std::vector<int> ha(n), hb(n);
            for (std::size_t i = 0; i < n; ++i)
            {
                ha[i] = int(std::uint32_t(rng()));
                hb[i] = int(std::uint32_t(rng()));
            }
            dvec<int> a(n, alloc), b(n, alloc), c(n, alloc);
            copy(par, ha.begin(), ha.end(), a.begin());
            copy(par, hb.begin(), hb.end(), b.begin());
            transform(par, a.begin(), a.end(), b.begin(), c.begin(), ops::plus<int>{});
            transform(par, c.begin(), c.end(), c.begin(), ops::scale<int>{7});
            transform(par, a.begin(), a.end(), c.begin(), b.begin(), ops::triad<int>{-3});
            std::vector<int> hc(n), hb2(n);
            copy(par, c.begin(), c.end(), hc.data());
            copy(par, b.begin(), b.end(), hb2.data());
            for (std::size_t i = 0; i < n; ++i)
            {
                std::uint32_t const sum = std::uint32_t(ha[i]) + std::uint32_t(hb[i]);
                std::uint32_t const sc = sum * 7u;
                EXPECT(hc[i] == int(sc));
                EXPECT(hb2[i] == int(std::uint32_t(ha[i]) + sc * std::uint32_t(-3)));
            }
        }
        {
            cuda::block_allocator<std::uint64_t> alloc(targets);
            std::vector<std::uint64_t> h(n);
            for (auto& x : h)
                x = rng();
            dvec<std::uint64_t> v(n, alloc), w(n, alloc);
            copy(par, h.begin(), h.end(), v.begin());
            transform(par, v.begin(), v.end(), v.begin(), w.begin(), std::plus<>{});
            for_each(par, w.begin(), w.end(), ops::multiply_by<std::uint64_t>{0x9E3779B97F4A7C15ull});
            std::vector<std::uint64_t> back(n);
            copy(par, w.begin(), w.end(), back.data());
            for (std::size_t i = 0; i < n; ++i)
                EXPECT(back[i] == (h[i] + h[i]) * 0x9E3779B97F4A7C15ull);
        }
    });

    run("mismatched partitions: shape follows the destination", [&] {
        cuda::block_allocator<double> a1(std::vector<cuda::target>{targets[0]});
        cuda::block_allocator<double> a3(targets);
        std::size_t const n = 50021;
        auto src = dvec<double>::generate(n, ops::iota<double>{0.0}, a1);
        dvec<double> dst(n, -1.0, a3);
        copy(par, src.begin(), src.end(), dst.begin());
        transform(par, dst.begin(), dst.end(), dst.begin(), ops::scale<double>{2.0});
        auto h = to_host(dst);
        for (std::size_t i = 0; i < n; ++i)
            EXPECT(h[i] == 2.0 * double(i));
    });

    run("sub-ranges at odd offsets", [&] {
        cuda::block_allocator<double> alloc(targets);
        std::size_t const n = 10007;
        auto a = dvec<double>::generate(n, ops::iota<double>{0.0}, alloc);
        dvec<double> b(n, 0.0, alloc);
        copy(par, a.begin() + 3, a.end() - 5, b.begin() + 1);
        auto h = to_host(b);
        EXPECT(h[0] == 0.0 && h[1] == 3.0 && h[n - 8] == double(n - 6) && h[n - 7] == 0.0);
        EXPECT(throws<std::invalid_argument>([&] { copy(par, a.begin(), a.begin() + 100, a.begin() + 50); }));
    });

    run("listing 3: hello world to upper", [&] {
        cuda::block_allocator<char> alloc(targets);
        vector<char, cuda::block_allocator<char>> s({'h', 'e', 'l', 'l', 'o', 'w', 'o', 'r', 'l', 'd'}, alloc);
        cuda_block_executor exec(targets);
        transform(par.on(exec), s.begin(), s.end(), s.begin(), ops::to_upper{});
        std::string out(s.size(), ' ');
        copy(par, s.begin(), s.end(), out.data());
        EXPECT(out == "HELLOWORLD");
        for_each(par.on(exec), s.begin(), s.end(), ops::assign<char>{'z'});
        copy(par, s.begin(), s.end(), out.data());
        EXPECT(out == "zzzzzzzzzz");
    });

    run("for_each and proxies are ordered on the owning stream", [&] {
        cuda::allocator<double> alloc(targets[0]);
        coloc::vector<double, cuda::allocator<double>> v(1000, 1.0, alloc);
        cuda_executor exec(targets[0], executor_options{false});    // stream-ordered
        for_each(par.on(exec), v.begin(), v.end(), ops::multiply_by<double>{3.0});
        v[5] = 42.0;                                 // proxy write after the kernel
        for_each(par.on(exec), v.begin(), v.end(), ops::multiply_by<double>{2.0});
        EXPECT(double(v[4]) == 6.0 && double(v[5]) == 84.0);
        EXPECT(v.at(999) == 6.0);
        EXPECT(throws<std::out_of_range>([&] { (void) double(v.at(1000)); }));
    });

    run("futures: bulk_async_execute and async_execute settle", [&] {
        cuda::block_allocator<double> alloc(targets);
        cuda_block_executor exec(targets, executor_options{false});
        dvec<double> v(1 << 20, 1.0, alloc);
        transform(par.on(exec), v.begin(), v.end(), v.begin(), ops::scale<double>{2.0});
        int seen = 0;
        auto f = exec.executor(0).async_execute([&] { return ++seen; });
        EXPECT(f.get() == 1);
        exec.drain();
        EXPECT(double(v[12345]) == 2.0);
    });

    run("device generators equal the host generator", [&] {
        cuda::block_allocator<float> alloc(targets);
        ops::uniform_random<float> g{0x220606302ULL, 2, 1000};
        auto v = coloc::vector<float, cuda::block_allocator<float>>::generate(4099, g, alloc);
        std::vector<float> h(v.size());
        copy(par, v.begin(), v.end(), h.data());
        for (std::size_t i = 0; i < h.size(); ++i)
            EXPECT(h[i] == g(i));
    });

    run("allocation failure is allocation_error naming the target", [&] {
        cuda::block_allocator<double> alloc(targets[0]);
        bool ok = false;
        try
        {
            dvec<double> huge(std::size_t(1) << 45, alloc);
        }
        catch (allocation_error const& e)
        {
            ok = e.requested_bytes() == (std::size_t(1) << 48) && e.place() == "cuda:0";
        }
        EXPECT(ok);
    });

    run("invalid device is invalid_target_error", [&] {
        EXPECT(throws<invalid_target_error>([] { cuda::target t(97); }));
    });

    run("first error wins on GPU launches: later ranges cancelled, both forms rethrow", [&] {
        // detail/bulk.hpp:67-91 (first-error-wins, remaining ranges not
        // run) at launch granularity: the range of block 1 fails to launch
        // (null destination -> COLOC_ERR_INVALID_ARGUMENT), block 0's fill
        // really runs on its stream, block 2's is never launched.
        std::vector<cuda::target> ts = cuda::make_targets(std::vector<int>{devs[0], devs[0], devs[0]});
        std::size_t const n = 3 * 4096;
        std::vector<double*> bufs(3, nullptr);
        for (int b = 0; b < 3; ++b)
        {
            void* p = nullptr;
            detail::check(coloc_cuda_malloc(ts[b].device(), 4096 * sizeof(double), &p), "malloc");
            bufs[std::size_t(b)] = static_cast<double*>(p);
            detail::check(coloc_cuda_fill_f64(ts[b].device(), ts[b].stream(), bufs[b], 4096, 0.0), "fill");
        }
        struct failing_fill
        {
            std::vector<double*>* bufs;
            std::vector<int>* launched;
            double value;
            void launch(cuda::target const& t, index_range const& r) const
            {
                (*launched)[r.block] += 1;
                double* dst = r.block == 1 ? nullptr : (*bufs)[r.block];
                detail::check(coloc_cuda_fill_f64(t.device(), t.stream(), dst, r.size(), value),
                    "fill range");
            }
        };
        shape s{{0, 4096, 0}, {4096, 8192, 1}, {8192, n, 2}};
        for (int form = 0; form < 2; ++form)
        {
            std::vector<int> launched(3, 0);
            double const v = 1.0 + form;
            cuda_block_executor exec(ts);
            failing_fill k{&bufs, &launched, v};
            bool threw = false;
            try
            {
                if (form == 0)
                    executor_traits<cuda_block_executor>::bulk_execute(exec, k, s);
                else
                    executor_traits<cuda_block_executor>::bulk_async_execute(exec, k, s).get();
            }
            catch (std::invalid_argument const&)
            {
                threw = true;
            }
            EXPECT(threw);
            EXPECT(launched[0] == 1 && launched[1] == 1 && launched[2] == 0);
            exec.drain();
            double got[3] = {-1, -1, -1};
            for (int b = 0; b < 3; ++b)
                detail::check(coloc_cuda_memcpy_async(ts[b].device(), ts[b].stream(), &got[b],
                                  bufs[std::size_t(b)] + 4095, sizeof(double)),
                    "read back");
            for (auto const& t : ts)
                t.synchronize();
            // block 0 ran (this form's value), blocks 1 and 2 were never written
            EXPECT(got[0] == v && got[1] == 0.0 && got[2] == 0.0);
        }
        for (int b = 0; b < 3; ++b)
            (void) coloc_cuda_free(ts[b].device(), bufs[std::size_t(b)]);
    });

    run("NCCL rank path through the C ABI alone (nranks = 1, the MPI form)", [&] {
        // id -> (any transport) -> init_rank ->
        // allreduce on the rank's stream; here one rank.
        char id[COLOC_NCCL_ID_BYTES];
        detail::check(coloc_cuda_nccl_unique_id(id, sizeof id), "nccl_unique_id");
        void* comm = nullptr;
        detail::check(coloc_cuda_nccl_init_rank(devs[0], 1, id, 0, &comm), "nccl_init_rank");
        auto const& t = targets[0];
        void* buf = nullptr;
        detail::check(coloc_cuda_malloc(t.device(), 4 * sizeof(double), &buf), "malloc");
        double h[4] = {1.5, -2.0, 7.25, 0.0};
        detail::check(coloc_cuda_memcpy_async(t.device(), t.stream(), buf, h, sizeof h), "upload");
        auto* d = static_cast<double*>(buf);
        for (int op : {COLOC_REDUCE_SUM, COLOC_REDUCE_MAX, COLOC_REDUCE_MIN})
            detail::check(coloc_cuda_nccl_allreduce_f64(comm, t.device(), t.stream(), d, d, 4, op),
                "nccl_allreduce_f64");
        double back[4] = {};
        detail::check(coloc_cuda_memcpy_async(t.device(), t.stream(), back, buf, sizeof back), "download");
        t.synchronize();
        for (int i = 0; i < 4; ++i)
            EXPECT(back[i] == h[i]);
        EXPECT(coloc_cuda_nccl_init_rank(devs[0], 1, id, 3, &comm) == COLOC_ERR_INVALID_ARGUMENT);
        (void) coloc_cuda_free(t.device(), buf);
        void* comms[1] = {comm};
        detail::check(coloc_cuda_nccl_destroy(1, comms), "nccl_destroy");
    });

    run("co-location audit: every launch runs on its block's target", [&] {
        // SPEC.md:608 (criterion 6) on the GPU path: with the recording
        // scheduler on, 100% of the launches for block i execute on the
        // target (GPU + stream) that owns block i, and they cover [0, n).
        auto& log = schedule_log::global();
        log.clear();
        log.set_enabled(true);
        cuda::block_allocator<double> alloc(targets);
        cuda_block_executor exec(targets);
        std::size_t const n = 100'003;
        dvec<double> a(n, 1.0, alloc), b(n, 2.0, alloc), c(n, 0.0, alloc);
        copy(par.on(exec), a.begin(), a.end(), c.begin());
        transform(par.on(exec), c.begin(), c.end(), b.begin(), ops::scale<double>{3.0});
        transform(par.on(exec), a.begin(), a.end(), b.begin(), c.begin(), ops::plus<double>{});
        transform(par.on(exec), b.begin(), b.end(), c.begin(), a.begin(), ops::triad<double>{3.0});
        log.set_enabled(false);
        auto entries = log.entries();
        EXPECT(entries.size() == 4 * targets.size());
        std::size_t covered = 0;
        for (auto const& e : entries)
        {
            auto const& owner = a.distribution().blocks[e.block].target;
            EXPECT(e.device == owner.device() && e.stream == owner.stream());
            EXPECT(e.data_device == e.device && e.data_stream == e.stream);
            covered += e.end - e.begin;
        }
        EXPECT(covered == 4 * n);
        log.clear();
    });
}

}    // namespace

// A device fault inside bulk_async_execute settles its future with an
// error (the stream callback carries the failed status), not a success.
// Run alone (--fault): the fault leaves the CUDA context unusable.
void fault_test()
{
    using namespace coloc;
    run("device fault settles the bulk future with an error", [] {
        auto targets = cuda::make_targets(std::vector<int>{0});
        cuda_block_executor exec(targets, executor_options{false});
        struct faulting_fill
        {
            void launch(cuda::target const& t, index_range const& r) const
            {
                // a non-null address no allocation covers: the kernel faults
                auto* bogus = reinterpret_cast<double*>(std::uintptr_t(1) << 44);
                detail::check(coloc_cuda_fill_f64(t.device(), t.stream(), bogus, r.size(), 1.0), "fill");
            }
        };
        shape s{{0, 1 << 20, 0}};
        auto f = executor_traits<cuda_block_executor>::bulk_async_execute(exec, faulting_fill{}, s);
        bool threw = false;
        try
        {
            f.get();
        }
        catch (coloc::error const& e)
        {
            threw = std::string(e.what()).find("failed") != std::string::npos;
        }
        EXPECT(threw);
    });
}

int main(int argc, char** argv)
{
    bool cpu = false, gpu = false;
    for (int i = 1; i < argc; ++i)
    {
        cpu = cpu || std::strcmp(argv[i], "--cpu") == 0;
        gpu = gpu || std::strcmp(argv[i], "--gpu") == 0;
        if (std::strcmp(argv[i], "--fault") == 0)
        {
            fault_test();
            std::printf("%d/%d passed\n", g_run - g_failed, g_run);
            return g_failed ? 1 : 0;
        }
    }
    if (!cpu && !gpu)
        cpu = true;
    if (cpu)
        cpu_tests();
    if (gpu)
    {
        gpu_tests();
        // the staging rings are process-lifetime caches: hand them back so
        // a leak check (compute-sanitizer --leak-check full) sees none
        if (coloc_cuda_staging_release() != COLOC_OK)
            ++g_failed;
    }
    std::printf("%d/%d passed\n", g_run - g_failed, g_run);
    return g_failed ? 1 : 0;
}
