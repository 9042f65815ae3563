// ref_stream_cpu.cpp -- drives the UNMODIFIED reference library `coloc`
// (/root/reference/proj, compiled from its own sources by oracle/Makefile)
// through its public API.
//
// TEST / BASELINE INFRASTRUCTURE ONLY: this binary is the reference CPU
// path.  It is used (1) to generate the golden fixtures under tests/golden
// that pin the C oracle, and (2) as bench.py's cpu_baseline and
// `--impl reference` arm.  Nothing in the product links it.
//
// The STREAM driver itself is not shipped by the reference; this follows
// PAPER.md:514-529 (Listing 4) and SPEC.md:529-547 (run_stream/validate):
// a=1, b=2, c=0, scalar 3; Copy c<-a, Scale b<-3c, Add c<-a+b,
// Triad a<-b+3c; per-kernel std::chrono::steady_clock; first iteration
// excluded; bytes 2/2/3/3 * n * sizeof(T).
//
// Placement: probe_topology() -> get_numa_domains() -> block_allocator +
// block_executor over the same targets, as BASELINE.md section 4 says.
// Always `par.on(exec)`: bare `par` on raw pointers hits the vexing parse
// at include/coloc/algorithms.hpp:277.
//
// Modes
//   stream         --dtype f64|f32 --n N --ntimes K [--warmup W] [--threads T] [--random SEED]
//   kernels        --dtype f64|f32 --n N --seed S --out DIR
//   partition      --n N --k K
//   shape          --n N --domains "0-5;6-11" [--offset O --len L]
//   helloworld

#include <coloc/algorithms.hpp>
#include <coloc/affinity.hpp>
#include <coloc/topology.hpp>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

namespace {

constexpr std::uint64_t golden = 0x9E3779B97F4A7C15ULL;
constexpr std::uint64_t array_stride = 0xD1B54A32D192ED03ULL;

std::uint64_t mix64(std::uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

std::uint64_t random_bits(std::uint64_t seed, unsigned k, std::uint64_t i)
{
    return mix64(seed + std::uint64_t(k) * array_stride + (i + 1) * golden);
}

template <typename T>
T to_value(std::uint64_t x)
{
    if constexpr (sizeof(T) == 8)
        return double(x >> 11) * 0x1p-53 * 2.0 - 1.0;
    else
        return float(x >> 40) * 0x1p-24f * 2.0f - 1.0f;
}

template <typename T>
std::uint64_t bits_of(T v)
{
    if constexpr (sizeof(T) == 8)
    {
        std::uint64_t u;
        std::memcpy(&u, &v, 8);
        return u;
    }
    else
    {
        std::uint32_t u;
        std::memcpy(&u, &v, 4);
        return u;
    }
}

struct args
{
    std::map<std::string, std::string> kv;
    std::string get(std::string const& k, std::string const& d = "") const
    {
        auto it = kv.find(k);
        return it == kv.end() ? d : it->second;
    }
};

args parse(int argc, char** argv)
{
    args a;
    for (int i = 2; i < argc; ++i)
    {
        std::string k = argv[i];
        if (k.rfind("--", 0) == 0 && i + 1 < argc)
            a.kv[k.substr(2)] = argv[++i];
    }
    return a;
}

std::string read_first_line(std::string const& path)
{
    std::ifstream in(path);
    std::string s;
    std::getline(in, s);
    return s;
}

std::string cpu_model()
{
    std::ifstream in("/proc/cpuinfo");
    std::string line;
    while (std::getline(in, line))
        if (line.rfind("model name", 0) == 0)
        {
            auto p = line.find(':');
            return p == std::string::npos ? line : line.substr(p + 2);
        }
    return "unknown";
}

std::string json_escape(std::string const& s)
{
    std::string o;
    for (char ch : s)
    {
        if (ch == '"' || ch == '\\')
            o += '\\';
        o += ch;
    }
    return o;
}

// Targets: NUMA domains of the probed topology, optionally restricted to
// the first `threads` schedulable PUs (domains emptied by the restriction
// are dropped).
std::vector<coloc::host::target> stream_targets(std::size_t threads)
{
    auto domains = coloc::get_numa_domains(coloc::probe_topology());
    if (threads == 0)
        return domains;
    std::vector<coloc::host::target> out;
    std::size_t left = threads;
    for (auto const& d : domains)
    {
        if (left == 0)
            break;
        coloc::cpu_set keep;
        for (std::size_t pu : d.cpuset().to_list())
        {
            if (left == 0)
                break;
            keep.set(pu);
            --left;
        }
        out.push_back(coloc::restrict_target(d, keep));
    }
    return out;
}

template <typename T>
int run_stream(args const& a)
{
    using clock = std::chrono::steady_clock;
    std::size_t const n = std::stoull(a.get("n", "10000000"));
    int const ntimes = std::stoi(a.get("ntimes", "10"));
    // Iterations excluded from the statistics (STREAM excludes the first).
    int const warmup = std::max(1, std::stoi(a.get("warmup", "1")));
    std::size_t const threads = std::stoull(a.get("threads", "0"));
    bool const random_init = !a.get("random").empty();
    std::uint64_t const seed =
        random_init ? std::stoull(a.get("random"), nullptr, 0) : 0;

    auto targets = stream_targets(threads);
    coloc::host::block_allocator<T> alloc(targets);
    coloc::block_executor exec(targets);
    auto policy = coloc::par.on(exec);

    using vec = coloc::vector<T, coloc::host::block_allocator<T>>;
    auto t_init0 = clock::now();
    vec as = random_init ?
        vec::generate(n, [seed](std::size_t i) { return to_value<T>(random_bits(seed, 0, i)); }, alloc) :
        vec(n, T(1.0), alloc);
    vec bs = random_init ?
        vec::generate(n, [seed](std::size_t i) { return to_value<T>(random_bits(seed, 1, i)); }, alloc) :
        vec(n, T(2.0), alloc);
    vec cs = random_init ?
        vec::generate(n, [seed](std::size_t i) { return to_value<T>(random_bits(seed, 2, i)); }, alloc) :
        vec(n, T(0.0), alloc);
    double const init_s =
        std::chrono::duration<double>(clock::now() - t_init0).count();

    T const scalar = T(3.0);
    std::vector<double> times[4];
    for (int k = 0; k < ntimes; ++k)
    {
        // Listing 4, verbatim modulo the element type.
        auto t0 = clock::now();
        coloc::copy(policy, as.begin(), as.end(), cs.begin());
        auto t1 = clock::now();
        coloc::transform(policy, cs.begin(), cs.end(), bs.begin(),
            [scalar](T c) { return c * scalar; });
        auto t2 = clock::now();
        coloc::transform(policy, as.begin(), as.end(), bs.begin(), cs.begin(),
            [](T x, T y) { return x + y; });
        auto t3 = clock::now();
        coloc::transform(policy, bs.begin(), bs.end(), cs.begin(), as.begin(),
            [scalar](T b, T c) { return b + c * scalar; });
        auto t4 = clock::now();
        times[0].push_back(std::chrono::duration<double>(t1 - t0).count());
        times[1].push_back(std::chrono::duration<double>(t2 - t1).count());
        times[2].push_back(std::chrono::duration<double>(t3 - t2).count());
        times[3].push_back(std::chrono::duration<double>(t4 - t3).count());
    }

    // Validation or checksums for random init.
    T const* pa = as.data_handle();
    T const* pb = bs.data_handle();
    T const* pc = cs.data_handle();
    std::ostringstream val;
    val.precision(17);
    bool ok = true;
    if (!random_init)
    {
        T ea = 1, eb = 2, ec = 0;
        for (int k = 0; k < ntimes; ++k)
        {
            ec = ea;
            eb = scalar * ec;
            ec = ea + eb;
            T t = scalar * ec;
            ea = eb + t;
        }
        double sa = 0, sb = 0, sc = 0;
        for (std::size_t j = 0; j < n; ++j)
        {
            // equal values (also equal infinities: f32 overflows after 32
            // iterations) count as 0, as in oracle_err_term
            auto term = [](double x, double e) { return x == e ? 0.0 : std::fabs(x - e); };
            sa += term(double(pa[j]), double(ea));
            sb += term(double(pb[j]), double(eb));
            sc += term(double(pc[j]), double(ec));
        }
        double const eps = sizeof(T) == 8 ? 1e-8 : 1e-6;
        double ra = n ? sa / n / std::fabs(double(ea)) : 0;
        double rb = n ? sb / n / std::fabs(double(eb)) : 0;
        double rc = n ? sc / n / std::fabs(double(ec)) : 0;
        ok = ra <= eps && rb <= eps && rc <= eps;
        val << "{\"expected\":[" << double(ea) << "," << double(eb) << ","
            << double(ec) << "],\"rel_err\":[" << ra << "," << rb << "," << rc
            << "],\"epsilon\":" << eps << ",\"passed\":" << (ok ? "true" : "false")
            << "}";
    }
    else
    {
        std::uint64_t h[3] = {0, 0, 0};
        for (std::size_t j = 0; j < n; ++j)
        {
            h[0] += mix64(bits_of(pa[j]) + j * golden);
            h[1] += mix64(bits_of(pb[j]) + j * golden);
            h[2] += mix64(bits_of(pc[j]) + j * golden);
        }
        val << "{\"checksums\":[\"0x" << std::hex << h[0] << "\",\"0x" << h[1]
            << "\",\"0x" << h[2] << "\"]}" << std::dec;
    }

    static char const* names[4] = {"copy", "scale", "add", "triad"};
    int const words[4] = {2, 2, 3, 3};
    std::size_t pus = 0;
    for (auto const& t : targets)
        pus += t.unit_count();

    std::ostringstream js;
    js.precision(17);
    js << "{\"impl\":\"reference-cpu\",\"dtype\":\""
       << (sizeof(T) == 8 ? "f64" : "f32") << "\",\"n\":" << n
       << ",\"ntimes\":" << ntimes << ",\"init_s\":" << init_s
       << ",\"validation\":" << val.str() << ",\"kernels\":{";
    for (int k = 0; k < 4; ++k)
    {
        auto const& t = times[k];
        double mn = 1e300, mx = 0, sum = 0;
        std::size_t cnt = 0;
        std::size_t const skip = t.size() > std::size_t(warmup) ? std::size_t(warmup) : 0;
        for (std::size_t i = skip; i < t.size(); ++i)
        {
            mn = std::min(mn, t[i]);
            mx = std::max(mx, t[i]);
            sum += t[i];
            ++cnt;
        }
        double avg = cnt ? sum / cnt : 0;
        double bytes = double(words[k]) * double(n) * sizeof(T);
        js << (k ? "," : "") << "\"" << names[k] << "\":{\"bytes\":" << bytes
           << ",\"min_time_s\":" << mn << ",\"avg_time_s\":" << avg
           << ",\"max_time_s\":" << mx << ",\"sum_time_s\":" << sum << ",\"count\":" << cnt
           << ",\"best_gbs\":" << bytes / mn / 1e9
           << ",\"avg_gbs\":" << bytes / avg / 1e9 << "}";
    }
    // whole Listing-4 iterations (all four kernels), warm-up included:
    // the e2e rule of bench.py (STREAM bytes of whole runs / their time)
    js << "},\"warmup\":" << warmup << ",\"iter_time_s\":[";
    for (int i = 0; i < ntimes; ++i)
        js << (i ? "," : "") << times[0][std::size_t(i)] + times[1][std::size_t(i)] +
                times[2][std::size_t(i)] + times[3][std::size_t(i)];
    js << "],\"host\":{\"pus_used\":" << pus << ",\"nproc\":"
       << coloc::os_schedulable_units().count() << ",\"numa\":[";
    auto all = coloc::get_numa_domains(coloc::probe_topology());
    for (std::size_t d = 0; d < all.size(); ++d)
        js << (d ? "," : "") << "\"" << all[d].cpuset().to_string() << "\"";
    js << "],\"targets\":[";
    for (std::size_t d = 0; d < targets.size(); ++d)
        js << (d ? "," : "") << "\"" << json_escape(targets[d].description())
           << "\"";
    js << "],\"cpu_model\":\"" << json_escape(cpu_model())
       << "\",\"compile\":\"" << COLOC_REF_FLAGS << "\"}}";
    std::cout << js.str() << std::endl;
    return ok ? 0 : 3;
}

// One application of each kernel to seeded random inputs, via the
// reference algorithms; raw outputs written for fixture generation.
template <typename T>
int run_kernels(args const& a)
{
    std::size_t const n = std::stoull(a.get("n", "1000"));
    std::uint64_t const seed = std::stoull(a.get("seed", "0x220606302"), nullptr, 0);
    std::string const out = a.get("out", ".");
    auto targets = stream_targets(std::stoull(a.get("threads", "0")));
    coloc::host::block_allocator<T> alloc(targets);
    coloc::block_executor exec(targets);
    auto policy = coloc::par.on(exec);
    using vec = coloc::vector<T, coloc::host::block_allocator<T>>;

    auto gen = [&](unsigned k) {
        return vec::generate(
            n, [seed, k](std::size_t i) { return to_value<T>(random_bits(seed, k, i)); },
            alloc);
    };
    vec as = gen(0), bs = gen(1), cs = gen(2);
    vec o_copy(n, T(0), alloc), o_scale(n, T(0), alloc), o_add(n, T(0), alloc),
        o_triad(n, T(0), alloc);
    T const scalar = T(3.0);
    coloc::copy(policy, as.begin(), as.end(), o_copy.begin());
    coloc::transform(policy, cs.begin(), cs.end(), o_scale.begin(),
        [scalar](T c) { return c * scalar; });
    coloc::transform(policy, as.begin(), as.end(), bs.begin(), o_add.begin(),
        [](T x, T y) { return x + y; });
    coloc::transform(policy, bs.begin(), bs.end(), cs.begin(), o_triad.begin(),
        [scalar](T b, T c) { return b + c * scalar; });

    auto dump = [&](vec const& v, char const* name) {
        std::ofstream f(out + "/" + name + ".bin", std::ios::binary);
        f.write(reinterpret_cast<char const*>(v.data_handle()),
            std::streamsize(n * sizeof(T)));
    };
    dump(as, "a");
    dump(bs, "b");
    dump(cs, "c");
    dump(o_copy, "copy");
    dump(o_scale, "scale");
    dump(o_add, "add");
    dump(o_triad, "triad");
    std::cout << "{\"n\":" << n << ",\"seed\":" << seed << "}" << std::endl;
    return 0;
}

int run_partition(args const& a)
{
    std::size_t const n = std::stoull(a.get("n", "10"));
    std::size_t const k = std::stoull(a.get("k", "3"));
    std::vector<int> targets(k);
    for (std::size_t i = 0; i < k; ++i)
        targets[i] = int(i);
    try
    {
        auto p = coloc::partition_block(n, targets);
        std::cout << "[";
        for (std::size_t i = 0; i < p.blocks.size(); ++i)
            std::cout << (i ? "," : "") << "[" << p.blocks[i].target << ","
                      << p.blocks[i].offset << "," << p.blocks[i].length << "]";
        std::cout << "]" << std::endl;
    }
    catch (std::invalid_argument const& e)
    {
        std::cout << "{\"error\":\"invalid_argument\"}" << std::endl;
    }
    return 0;
}

// algorithm_shape over a block_executor whose targets are the given mock
// cpusets (pinning is logical when the machine is smaller): dumps the
// ranges for a destination sub-range [offset, offset+len) of an n-vector.
int run_shape(args const& a)
{
    std::size_t const n = std::stoull(a.get("n", "100"));
    std::string spec = a.get("domains", "0-5;6-11");
    std::vector<coloc::host::target> targets;
    std::stringstream ss(spec);
    std::string item;
    while (std::getline(ss, item, ';'))
        targets.emplace_back(coloc::cpu_set::parse(item));
    std::size_t const off = std::stoull(a.get("offset", "0"));
    std::size_t const len = std::stoull(a.get("len", std::to_string(n - off)));
    coloc::host::block_allocator<double> alloc(targets);
    coloc::block_executor exec(targets);
    coloc::vector<double, coloc::host::block_allocator<double>> v(n, 0.0, alloc);
    auto s = coloc::detail::algorithm_shape(exec, v.begin() + std::ptrdiff_t(off), len);
    std::cout << "[";
    for (std::size_t i = 0; i < s.size(); ++i)
        std::cout << (i ? "," : "") << "[" << s[i].begin << "," << s[i].end
                  << "," << s[i].block << "]";
    std::cout << "]" << std::endl;
    return 0;
}

int run_helloworld()
{
    auto targets = stream_targets(0);
    coloc::host::block_allocator<char> alloc(targets);
    coloc::block_executor exec(targets);
    coloc::vector<char, coloc::host::block_allocator<char>> s(
        {'h', 'e', 'l', 'l', 'o', 'w', 'o', 'r', 'l', 'd'}, alloc);
    coloc::transform(coloc::par.on(exec), s.begin(), s.end(), s.begin(),
        [](char c) { return char(std::toupper(static_cast<unsigned char>(c))); });
    std::string out(s.data_handle(), s.size());
    std::cout << out << std::endl;
    return 0;
}

}    // namespace

int main(int argc, char** argv)
{
    if (argc < 2)
    {
        std::cerr << "usage: ref_stream_cpu stream|kernels|partition|shape|helloworld [--opts]\n";
        return 2;
    }
    std::string mode = argv[1];
    args a = parse(argc, argv);
    bool f32 = a.get("dtype", "f64") == "f32";
    try
    {
        if (mode == "stream")
            return f32 ? run_stream<float>(a) : run_stream<double>(a);
        if (mode == "kernels")
            return f32 ? run_kernels<float>(a) : run_kernels<double>(a);
        if (mode == "partition")
            return run_partition(a);
        if (mode == "shape")
            return run_shape(a);
        if (mode == "helloworld")
            return run_helloworld();
    }
    catch (std::exception const& e)
    {
        std::cerr << "ref_stream_cpu: " << e.what() << "\n";
        return 1;
    }
    std::cerr << "unknown mode " << mode << "\n";
    return 2;
}
