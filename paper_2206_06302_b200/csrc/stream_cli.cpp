// stream_cli.cpp -- `stream_b200`: the SPEC stream_bench CLI
// on the GPU drop-in.
//
//   --size-mb X        decimal MB per array (repeatable: a sweep), or
//   --n N              elements per array (repeatable)
//   --iterations K     STREAM NTIMES (default 10; first excluded from stats)
//   --dtype f64|f32    element type (default f64)
//   --devices 0,1,...  one target per listed device (default: all GPUs)
//   --fma              triad as fma(c, s, b)
//   --sync             reference blocking semantics per algorithm call
//   --triad-scalar S   fault injection: Triad uses S instead of 3.0
//   --target device    the only target kind on this path (numa/cores are the
//                      reference's host library)
//   --compare-baseline also run the native CUDA STREAM (libstream_native.so)
//                      and the drop-in with blocking calls, both timed with the
//                      host clock, and print their ratio
//   --out PATH         write the report to PATH instead of stdout
//   --format human|csv|json
// Exit code 0 only when validation passes (criterion 9).
#include "coloc_cuda.h"
#include "coloc_stream.h"
#include "stream_native.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

namespace {

struct kernel_stats
{
    char const* name;
    double bytes;
    double min_s = 1e300, max_s = 0, sum_s = 0;
    int count = 0;
};

int die(char const* what, int st)
{
    std::fprintf(stderr, "stream_b200: %s failed (%d): %s\n", what, st, coloc_stream_last_error());
    return 2;
}

}    // namespace

int main(int argc, char** argv)
{
    std::vector<std::uint64_t> sizes;
    int iterations = 10;
    bool f32 = false, fma = false, sync = false, compare = false;
    std::string out_path;
    double triad_scalar = 3.0;
    std::string format = "human";
    std::vector<int> devices;
    for (int i = 1; i < argc; ++i)
    {
        std::string a = argv[i];
        auto next = [&]() -> std::string {
            if (i + 1 >= argc)
            {
                std::fprintf(stderr, "missing value for %s\n", a.c_str());
                std::exit(2);
            }
            return argv[++i];
        };
        if (a == "--size-mb")
            sizes.push_back(0x8000000000000000ULL | std::uint64_t(std::stod(next()) * 1e6));
        else if (a == "--n")
            sizes.push_back(std::stoull(next()));
        else if (a == "--iterations")
            iterations = std::stoi(next());
        else if (a == "--dtype")
            f32 = next() == "f32";
        else if (a == "--fma")
            fma = true;
        else if (a == "--sync")
            sync = true;
        else if (a == "--triad-scalar")
            triad_scalar = std::stod(next());
        else if (a == "--format")
            format = next();
        else if (a == "--compare-baseline")
            compare = true;
        else if (a == "--out")
            out_path = next();
        else if (a == "--target")
        {
            std::string t = next();
            if (t != "device")
            {
                std::fprintf(stderr, "stream_b200: --target %s: only 'device' (GPUs) is on this path; "
                                     "numa/cores targets belong to the reference's host library\n",
                    t.c_str());
                return 2;
            }
        }
        else if (a == "--devices")
        {
            std::stringstream ss(next());
            std::string tok;
            while (std::getline(ss, tok, ','))
                devices.push_back(std::stoi(tok));
        }
        else
        {
            std::fprintf(stderr, "unknown flag %s\n", a.c_str());
            return 2;
        }
    }
    if (iterations < 1)
        iterations = 1;
    if (!out_path.empty() && !std::freopen(out_path.c_str(), "w", stdout))
    {
        std::fprintf(stderr, "stream_b200: cannot write %s\n", out_path.c_str());
        return 2;
    }
    if (sizes.empty())
        sizes.push_back(10000000);
    if (devices.empty())
    {
        int n = 0;
        coloc_cuda_device_count(&n);
        for (int d = 0; d < n; ++d)
            devices.push_back(d);
        if (devices.empty())
        {
            std::fprintf(stderr, "stream_b200: no CUDA device\n");
            return 2;
        }
    }
    std::size_t const elem = f32 ? 4 : 8;
    bool all_ok = true;
    bool first_row = true;
    if (format == "csv")
        std::printf("n,kernel,bytes,min_time_s,avg_time_s,max_time_s,best_mbps,validated\n");
    if (format == "json")
        std::printf("[");
    for (std::uint64_t raw : sizes)
    {
        std::uint64_t n = (raw & 0x8000000000000000ULL) ?
            (raw & ~0x8000000000000000ULL) / elem :
            raw;
        coloc_stream_config cfg{};
        cfg.dtype = f32 ? COLOC_STREAM_F32 : COLOC_STREAM_F64;
        cfg.init = COLOC_STREAM_INIT_STREAM;
        cfg.fma = fma;
        cfg.synchronous = sync;
        cfg.ntargets = int(devices.size());
        cfg.devices = devices.data();
        cfg.count = n;
        cfg.scalar = 3.0;
        cfg.triad_scalar = triad_scalar;
        void* h = nullptr;
        int st = coloc_stream_create(&cfg, &h);
        if (st)
            return die("create", st);
        for (int k = 0; k < iterations; ++k)
            if ((st = coloc_stream_iterate(h, 1)))
                return die("iterate", st);
        kernel_stats ks[4] = {{"Copy", 2.0 * n * elem}, {"Scale", 2.0 * n * elem},
            {"Add", 3.0 * n * elem}, {"Triad", 3.0 * n * elem}};
        int rec = 0;
        coloc_stream_recorded(h, &rec);
        for (int i = rec > 1 ? 1 : 0; i < rec; ++i)
        {
            double ms[4];
            if ((st = coloc_stream_kernel_ms(h, i, ms)))
                return die("kernel_ms", st);
            for (int k = 0; k < 4; ++k)
            {
                double s = ms[k] * 1e-3;
                ks[k].min_s = std::min(ks[k].min_s, s);
                ks[k].max_s = std::max(ks[k].max_s, s);
                ks[k].sum_s += s;
                ks[k].count++;
            }
        }
        double expected[3], sums[3];
        if ((st = coloc_stream_err_sums(h, expected, sums, nullptr)))
            return die("validate", st);
        double const eps = f32 ? 1e-6 : 1e-8;
        bool ok = true;
        double rel[3];
        for (int j = 0; j < 3; ++j)
        {
            rel[j] = n ? sums[j] / double(n) / std::fabs(expected[j]) : 0.0;
            ok = ok && rel[j] <= eps;
        }
        all_ok = all_ok && ok;
        for (auto& k : ks)
        {
            double avg = k.count ? k.sum_s / k.count : 0;
            double mbps = k.bytes / k.min_s / 1e6;
            if (format == "csv")
                std::printf("%llu,%s,%.0f,%.9f,%.9f,%.9f,%.1f,%s\n", (unsigned long long) n,
                    k.name, k.bytes, k.min_s, avg, k.max_s, mbps, ok ? "true" : "false");
            else if (format == "json")
            {
                std::printf("%s{\"n\":%llu,\"kernel\":\"%s\",\"bytes\":%.0f,\"min_time_s\":%.9g,"
                            "\"avg_time_s\":%.9g,\"max_time_s\":%.9g,\"best_mbps\":%.1f,"
                            "\"validated\":%s}",
                    first_row ? "" : ",", (unsigned long long) n, k.name, k.bytes, k.min_s, avg,
                    k.max_s, mbps, ok ? "true" : "false");
                first_row = false;
            }
            else
                std::printf("%-6s n=%llu best %10.1f MB/s  min %.6f s  avg %.6f s  max %.6f s\n",
                    k.name, (unsigned long long) n, mbps, k.min_s, avg, k.max_s);
        }
        if (format == "human")
            std::printf("validation: %s (rel err a=%.3g b=%.3g c=%.3g, eps %.0e)\n",
                ok ? "PASSED" : "*** FAILED ***", rel[0], rel[1], rel[2], eps);
        coloc_stream_destroy(h);
        if (compare)
        {
            // SPEC run_baseline: drop-in (blocking calls) vs the native CUDA
            // STREAM, timed identically with the host clock
            int const dt = f32 ? COLOC_STREAM_F32 : COLOC_STREAM_F64;
            coloc_stream_timing ab{}, nat{};
            if ((st = coloc_stream_blocking_run(COLOC_STREAM_ARM_DROPIN, dt, devices[0], n, iterations, &ab)))
                return die("blocking_run", st);
            if ((st = stream_native_run(dt, devices[0], n, iterations, &nat)))
            {
                std::fprintf(stderr, "stream_b200: native baseline failed: %s\n", stream_native_last_error());
                return 2;
            }
            all_ok = all_ok && ab.validated && nat.validated;
            for (int k = 0; k < 4; ++k)
            {
                double const ba = ks[k].bytes / ab.avg_s[k] / 1e6, bn = ks[k].bytes / nat.avg_s[k] / 1e6;
                if (format == "csv")
                    std::printf("%llu,%s-baseline,%.0f,%.9f,%.9f,%.9f,%.1f,%s\n", (unsigned long long) n,
                        ks[k].name, ks[k].bytes, nat.min_s[k], nat.avg_s[k], nat.max_s[k],
                        ks[k].bytes / nat.min_s[k] / 1e6, nat.validated ? "true" : "false");
                else if (format == "json")
                    std::printf(",{\"n\":%llu,\"kernel\":\"%s\",\"baseline_avg_mbps\":%.1f,"
                                "\"abstraction_avg_mbps\":%.1f,\"ratio\":%.4f,\"validated\":%s}",
                        (unsigned long long) n, ks[k].name, bn, ba, ba / bn,
                        ab.validated && nat.validated ? "true" : "false");
                else
                    std::printf("%-6s n=%llu blocking, host clock: abstraction avg %10.1f MB/s  "
                                "native avg %10.1f MB/s  ratio %.4f\n",
                        ks[k].name, (unsigned long long) n, ba, bn, ba / bn);
            }
        }
    }
    if (format == "json")
        std::printf("]\n");
    return all_ok ? 0 : 1;
}
