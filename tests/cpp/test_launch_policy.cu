// Host-only checks of the launch policy (kernels/launch.cuh): the shape and
// cache policy resolve_shape picks per array size, and the pack split of a
// range.  Compiled by nvcc, runs without a GPU (no CUDA call is made).
#include "coloc_b200/kernels/launch.cuh"

#include <cstdio>
#include <cstdlib>

using namespace coloc_cuda;

static int failures = 0;
#define CHECK(cond)                                                          \
    do                                                                       \
    {                                                                        \
        if (!(cond))                                                         \
        {                                                                    \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);      \
            ++failures;                                                      \
        }                                                                    \
    } while (0)

int main()
{
    std::size_t const MiB = std::size_t(1) << 20;
    std::size_t const L2 = 133 * 1000 * 1000;    // B200 (cudaDeviceProp::l2CacheSize)

    // cache policy by destination size
    CHECK(auto_hint(8 * MiB, L2) == 0);      // three arrays fit in 0.6 L2
    CHECK(auto_hint(24 * MiB, L2) == 0);
    CHECK(auto_hint(32 * MiB, L2) == 3);     // one output fits: evict-last stores
    CHECK(auto_hint(80'000'000, L2) == 3);   // C1
    CHECK(auto_hint(96 * MiB, L2) == 5);     // a share of the output kept
    CHECK(auto_hint(112 * MiB, L2) == 5);
    CHECK(auto_hint(128 * MiB, L2) == 1);    // streaming
    CHECK(auto_hint(std::size_t(8) << 30, L2) == 1);    // C2 / C3
    CHECK(auto_hint(8 * MiB, 0) == 1);       // unknown L2: streaming

    // shapes: >= 256 MiB 1024 threads, 1 pack (one input) / 2 packs (two)
    launch_shape s = resolve_shape({}, 1, std::size_t(8) << 30, L2);
    CHECK(s.threads == 1024 && s.unroll == 1 && s.exact == 1 && s.variant == 1 && s.hint == 1);
    s = resolve_shape({}, 2, std::size_t(8) << 30, L2);
    CHECK(s.threads == 1024 && s.unroll == 2 && s.variant == 1);
    s = resolve_shape({}, 2, 80'000'000, L2);
    CHECK(s.threads == 256 && s.unroll == 2 && s.hint == 3);
    s = resolve_shape({}, 2, 16 * MiB, L2);    // small ranges: 8 KB tiles
    CHECK(s.threads == 256 && s.unroll == 1 && s.hint == 0);
    // hint 5 keeps ~0.6 L2 of the output
    s = resolve_shape({}, 2, 112 * MiB, L2);
    CHECK(s.hint == 5 && s.l2_keep_permille > 600 && s.l2_keep_permille < 700);
    // explicit settings win; unroll 4 caps the block at 512 threads
    launch_shape u;
    u.threads = 1024;
    u.unroll = 4;
    u.hint = 0;
    s = resolve_shape(u, 2, std::size_t(8) << 30, L2);
    CHECK(s.threads == 512 && s.unroll == 4 && s.hint == 0);
    // TMA defaults apply only when the TMA variant is asked for
    u = {};
    u.variant = 2;
    s = resolve_shape(u, 2, std::size_t(8) << 30, L2);
    CHECK(s.variant == 2 && s.chunk_bytes == 8192 && s.stages == 2 && s.ctas_per_sm == 3 && s.schedule == 2);

    // pack split: unaligned head < 32 B, 32-byte packs, tail < 32 B
    alignas(32) static double buf[64];
    pack_split p = split_range<double>(2, buf + 1, buf + 1, buf + 1, 20);
    CHECK(p.aligned && p.head == 3 && p.npacks == 4 && p.tail == 1);
    p = split_range<double>(2, buf + 1, buf + 2, buf + 1, 20);    // operands disagree mod 32 B
    CHECK(!p.aligned);
    p = split_range<double>(1, buf, buf, nullptr, 3);               // shorter than one pack
    CHECK(p.aligned && p.head == 0 && p.npacks == 0 && p.tail == 3);

    if (failures)
        return 1;
    std::printf("launch policy checks passed\n");
    return 0;
}
