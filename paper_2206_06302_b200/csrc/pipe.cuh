// pipe.cuh -- software-pipelined persistent variant of ew_pack_kernel
// (tuning.variant = 4; an experiment, never the automatic choice).
//
// One CTA per resident slot walks its tiles with the next tile's loads in
// flight while the current tile is computed and stored (two register
// buffers), so an SM never drains between tiles the way one-tile CTAs do
// at retirement.  Tile order: blocked (CTA c owns tiles [c*K, (c+1)*K)) or
// interleaved (grid stride).
#pragma once

#include "coloc_b200/kernels/elementwise.cuh"

namespace coloc_cuda {

template <typename T, typename Op, int U>
struct pipe_tile
{
    pack<T> x[U], y[U];

    __device__ __forceinline__ void load(T const* b0, T const* b1, std::size_t p0, unsigned stride,
        std::size_t npacks)
    {
        constexpr int E = kPackBytes / int(sizeof(T));
#pragma unroll
        for (int u = 0; u < U; ++u)
        {
            std::size_t const p = p0 + std::size_t(u) * stride;
            if (p < npacks)
            {
                if constexpr (Op::nin >= 1)
                    ld_pack<1>(b0 + p * E, x[u].w);
                if constexpr (Op::nin >= 2)
                    ld_pack<1>(b1 + p * E, y[u].w);
            }
        }
    }

    __device__ __forceinline__ void store(Op const& op, T* bd, std::size_t head, std::size_t p0,
        unsigned stride, std::size_t npacks) const
    {
        constexpr int E = kPackBytes / int(sizeof(T));
#pragma unroll
        for (int u = 0; u < U; ++u)
        {
            std::size_t const p = p0 + std::size_t(u) * stride;
            if (p < npacks)
            {
                pack<T> o;
                if constexpr (Op::identity)
                    o = x[u];
                else
                {
#pragma unroll
                    for (int j = 0; j < E; ++j)
                        o.v[j] = op(head + p * E + std::size_t(j), Op::nin >= 1 ? x[u].v[j] : T(),
                            Op::nin >= 2 ? y[u].v[j] : T());
                }
                st_pack<1>(bd + p * E, o.w);
            }
        }
    }
};

template <typename T, typename Op, int U, bool Blocked>
__global__ void __launch_bounds__(512) ew_pipe_kernel(Op op, T* dst, T const* s0, T const* s1,
    std::size_t head, std::size_t npacks, std::size_t tail)
{
    std::size_t const tile = std::size_t(blockDim.x) * U;
    std::size_t const ntiles = (npacks + tile - 1) / tile;
    std::size_t t, end, step;
    if constexpr (Blocked)
    {
        std::size_t const per = (ntiles + gridDim.x - 1) / gridDim.x;
        t = std::size_t(blockIdx.x) * per;
        end = t + per < ntiles ? t + per : ntiles;
        step = 1;
    }
    else
    {
        t = blockIdx.x;
        end = ntiles;
        step = gridDim.x;
    }
    T* bd = dst + head;
    T const* b0 = Op::nin >= 1 ? s0 + head : nullptr;
    T const* b1 = Op::nin >= 2 ? s1 + head : nullptr;
    pipe_tile<T, Op, U> a, b;
    if (t < end)
        a.load(b0, b1, t * tile + threadIdx.x, blockDim.x, npacks);
    // two tiles per trip so both register buffers have fixed names
    while (t < end)
    {
        std::size_t const t1 = t + step;
        if (t1 < end)
            b.load(b0, b1, t1 * tile + threadIdx.x, blockDim.x, npacks);
        a.store(op, bd, head, t * tile + threadIdx.x, blockDim.x, npacks);
        if (t1 >= end)
            break;
        std::size_t const t2 = t1 + step;
        if (t2 < end)
            a.load(b0, b1, t2 * tile + threadIdx.x, blockDim.x, npacks);
        b.store(op, bd, head, t1 * tile + threadIdx.x, blockDim.x, npacks);
        t = t2;
    }
    constexpr int E = kPackBytes / int(sizeof(T));
    if (blockIdx.x == gridDim.x - 1)
        for (std::size_t r = threadIdx.x; r < head + tail; r += blockDim.x)
        {
            std::size_t const i = r < head ? r : head + npacks * E + (r - head);
            dst[i] = op(i, Op::nin >= 1 ? s0[i] : T(), Op::nin >= 2 ? s1[i] : T());
        }
}

}    // namespace coloc_cuda
