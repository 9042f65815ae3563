// device_lambda.cuh -- coloc::transform / coloc::for_each with user-written
// __device__ callables, for code compiled by nvcc (--extended-lambda).
//
// The paper's CUDA executor runs "any callable that is marked with the CUDA
// specific __device__ attribute".  Precompiled kernels
// behind the C ABI can only offer named operations (ops.hpp); this header
// lifts that restriction for nvcc users: a device lambda (or a functor that
// opts in through coloc::is_device_callable) is instantiated into the same
// sm_100a kernel template the library uses (kernels/elementwise.cuh), with
// the same launch policy (kernels/launch.cuh) and the library's current
// tuning, inside the user's translation unit.  Listing 4 then compiles as
// written in the paper, with `__device__` added to its lambdas.
#pragma once

#if !defined(__CUDACC__)
#error "coloc_b200/device_lambda.cuh must be compiled by nvcc"
#endif

#include "coloc_b200/kernels/launch.cuh"
#include "coloc_b200/ops.hpp"
#include "coloc_cuda.h"

#include <cuda_runtime.h>

#include <array>
#include <mutex>
#include <cstddef>
#include <type_traits>

namespace coloc {

/// True for closure types of __device__ / __host__ __device__ extended
/// lambdas; specialise to true for functor types whose call operator is
/// __device__.
template <typename F>
struct is_device_callable
  : std::bool_constant<__nv_is_extended_device_lambda_closure_type(F) ||
        __nv_is_extended_host_device_lambda_closure_type(F)>
{
};

namespace detail {

template <typename F>
concept device_callable = is_device_callable<std::remove_cvref_t<F>>::value;

template <typename T, typename F>
struct op_user_unary
{
    static constexpr int nin = 1;
    static constexpr bool identity = false;
    F f;
    __device__ T operator()(std::size_t, T x, T) const { return f(x); }
};

template <typename T, typename F>
struct op_user_binary
{
    static constexpr int nin = 2;
    static constexpr bool identity = false;
    F f;
    __device__ T operator()(std::size_t, T a, T b) const { return f(a, b); }
};

template <typename T, typename F>
struct op_user_in_place
{
    static constexpr int nin = 1;
    static constexpr bool identity = false;
    F f;
    __device__ T operator()(std::size_t, T x, T) const
    {
        T y = x;
        f(y);
        return y;
    }
};

struct device_facts
{
    int sm_count = 0;
    std::size_t l2_bytes = 0;
};

inline device_facts facts_of(int dev)
{
    static std::mutex mu;
    static std::array<device_facts, 64> cache{};
    if (dev < 0 || dev >= int(cache.size()))
        return {};
    std::lock_guard<std::mutex> lock(mu);
    if (cache[std::size_t(dev)].sm_count == 0)
    {
        coloc_cuda_device_info info{};
        if (coloc_cuda_device_info_get(dev, &info) != COLOC_OK)
            return {};
        cache[std::size_t(dev)] = {info.sm_count, info.l2_bytes};
    }
    return cache[std::size_t(dev)];
}

// Launches a user op over [0, n) on (dev, stream) with the library tuning.
template <typename T, typename Op>
int launch_user(int dev, void* stream, Op const& op, T* dst, T const* s0, T const* s1,
    std::size_t n)
{
    if (n == 0)
        return COLOC_OK;
    device_facts const f = facts_of(dev);
    int const sms = f.sm_count;
    if (sms == 0 || cudaSetDevice(dev) != cudaSuccess)
    {
        (void) cudaGetLastError();
        return COLOC_ERR_INVALID_TARGET;
    }
    // a user kernel cannot take part in a tile chain: if one is open on
    // this stream, it restarts behind this launch (full dependency)
    if (int const st = coloc_cuda_chain_break(dev, stream); st != COLOC_OK)
        return st;
    coloc_cuda_tuning t{};
    (void) coloc_cuda_get_tuning(&t);
    coloc_cuda::launch_shape s;
    s.threads = t.threads;
    s.unroll = t.unroll;
    s.hint = t.cache_hint;
    s.exact = t.exact_grid;
    s.ctas_per_sm = t.ctas_per_sm;
    s.l2_keep_permille = t.l2_keep_permille;
    s = coloc_cuda::resolve_shape(s, Op::nin, n * sizeof(T), f.l2_bytes);
    cudaError_t const e = coloc_cuda::launch_elementwise<T, Op>(static_cast<cudaStream_t>(stream),
        sms, op, dst, s0, s1, n, s);
    if (e != cudaSuccess)
    {
        (void) cudaGetLastError();
        return e == cudaErrorInvalidValue ? COLOC_ERR_INVALID_ARGUMENT : COLOC_ERR_SUBMISSION;
    }
    return COLOC_OK;
}

template <typename F, typename T>
    requires device_callable<F>
struct device_unary<F, T>
{
    static constexpr bool supported = true;
    static int launch(F const& f, int dev, void* s, T* dst, T const* src, std::size_t n)
    {
        return launch_user<T>(dev, s, op_user_unary<T, F>{f}, dst, src, static_cast<T const*>(nullptr), n);
    }
};

template <typename F, typename T>
    requires device_callable<F>
struct device_binary<F, T>
{
    static constexpr bool supported = true;
    static int launch(F const& f, int dev, void* s, T* dst, T const* a, T const* b, std::size_t n)
    {
        return launch_user<T>(dev, s, op_user_binary<T, F>{f}, dst, a, b, n);
    }
};

template <typename F, typename T>
    requires device_callable<F>
struct device_in_place<F, T>
{
    static constexpr bool supported = true;
    static int launch(F const& f, int dev, void* s, T* x, std::size_t n)
    {
        return launch_user<T>(dev, s, op_user_in_place<T, F>{f}, x, x, static_cast<T const*>(nullptr), n);
    }
};

}    // namespace detail
}    // namespace coloc
