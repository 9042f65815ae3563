// ops.hpp -- named element operations.
//
// Listing 4 passes lambdas to copy/transform.  Lambdas
// cannot cross a C ABI into precompiled sm_100a kernels, so the drop-in
// names each STREAM operation as a function object.  Every op is also an
// ordinary host callable with the reference's arithmetic, so one driver
// source runs unchanged against the reference's host vectors (there the
// reference algorithms simply call operator()).
//
//   transform (unary)  : identity, scale (Listing 4 Scale: c * scalar), to_upper (Listing 3)
//   transform (binary) : plus / std::plus (Add: a + b), triad (Triad: b + c*scalar),
//                        triad_fma (fma(c, scalar, b): the FMA-contracted build)
//   for_each           : assign, multiply_by, make_upper
//   generators         : uniform_random (seeded splitmix64, = oracle), iota
#pragma once

#include "coloc_b200/memory.hpp"

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <type_traits>

namespace coloc::ops {

template <typename T>
struct identity
{
    T operator()(T x) const { return x; }
};

template <typename T>
struct scale
{
    T scalar;
    T operator()(T c) const { return c * scalar; }
};

template <typename T>
struct plus
{
    T operator()(T a, T b) const { return a + b; }
};

/// b + c*scalar with the product rounded before the sum (no contraction):
/// bit-identical to the reference built with its defaults.
template <typename T>
struct triad
{
    T scalar;
    T operator()(T b, T c) const
    {
        T volatile t = c * scalar;    // keep the host form uncontracted too
        return b + t;
    }
};

template <typename T>
struct triad_fma
{
    T scalar;
    T operator()(T b, T c) const { return std::fma(c, scalar, b); }
};

struct to_upper
{
    char operator()(char c) const { return (c >= 'a' && c <= 'z') ? char(c - 32) : c; }
    unsigned char operator()(unsigned char c) const
    {
        return (c >= 'a' && c <= 'z') ? (unsigned char) (c - 32) : c;
    }
};

template <typename T>
struct assign
{
    T value;
    void operator()(T& x) const { x = value; }
};

template <typename T>
struct multiply_by
{
    T scalar;
    void operator()(T& x) const { x = x * scalar; }
};

struct make_upper
{
    template <typename C>
    void operator()(C& c) const
    {
        c = to_upper{}(c);
    }
};

/// Element i of a seeded stream: splitmix64(seed + array*STRIDE + (first+i+1)*GOLDEN)
/// mapped to [-1, 1) -- the same numbers as oracle_fill_random_* and
/// coloc_cuda_generate_random_*.  `first` offsets the global index (a
/// rank's block of a larger array).
template <typename T>
struct uniform_random
{
    std::uint64_t seed = 0;
    std::uint32_t array = 0;
    std::uint64_t first = 0;

    T operator()(std::size_t i) const
    {
        std::uint64_t z = seed + std::uint64_t(array) * 0xD1B54A32D192ED03ULL +
            (first + i + 1) * 0x9E3779B97F4A7C15ULL;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        z ^= z >> 31;
        if constexpr (sizeof(T) == 8)
            return T(double(z >> 11) * 0x1p-53 * 2.0 - 1.0);
        else
            return T(float(z >> 40) * 0x1p-24f * 2.0f - 1.0f);
    }
};

template <typename T>
struct iota
{
    T first;
    T operator()(std::size_t i) const { return first + T(i); }
};

}    // namespace coloc::ops

namespace coloc::detail {

// ---------------------------------------------------------------------
// Device dispatch: which C-ABI kernel implements a named op for element
// type T.  `supported` is false for anything else, and the algorithms turn
// that into a compile error on device data (there is no CPU fallback).
// ---------------------------------------------------------------------

template <typename F, typename T>
struct device_unary
{
    static constexpr bool supported = false;
};

template <typename T>
struct device_unary<ops::identity<T>, T>
{
    static constexpr bool supported = true;
    static int launch(ops::identity<T> const&, int dev, void* s, T* dst, T const* src, std::size_t n)
    {
        return coloc_cuda_copy_bytes(dev, s, dst, src, n * sizeof(T));
    }
};

template <>
struct device_unary<ops::scale<double>, double>
{
    static constexpr bool supported = true;
    static int launch(ops::scale<double> const& f, int dev, void* s, double* dst,
        double const* src, std::size_t n)
    {
        return coloc_cuda_scale_f64(dev, s, dst, src, f.scalar, n);
    }
};

template <>
struct device_unary<ops::scale<float>, float>
{
    static constexpr bool supported = true;
    static int launch(ops::scale<float> const& f, int dev, void* s, float* dst,
        float const* src, std::size_t n)
    {
        return coloc_cuda_scale_f32(dev, s, dst, src, f.scalar, n);
    }
};

// Integer vectors (int, long, unsigned, ...): the i32/i64 kernels, the
// element bits reinterpreted (two's complement + and * are sign-agnostic).
template <typename T>
inline constexpr bool device_int_v = std::is_integral_v<T> && !std::is_same_v<T, bool> &&
    (sizeof(T) == 4 || sizeof(T) == 8);

template <typename T>
using device_int_t = std::conditional_t<sizeof(T) == 4, std::int32_t, std::int64_t>;

template <typename T>
    requires device_int_v<T>
struct device_unary<ops::scale<T>, T>
{
    static constexpr bool supported = true;
    static int launch(ops::scale<T> const& f, int dev, void* s, T* dst, T const* src, std::size_t n)
    {
        using I = device_int_t<T>;
        auto const k = static_cast<I>(f.scalar);
        if constexpr (sizeof(T) == 4)
            return coloc_cuda_scale_i32(dev, s, reinterpret_cast<I*>(dst), reinterpret_cast<I const*>(src), k, n);
        else
            return coloc_cuda_scale_i64(dev, s, reinterpret_cast<I*>(dst), reinterpret_cast<I const*>(src), k, n);
    }
};

template <typename C>
    requires(sizeof(C) == 1 && std::is_integral_v<C>)
struct device_unary<ops::to_upper, C>
{
    static constexpr bool supported = true;
    static int launch(ops::to_upper const&, int dev, void* s, C* dst, C const* src, std::size_t n)
    {
        return coloc_cuda_to_upper_u8(dev, s, reinterpret_cast<unsigned char*>(dst),
            reinterpret_cast<unsigned char const*>(src), n);
    }
};

template <typename F, typename T>
struct device_binary
{
    static constexpr bool supported = false;
};

template <typename T>
    requires(std::is_same_v<T, double> || std::is_same_v<T, float> || device_int_v<T>)
struct device_binary_add
{
    static constexpr bool supported = true;
    template <typename F>
    static int launch(F const&, int dev, void* s, T* dst, T const* a, T const* b, std::size_t n)
    {
        if constexpr (std::is_same_v<T, double>)
            return coloc_cuda_add_f64(dev, s, dst, a, b, n);
        else if constexpr (std::is_same_v<T, float>)
            return coloc_cuda_add_f32(dev, s, dst, a, b, n);
        else
        {
            using I = device_int_t<T>;
            auto* d = reinterpret_cast<I*>(dst);
            auto const* x = reinterpret_cast<I const*>(a);
            auto const* y = reinterpret_cast<I const*>(b);
            if constexpr (sizeof(T) == 4)
                return coloc_cuda_add_i32(dev, s, d, x, y, n);
            else
                return coloc_cuda_add_i64(dev, s, d, x, y, n);
        }
    }
};

template <typename T>
struct device_binary<ops::plus<T>, T> : device_binary_add<T>
{
};
template <typename T>
struct device_binary<std::plus<T>, T> : device_binary_add<T>
{
};
template <typename T>
struct device_binary<std::plus<>, T> : device_binary_add<T>
{
};

template <typename T, bool Fma>
    requires(std::is_same_v<T, double> || std::is_same_v<T, float>)
struct device_binary_triad
{
    static constexpr bool supported = true;
    template <typename F>
    static int launch(F const& f, int dev, void* s, T* dst, T const* b, T const* c, std::size_t n)
    {
        if constexpr (std::is_same_v<T, double>)
            return coloc_cuda_triad_f64(dev, s, dst, b, c, f.scalar, n, Fma ? 1 : 0);
        else
            return coloc_cuda_triad_f32(dev, s, dst, b, c, f.scalar, n, Fma ? 1 : 0);
    }
};

template <typename T>
    requires device_int_v<T>
struct device_binary_triad_int
{
    static constexpr bool supported = true;
    template <typename F>
    static int launch(F const& f, int dev, void* s, T* dst, T const* b, T const* c, std::size_t n)
    {
        using I = device_int_t<T>;
        auto* d = reinterpret_cast<I*>(dst);
        auto const* x = reinterpret_cast<I const*>(b);
        auto const* y = reinterpret_cast<I const*>(c);
        auto const k = static_cast<I>(f.scalar);
        if constexpr (sizeof(T) == 4)
            return coloc_cuda_triad_i32(dev, s, d, x, y, k, n);
        else
            return coloc_cuda_triad_i64(dev, s, d, x, y, k, n);
    }
};

template <typename T>
    requires(!device_int_v<T>)
struct device_binary<ops::triad<T>, T> : device_binary_triad<T, false>
{
};
template <typename T>
    requires device_int_v<T>
struct device_binary<ops::triad<T>, T> : device_binary_triad_int<T>
{
};
template <typename T>
struct device_binary<ops::triad_fma<T>, T> : device_binary_triad<T, true>
{
};

// for_each ops: in-place launches over one range.
template <typename F, typename T>
struct device_in_place
{
    static constexpr bool supported = false;
};

template <typename T>
struct device_in_place<ops::assign<T>, T>
{
    static constexpr bool supported = true;
    static int launch(ops::assign<T> const& f, int dev, void* s, T* x, std::size_t n)
    {
        static_assert(sizeof(T) == 1 || sizeof(T) == 2 || sizeof(T) == 4 || sizeof(T) == 8,
            "ops::assign on device supports 1/2/4/8-byte elements");
        return coloc_cuda_fill(dev, s, x, n, &f.value, sizeof(T));
    }
};

template <typename T>
struct device_in_place<ops::multiply_by<T>, T>
{
    static constexpr bool supported = device_unary<ops::scale<T>, T>::supported;
    static int launch(ops::multiply_by<T> const& f, int dev, void* s, T* x, std::size_t n)
    {
        return device_unary<ops::scale<T>, T>::launch(ops::scale<T>{f.scalar}, dev, s, x, x, n);
    }
};

template <typename C>
    requires(sizeof(C) == 1 && std::is_integral_v<C>)
struct device_in_place<ops::make_upper, C>
{
    static constexpr bool supported = true;
    static int launch(ops::make_upper const&, int dev, void* s, C* x, std::size_t n)
    {
        return coloc_cuda_to_upper_u8(dev, s, reinterpret_cast<unsigned char*>(x),
            reinterpret_cast<unsigned char const*>(x), n);
    }
};

}    // namespace coloc::detail

namespace coloc::cuda {

/// Device kernels for the generators vector::generate / bulk_generate
/// recognise (memory.hpp).  `first_index` is the generator index of `at`.
template <typename T, typename Gen>
void generate_on_device(segment<T> const& s, T* at, std::size_t first_index,
    std::size_t count, Gen const& gen)
{
    int st = COLOC_ERR_UNSUPPORTED;
    if constexpr (std::is_same_v<Gen, ops::uniform_random<double>> && std::is_same_v<T, double>)
        st = coloc_cuda_generate_random_f64(s.where.device(), s.where.stream(), at, count,
            gen.seed, gen.array, gen.first + first_index);
    else if constexpr (std::is_same_v<Gen, ops::uniform_random<float>> && std::is_same_v<T, float>)
        st = coloc_cuda_generate_random_f32(s.where.device(), s.where.stream(), at, count,
            gen.seed, gen.array, gen.first + first_index);
    else if constexpr (std::is_same_v<Gen, ops::iota<double>> && std::is_same_v<T, double>)
        st = coloc_cuda_iota_f64(s.where.device(), s.where.stream(), at, count,
            gen.first + double(first_index));
    else
        static_assert(sizeof(Gen) == 0, "no device kernel for this generator/element type");
    coloc::detail::check(st, "coloc::cuda bulk_generate");
}

}    // namespace coloc::cuda
