// SPDX-License-Identifier: Apache-2.0
// Restates the public interface of the reference coloc library's allocator_traits.hpp, block_allocator.hpp and device_allocator.hpp
// (arXiv 2206.06302; /root/reference/proj/include/coloc, Apache-2.0): the
// names, signatures and semantics are kept for drop-in compatibility.
// memory.hpp -- target-bound allocation on GPUs.
//
//   reference                                          here
//   allocator_traits (allocator_traits.hpp:44-153)     coloc::allocator_traits (same contract)
//   host::block_allocator (block_allocator.hpp:65-214) cuda::block_allocator: one cudaMalloc
//     one aligned operator new, first touch by           per target, construction by a fill
//     pinned workers                                      kernel on the owning GPU
//   device::device_allocator (device_allocator.hpp:    cuda::allocator: one target
//     113-245), arena + queue construction
//   device_ptr / device_proxy (24-108)                 segmented_ptr / device_proxy
//
// Storage of a block allocation is segmented: block i of
// partition_block(n, targets) lives in the HBM of targets[i].device()
// (hard part 3: per-GPU cudaMalloc instead of one
// contiguous allocation).  Segment i always corresponds to partition block
// i, including zero-length blocks.
#pragma once

#include "coloc_b200/errors.hpp"
#include "coloc_b200/index_space.hpp"
#include "coloc_b200/targets.hpp"

#include <cstddef>
#include <cstdint>
#include <cstring>
#include <memory>
#include <type_traits>
#include <utility>
#include <vector>

namespace coloc {

namespace ops {
template <typename T>
struct uniform_random;
template <typename T>
struct iota;
}    // namespace ops

namespace cuda {

/// Memory-space tag used by the algorithms' dispatch (algorithms.hpp:118-149).
struct cuda_memory_space
{
};

template <typename T>
struct segment
{
    target where;
    T* base = nullptr;    // device address of element `offset`
    std::size_t offset = 0;
    std::size_t length = 0;

    std::size_t end() const noexcept { return offset + length; }
};

namespace detail {

template <typename T>
class storage
{
public:
    storage(std::vector<target> const& targets, std::size_t n)
      : size_(n)
    {
        auto part = partition_block(n, targets);
        segs_.reserve(part.blocks.size());
        for (auto const& b : part.blocks)
        {
            segment<T> s{b.target, nullptr, b.offset, b.length};
            if (b.length != 0)
            {
                void* p = nullptr;
                std::size_t const bytes = b.length * sizeof(T);
                int st = coloc_cuda_malloc(b.target.device(), bytes, &p);
                if (st != COLOC_OK)
                {
                    release();
                    if (st == COLOC_ERR_ALLOCATION)
                        throw allocation_error(bytes, b.target.description());
                    coloc::detail::throw_status(st, "coloc::cuda allocate", bytes,
                        b.target.description());
                }
                s.base = static_cast<T*>(p);
            }
            segs_.push_back(std::move(s));
        }
    }

    ~storage() { release(); }
    storage(storage const&) = delete;
    storage& operator=(storage const&) = delete;

    std::vector<segment<T>> const& segments() const noexcept { return segs_; }
    std::size_t size() const noexcept { return size_; }

    /// Segment holding element i (i < size()).
    std::size_t locate(std::size_t i) const noexcept
    {
        std::size_t lo = 0, hi = segs_.size();
        while (lo < hi)
        {
            std::size_t mid = lo + (hi - lo) / 2;
            if (segs_[mid].end() <= i)
                lo = mid + 1;
            else
                hi = mid;
        }
        while (lo < segs_.size() && segs_[lo].length == 0)
            ++lo;
        return lo;
    }

private:
    void release() noexcept
    {
        for (auto& s : segs_)
            if (s.base)
            {
                (void) coloc_cuda_free(s.where.device(), s.base);
                s.base = nullptr;
            }
    }

    std::size_t size_;
    std::vector<segment<T>> segs_;
};

}    // namespace detail

/// Element handle into segmented device storage: (allocation, index).
/// Keeps the allocation alive.  Raw addresses are only for kernels.
template <typename T>
class segmented_ptr
{
public:
    segmented_ptr() = default;
    segmented_ptr(std::shared_ptr<detail::storage<T> const> st, std::size_t index) noexcept
      : st_(std::move(st))
      , index_(index)
    {
    }

    explicit operator bool() const noexcept { return st_ != nullptr; }
    std::size_t index() const noexcept { return index_; }
    detail::storage<T> const& storage() const noexcept { return *st_; }
    std::vector<segment<T>> const& segments() const noexcept { return st_->segments(); }

    /// Segment number (== partition block) holding element index()+d.
    std::size_t segment_of(std::size_t d = 0) const noexcept
    {
        return st_->locate(index_ + d);
    }

    /// Device address of element index()+d.
    T* raw(std::size_t d = 0) const noexcept
    {
        auto const& s = st_->segments()[segment_of(d)];
        return s.base + (index_ + d - s.offset);
    }

    segmented_ptr operator+(std::ptrdiff_t d) const noexcept
    {
        return segmented_ptr(st_, index_ + std::size_t(d));
    }
    segmented_ptr& operator+=(std::ptrdiff_t d) noexcept
    {
        index_ += std::size_t(d);
        return *this;
    }

    friend bool operator==(segmented_ptr const& a, segmented_ptr const& b) noexcept
    {
        return a.st_ == b.st_ && a.index_ == b.index_;
    }

private:
    std::shared_ptr<detail::storage<T> const> st_;
    std::size_t index_ = 0;
};

/// Staged element access (device_allocator.hpp:79-108): reads and writes
/// are ordered on the owning target's stream, then waited for.
template <typename T>
class device_proxy
{
public:
    explicit device_proxy(segmented_ptr<T> p) noexcept
      : p_(std::move(p))
    {
    }

    operator T() const
    {
        auto const& s = p_.segments()[p_.segment_of()];
        T value;
        coloc::detail::check(coloc_cuda_memcpy_async(s.where.device(), s.where.stream(),
                                 &value, p_.raw(), sizeof(T)),
            "coloc::cuda::device_proxy read");
        s.where.synchronize();
        return value;
    }

    device_proxy& operator=(T const& value)
    {
        auto const& s = p_.segments()[p_.segment_of()];
        T staged = value;
        coloc::detail::check(coloc_cuda_memcpy_async(s.where.device(), s.where.stream(),
                                 p_.raw(), &staged, sizeof(T)),
            "coloc::cuda::device_proxy write");
        s.where.synchronize();
        return *this;
    }

    device_proxy& operator=(device_proxy const& rhs) { return *this = static_cast<T>(rhs); }

private:
    segmented_ptr<T> p_;
};

namespace detail {

// Fill n elements starting at p with one bit pattern, per owning segment.
template <typename T>
void fill_segments(segmented_ptr<T> const& p, std::size_t n, T const& value)
{
    if (n == 0)
        return;
    std::size_t const lo = p.index(), hi = lo + n;
    std::vector<target const*> touched;
    for (auto const& s : p.segments())
    {
        std::size_t const b = std::max(lo, s.offset), e = std::min(hi, s.end());
        if (b >= e)
            continue;
        T* at = s.base + (b - s.offset);
        int st;
        if constexpr (sizeof(T) == 1 || sizeof(T) == 2 || sizeof(T) == 4 ||
            sizeof(T) == 8)
            st = coloc_cuda_fill(s.where.device(), s.where.stream(), at, e - b, &value,
                sizeof(T));
        else
        {
            // Odd-sized elements: stage one pinned copy and replicate by
            // doubling device-to-device copies.
            st = coloc_cuda_memcpy_async(s.where.device(), s.where.stream(), at, &value,
                sizeof(T));
            if (st == COLOC_OK)
                s.where.synchronize();
            for (std::size_t have = 1; st == COLOC_OK && have < e - b; have *= 2)
                st = coloc_cuda_copy_bytes(s.where.device(), s.where.stream(), at + have,
                    at, std::min(have, e - b - have) * sizeof(T));
        }
        coloc::detail::check(st, "coloc::cuda bulk_construct");
        touched.push_back(&s.where);
    }
    for (auto const* t : touched)
        t->synchronize();
}

template <typename G>
struct is_device_generator : std::false_type
{
};
template <typename T>
struct is_device_generator<ops::uniform_random<T>> : std::true_type
{
};
template <typename T>
struct is_device_generator<ops::iota<T>> : std::true_type
{
};

}    // namespace detail

template <typename T>
class block_allocator;

// Generators with a device kernel (defined in ops.hpp) implement this.
template <typename T, typename Gen>
void generate_on_device(segment<T> const& s, T* at, std::size_t first_index,
    std::size_t count, Gen const& gen);

/// Allocator over an ordered list of GPU targets using the block scheme
/// (block_allocator.hpp:65-214): element range split by partition_block,
/// block i allocated in, and constructed by, targets[i]'s GPU.
template <typename T>
class block_allocator
{
    static_assert(std::is_trivially_copyable_v<T>,
        "device storage holds trivially copyable element types only");

public:
    using value_type = T;
    using pointer = segmented_ptr<T>;
    using const_pointer = segmented_ptr<T>;
    using reference = device_proxy<T>;
    using const_reference = T;    // const reads materialise the value
    using size_type = std::size_t;
    using difference_type = std::ptrdiff_t;
    using target_type = std::vector<cuda::target>;
    using memory_space = cuda_memory_space;

    template <typename U>
    struct rebind
    {
        using other = block_allocator<U>;
    };

    explicit block_allocator(cuda::target t)
      : block_allocator(target_type{std::move(t)})
    {
    }

    explicit block_allocator(target_type targets)
    {
        if (targets.empty())
            throw invalid_target_error("cuda block allocator requires at least one target");
        for (auto const& t : targets)
            if (!t.valid())
                throw invalid_target_error("cuda block allocator: default-constructed target");
        targets_ = std::make_shared<target_type const>(std::move(targets));
    }

    template <typename U>
    block_allocator(block_allocator<U> const& other) noexcept
      : targets_(other.targets_)
    {
    }

    pointer allocate(size_type n)
    {
        return pointer(std::make_shared<detail::storage<T> const>(*targets_, n), 0);
    }

    /// Storage is released when the last handle into it is dropped, so
    /// work still queued on a stream never sees freed memory.
    void deallocate(pointer, size_type) noexcept {}

    target_type const& target() const noexcept { return *targets_; }

    partition<cuda::target> partition_of(size_type n) const
    {
        return partition_block(n, *targets_);
    }

    /// Every element of [p, p+n) set to T(vs...), on the owning GPUs
    /// ("first touch", block_allocator.hpp:127-133).  Blocks until done,
    /// like the reference's construction (.get(), block_allocator.hpp:444).
    template <typename... Ts>
    void bulk_construct(pointer p, size_type n, Ts const&... vs)
    {
        T const value(vs...);
        detail::fill_segments(p, n, value);
    }

    /// Element i built from gen(i) (block_allocator.hpp:135-141).  Device
    /// generators (ops::uniform_random, ops::iota) run as kernels on the
    /// owning GPU; any other callable is evaluated on the host per block and
    /// staged over (initializer lists, arbitrary user functions).
    template <typename Gen>
    void bulk_generate(pointer p, size_type n, Gen gen)
    {
        std::size_t const lo = p.index(), hi = lo + n;
        std::vector<cuda::target const*> touched;
        for (auto const& s : p.segments())
        {
            std::size_t const b = std::max(lo, s.offset), e = std::min(hi, s.end());
            if (b >= e)
                continue;
            T* at = s.base + (b - s.offset);
            if constexpr (detail::is_device_generator<Gen>::value)
                generate_on_device(s, at, b - lo, e - b, gen);
            else
            {
                std::vector<T> staged(e - b);
                for (std::size_t i = b; i < e; ++i)
                    staged[i - b] = T(gen(i - lo));
                coloc::detail::check(coloc_cuda_memcpy_async(s.where.device(),
                                         s.where.stream(), at, staged.data(),
                                         staged.size() * sizeof(T)),
                    "coloc::cuda bulk_generate");
                s.where.synchronize();
            }
            touched.push_back(&s.where);
        }
        for (auto const* t : touched)
            t->synchronize();
    }

    void bulk_destroy(pointer, size_type) noexcept {}

    reference make_reference(pointer p, size_type i) const
    {
        return reference(p + std::ptrdiff_t(i));
    }

    const_reference make_const_reference(pointer p, size_type i) const
    {
        return static_cast<T>(reference(p + std::ptrdiff_t(i)));
    }

    friend bool operator==(block_allocator const& a, block_allocator const& b) noexcept
    {
        return *a.targets_ == *b.targets_;
    }

private:
    template <typename>
    friend class block_allocator;
    template <typename>
    friend class allocator;

    std::shared_ptr<target_type const> targets_;
};

/// Single-GPU allocator: the device_allocator analogue
/// (device_allocator.hpp:113-245) with target_type = cuda::target.
template <typename T>
class allocator
{
public:
    using value_type = T;
    using pointer = segmented_ptr<T>;
    using const_pointer = segmented_ptr<T>;
    using reference = device_proxy<T>;
    using const_reference = T;
    using size_type = std::size_t;
    using difference_type = std::ptrdiff_t;
    using target_type = cuda::target;
    using memory_space = cuda_memory_space;

    template <typename U>
    struct rebind
    {
        using other = allocator<U>;
    };

    explicit allocator(cuda::target t)
      : impl_(t)
      , target_(std::move(t))
    {
    }

    template <typename U>
    allocator(allocator<U> const& other)
      : impl_(other.impl_)
      , target_(other.target_)
    {
    }

    pointer allocate(size_type n) { return impl_.allocate(n); }
    void deallocate(pointer p, size_type n) noexcept { impl_.deallocate(p, n); }
    target_type const& target() const noexcept { return target_; }

    template <typename... Ts>
    void bulk_construct(pointer p, size_type n, Ts const&... vs)
    {
        impl_.bulk_construct(p, n, vs...);
    }
    template <typename Gen>
    void bulk_generate(pointer p, size_type n, Gen gen)
    {
        impl_.bulk_generate(p, n, std::move(gen));
    }
    void bulk_destroy(pointer, size_type) noexcept {}
    reference make_reference(pointer p, size_type i) const { return impl_.make_reference(p, i); }
    const_reference make_const_reference(pointer p, size_type i) const
    {
        return impl_.make_const_reference(p, i);
    }

    friend bool operator==(allocator const& a, allocator const& b) noexcept
    {
        return a.target_ == b.target_;
    }

private:
    template <typename>
    friend class allocator;

    block_allocator<T> impl_;
    cuda::target target_;
};

/// Standard allocator of page-locked host memory (coloc_cuda_host_alloc:
/// huge-page backed and registered for >= 64 MiB): a reference user's
/// `std::vector<T, cuda::pinned_allocator<T>>` is copied to and from GPU
/// vectors by the copy engines directly, at the PCIe rate and overlapped
/// with kernels under a stream-ordered executor, where ordinary pageable
/// vectors go through the library's staging workers (bounded by host
/// memory bandwidth).
template <typename T>
struct pinned_allocator
{
    using value_type = T;

    pinned_allocator() noexcept = default;
    template <typename U>
    pinned_allocator(pinned_allocator<U> const&) noexcept
    {
    }

    T* allocate(std::size_t n)
    {
        void* p = nullptr;
        coloc::detail::check(coloc_cuda_host_alloc(n * sizeof(T), &p), "pinned_allocator");
        return static_cast<T*>(p);
    }
    void deallocate(T* p, std::size_t) noexcept { (void) coloc_cuda_host_free(p); }

    template <typename U>
    bool operator==(pinned_allocator<U> const&) const noexcept
    {
        return true;
    }
};

}    // namespace cuda

namespace detail {

template <typename A, typename = void>
struct alloc_reference
{
    using type = typename A::value_type&;
};
template <typename A>
struct alloc_reference<A, std::void_t<typename A::reference>>
{
    using type = typename A::reference;
};
template <typename A, typename = void>
struct alloc_const_reference
{
    using type = typename A::value_type const&;
};
template <typename A>
struct alloc_const_reference<A, std::void_t<typename A::const_reference>>
{
    using type = typename A::const_reference;
};

}    // namespace detail

/// std::allocator_traits plus the target binding and bulk construction
/// interface (allocator_traits.hpp:44-153).  Members an allocator lacks
/// fall back to the standard element-wise behaviour.
template <typename Allocator>
struct allocator_traits : std::allocator_traits<Allocator>
{
    using base_type = std::allocator_traits<Allocator>;
    using typename base_type::pointer;
    using typename base_type::size_type;
    using typename base_type::value_type;
    using reference = typename detail::alloc_reference<Allocator>::type;
    using const_reference = typename detail::alloc_const_reference<Allocator>::type;
    using target_type = typename Allocator::target_type;

    static decltype(auto) target(Allocator const& a) { return a.target(); }

    template <typename... Ts>
    static void bulk_construct(Allocator& a, pointer p, size_type n, Ts&&... vs)
    {
        if constexpr (requires { a.bulk_construct(p, n, vs...); })
            a.bulk_construct(p, n, std::forward<Ts>(vs)...);
        else
        {
            size_type i = 0;
            try
            {
                for (; i < n; ++i)
                    base_type::construct(a, std::addressof(p[i]), vs...);
            }
            catch (...)
            {
                while (i > 0)
                    base_type::destroy(a, std::addressof(p[--i]));
                throw;
            }
        }
    }

    template <typename Gen>
    static void bulk_generate(Allocator& a, pointer p, size_type n, Gen&& gen)
    {
        if constexpr (requires { a.bulk_generate(p, n, gen); })
            a.bulk_generate(p, n, std::forward<Gen>(gen));
        else
        {
            size_type i = 0;
            try
            {
                for (; i < n; ++i)
                    base_type::construct(a, std::addressof(p[i]), gen(i));
            }
            catch (...)
            {
                while (i > 0)
                    base_type::destroy(a, std::addressof(p[--i]));
                throw;
            }
        }
    }

    static void bulk_destroy(Allocator& a, pointer p, size_type n) noexcept
    {
        if constexpr (requires { a.bulk_destroy(p, n); })
            a.bulk_destroy(p, n);
        else
            for (size_type i = 0; i < n; ++i)
                base_type::destroy(a, std::addressof(p[i]));
    }

    static reference make_reference(Allocator& a, pointer p, size_type i)
    {
        if constexpr (requires { a.make_reference(p, i); })
            return a.make_reference(p, i);
        else
            return p[i];
    }

    static const_reference make_const_reference(Allocator const& a, pointer p, size_type i)
    {
        if constexpr (requires { a.make_const_reference(p, i); })
            return a.make_const_reference(p, i);
        else
            return p[i];
    }
};

}    // namespace coloc
