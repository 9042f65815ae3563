// SPDX-License-Identifier: Apache-2.0
// Restates the public interface of the reference coloc library's partition.hpp and shape.hpp
// (arXiv 2206.06302; /root/reference/proj/include/coloc, Apache-2.0): the
// names, signatures and semantics are kept for drop-in compatibility.
// index_space.hpp -- how an index range is split across targets and work
// items.  Same arithmetic as the reference, so block ownership matches the
// CPU oracle element for element:
//   partition / partition_block   include/coloc/partition.hpp:17-76
//   index_range / shape / chunk_range   include/coloc/shape.hpp:14-64
#pragma once

#include <algorithm>
#include <cstddef>
#include <stdexcept>
#include <vector>

namespace coloc {

/// Tag for work not bound to any partition block.
inline constexpr std::size_t no_block = ~std::size_t(0);

/// Ordered, contiguous, disjoint split of [0, n) over a target list;
/// block i belongs to the i-th target.
template <typename Target>
struct partition
{
    struct block
    {
        Target target;
        std::size_t offset = 0;
        std::size_t length = 0;

        std::size_t end() const noexcept { return offset + length; }
    };

    std::vector<block> blocks;

    std::size_t size() const noexcept { return blocks.size(); }

    std::size_t total() const noexcept
    {
        std::size_t sum = 0;
        for (block const& b : blocks)
            sum += b.length;
        return sum;
    }

    /// Block holding element `index`, or no_block past the end.  Zero-length
    /// blocks never own an element.
    std::size_t block_of(std::size_t index) const noexcept
    {
        std::size_t lo = 0, hi = blocks.size();
        while (lo < hi)    // first block whose end() exceeds index
        {
            std::size_t mid = lo + (hi - lo) / 2;
            if (blocks[mid].end() <= index)
                lo = mid + 1;
            else
                hi = mid;
        }
        if (lo == blocks.size() || index < blocks[lo].offset)
            return no_block;
        return lo;
    }
};

/// Even split of n elements over k = targets.size() blocks: the first
/// n mod k blocks hold ceil(n/k) elements, the rest floor(n/k).
/// Throws std::invalid_argument for an empty target list.
template <typename Target>
partition<Target> partition_block(std::size_t n, std::vector<Target> const& targets)
{
    if (targets.empty())
        throw std::invalid_argument("partition_block: empty target list");
    std::size_t const k = targets.size();
    std::size_t const quotient = n / k;
    std::size_t const extra = n % k;
    partition<Target> out;
    out.blocks.reserve(k);
    std::size_t at = 0;
    for (std::size_t i = 0; i < k; ++i)
    {
        std::size_t const len = quotient + (i < extra ? 1 : 0);
        out.blocks.push_back({targets[i], at, len});
        at += len;
    }
    return out;
}

/// Half-open range of indices, tagged with the partition block whose
/// target runs it.
struct index_range
{
    std::size_t begin = 0;
    std::size_t end = 0;
    std::size_t block = no_block;

    std::size_t size() const noexcept { return end - begin; }
    friend bool operator==(index_range const&, index_range const&) = default;
};

/// Work shape for bulk submission: disjoint ranges.
using shape = std::vector<index_range>;

inline std::size_t shape_size(shape const& s) noexcept
{
    std::size_t n = 0;
    for (index_range const& r : s)
        n += r.size();
    return n;
}

inline shape single_range(std::size_t n, std::size_t block = no_block)
{
    return n == 0 ? shape{} : shape{index_range{0, n, block}};
}

/// Appends [begin, end) cut into min(max(parts, 1), end-begin) pieces,
/// longer pieces first, each tagged with `block`.
inline void chunk_range(shape& out, std::size_t begin, std::size_t end,
    std::size_t parts, std::size_t block = no_block)
{
    if (end <= begin)
        return;
    std::size_t const n = end - begin;
    parts = std::clamp<std::size_t>(parts, 1, n);
    std::size_t const quotient = n / parts;
    std::size_t const extra = n % parts;
    for (std::size_t i = 0, at = begin; i < parts; ++i)
    {
        std::size_t const len = quotient + (i < extra ? 1 : 0);
        out.push_back({at, at + len, block});
        at += len;
    }
}

}    // namespace coloc
