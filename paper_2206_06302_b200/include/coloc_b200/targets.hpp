// targets.hpp -- places on the GPU side of the system.
//
// The reference names a device place as {device_id, queue_id}
// (include/coloc/device.hpp:29-41) backed by a mock FIFO thread, and the
// paper defines a CUDA target as "a wrapper for an integer representing the
// device and a CUDA stream attached to that device".
// That is exactly cuda::target: an ordinal plus a shared, non-blocking
// stream.  get_targets() is the GPU counterpart of get_targets(topology)
// (topology.hpp:620, src/topology.cpp:208-221): one target per GPU.
#pragma once

#include "coloc_b200/errors.hpp"

#include <cstddef>
#include <memory>
#include <string>
#include <vector>

namespace coloc::cuda {

inline int device_count()
{
    int n = 0;
    detail::check(coloc_cuda_device_count(&n), "coloc::cuda::device_count");
    return n;
}

inline coloc_cuda_device_info device_info(int dev)
{
    coloc_cuda_device_info info{};
    detail::check(coloc_cuda_device_info_get(dev, &info), "coloc::cuda::device_info");
    return info;
}

namespace detail {

/// Owns one cudaStream_t; destroyed with the last target copy using it.
class stream_owner
{
public:
    explicit stream_owner(int dev)
      : dev_(dev)
    {
        int st = coloc_cuda_stream_create(dev, &stream_);
        if (st != COLOC_OK)
            coloc::detail::throw_status(st == COLOC_ERR_INVALID_ARGUMENT ?
                    COLOC_ERR_INVALID_TARGET :
                    st,
                "cuda target " + std::to_string(dev));
    }
    ~stream_owner() { (void) coloc_cuda_stream_destroy(dev_, stream_); }
    stream_owner(stream_owner const&) = delete;
    stream_owner& operator=(stream_owner const&) = delete;

    void* get() const noexcept { return stream_; }

private:
    int dev_;
    void* stream_ = nullptr;
};

}    // namespace detail

/// A GPU place: device ordinal + in-order stream.  Copies share the stream,
/// so work submitted through any copy is ordered (the fifo_queue guarantee,
/// device.hpp:26-28).
class target
{
public:
    target() = default;

    /// Fresh stream on `device` (system::make_target, src/device.cpp:173-177).
    /// Throws invalid_target_error when the device does not exist.
    explicit target(int device)
      : device_(device)
      , stream_(std::make_shared<detail::stream_owner>(device))
    {
    }

    int device() const noexcept { return device_; }
    void* stream() const noexcept { return stream_ ? stream_->get() : nullptr; }
    bool valid() const noexcept { return stream_ != nullptr; }

    /// Blocks until all work submitted to this target has finished.
    void synchronize() const
    {
        coloc::detail::check(coloc_cuda_stream_sync(device_, stream()),
            "coloc::cuda::target::synchronize");
    }

    std::string description() const
    {
        return "cuda:" + std::to_string(device_);
    }

    friend bool operator==(target const& a, target const& b) noexcept
    {
        return a.device_ == b.device_ && a.stream_ == b.stream_;
    }

private:
    int device_ = -1;
    std::shared_ptr<detail::stream_owner> stream_;
};

/// Fresh-stream target for one device (device::make_device_target,
/// device.hpp:177-180).
inline target make_target(int device)
{
    return target(device);
}

/// One target per visible GPU, in ordinal order.
inline std::vector<target> get_targets()
{
    std::vector<target> out;
    int const n = device_count();
    out.reserve(std::size_t(n));
    for (int d = 0; d < n; ++d)
        out.emplace_back(d);
    return out;
}

/// One target (with its own stream) per listed ordinal; repeating an
/// ordinal places several blocks on one GPU.
inline std::vector<target> make_targets(std::vector<int> const& devices)
{
    std::vector<target> out;
    out.reserve(devices.size());
    for (int d : devices)
        out.emplace_back(d);
    return out;
}

}    // namespace coloc::cuda
