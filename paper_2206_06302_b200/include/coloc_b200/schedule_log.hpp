// schedule_log.hpp -- co-location audit of GPU launches.
//
// The reference's recording scheduler (include/coloc/schedule_log.hpp:19-81,
// enabled by COLOC_RECORD_SCHEDULE, src/schedule_log.cpp:14) logs which
// place ran which index range, so tests can check that every work item of
// block i ran on block i's target (criterion 6).  Here a record
// is one kernel launch (or staged copy) piece: the index range, the
// partition block, the target that executed it (device + stream) and the
// device holding the destination data.  Off unless enabled; recording costs
// a mutex per launch, so it is not meant for timed runs.
#pragma once

#include <cstddef>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

namespace coloc {

struct launch_record
{
    std::size_t begin = 0;    // relative to the algorithm's first element
    std::size_t end = 0;
    std::size_t block = 0;    // partition block of the destination range
    int device = -1;          // executing target
    void* stream = nullptr;
    int data_device = -1;     // owner of the destination elements
    void* data_stream = nullptr;
    std::string what;
};

class schedule_log
{
public:
    static schedule_log& global()
    {
        static schedule_log log(std::getenv("COLOC_RECORD_SCHEDULE") != nullptr);
        return log;
    }

    explicit schedule_log(bool enabled = false)
      : enabled_(enabled)
    {
    }

    bool enabled() const noexcept { return enabled_; }
    void set_enabled(bool on) noexcept { enabled_ = on; }

    void record(launch_record r)
    {
        std::lock_guard<std::mutex> lock(mu_);
        entries_.push_back(std::move(r));
    }

    std::vector<launch_record> entries() const
    {
        std::lock_guard<std::mutex> lock(mu_);
        return entries_;
    }

    void clear()
    {
        std::lock_guard<std::mutex> lock(mu_);
        entries_.clear();
    }

private:
    bool enabled_;
    mutable std::mutex mu_;
    std::vector<launch_record> entries_;
};

}    // namespace coloc
