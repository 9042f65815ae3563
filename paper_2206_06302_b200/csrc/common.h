// common.h -- status plumbing shared by the C-ABI translation units.
//
// Every C entry point returns an int status and leaves a thread-local
// message (coloc_cuda_last_error).  CUDA errors are mapped onto the
// reference's error taxonomy (error.hpp:11-57) so the C++ layer can
// rethrow allocation_error / invalid_target_error / submission_error.
#pragma once

#include "coloc_cuda.h"

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>

namespace coloc_cuda {

void set_error(std::string msg);
void clear_error();
int status_of(cudaError_t e);
int fail(int status, std::string const& msg);
int fail_cuda(cudaError_t e, char const* what);

// Makes `dev` current on this thread (cheap when it already is).
int use_device(int dev);

struct device_props
{
    int sm_count = 0;
    int max_threads_per_sm = 0;
    std::size_t l2_bytes = 0;
};
// Cached per-device properties; nullptr when dev is invalid.
device_props const* props(int dev);

extern std::atomic<std::uint64_t> g_launches;

// Drops the tile-chain state of a stream being destroyed (kernels.cu), so a
// later stream with the same handle value starts clean.
void chain_forget(int dev, void* stream);

}    // namespace coloc_cuda

#define COLOC_TRY_CUDA(expr, what)                                             \
    do                                                                         \
    {                                                                          \
        cudaError_t coloc_e_ = (expr);                                         \
        if (coloc_e_ != cudaSuccess)                                           \
            return ::coloc_cuda::fail_cuda(coloc_e_, what);                    \
    } while (0)

#define COLOC_TRY(expr)                                                        \
    do                                                                         \
    {                                                                          \
        int coloc_s_ = (expr);                                                 \
        if (coloc_s_ != COLOC_OK)                                              \
            return coloc_s_;                                                   \
    } while (0)
