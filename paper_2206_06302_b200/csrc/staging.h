// staging.h -- pinned staging of pageable host memory (staging.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace coloc_cuda {

// Copies of at least this many bytes with a pageable host side go through
// the staging ring.
constexpr std::size_t kStageMinBytes = std::size_t(4) << 20;

// Frees every staging ring once its copies are done (they are set up
// again on the next staged copy).
int staging_release();

bool is_pageable_host(void const* p);
bool is_device_memory(void const* p);
// Stream-ordered staged copy (pinned-memory semantics: returns at once,
// the host buffer must stay valid until the stream has passed the copy).
int staged_enqueue(int dev, cudaStream_t stream, void* dst, void const* src, std::size_t bytes,
    bool h2d);
// cudaMemcpyAsync's pageable semantics (H2D returns once the source is
// consumed, D2H once the data has arrived).
int staged_h2d(int dev, cudaStream_t stream, void* dst, void const* src, std::size_t bytes);
int staged_d2h(int dev, cudaStream_t stream, void* dst, void const* src, std::size_t bytes);

}    // namespace coloc_cuda
