// staging.h -- pinned staging of pageable host memory (staging.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace coloc_cuda {

// Copies of at least this many bytes with a pageable host side go through
// the staging ring.
constexpr std::size_t kStageMinBytes = std::size_t(4) << 20;

bool is_pageable_host(void const* p);
bool is_device_memory(void const* p);
int staged_h2d(int dev, cudaStream_t stream, void* dst, void const* src, std::size_t bytes);
int staged_d2h(int dev, cudaStream_t stream, void* dst, void const* src, std::size_t bytes);

}    // namespace coloc_cuda
