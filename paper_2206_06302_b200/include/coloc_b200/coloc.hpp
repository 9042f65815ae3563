// coloc.hpp -- umbrella header of the B200-native drop-in for the
// reference's STREAM hot path (targets, allocators, vector, executors,
// copy / transform / for_each).  Calls nothing but the C ABI in
// include/coloc_cuda.h.
#pragma once

#include "coloc_b200/container.hpp"
#include "coloc_b200/errors.hpp"
#include "coloc_b200/executors.hpp"
#include "coloc_b200/index_space.hpp"
#include "coloc_b200/memory.hpp"
#include "coloc_b200/ops.hpp"
#include "coloc_b200/parallel.hpp"
#include "coloc_b200/schedule_log.hpp"
#include "coloc_b200/targets.hpp"

// nvcc users may pass their own __device__ lambdas.
#if defined(__CUDACC__)
#include "coloc_b200/device_lambda.cuh"
#endif
