/*
 * stream_native.h -- the hand-written "native" CUDA STREAM baseline
 * (paper_2206_06302_b200/csrc/native_stream.cu, libstream_native.so).
 *
 * MEASUREMENT BASELINE, not part of the drop-in: it stands for the
 * reference CUDA STREAM the paper compares its abstraction against
 * and for SPEC's run_baseline:
 * plain arrays, plain kernels, no allocator / executor / algorithm layer,
 * timed identically to coloc_stream_blocking_run (host steady clock around
 * each blocking kernel call, first iteration excluded).
 */
#ifndef STREAM_NATIVE_H
#define STREAM_NATIVE_H

#include "coloc_stream.h"

#ifdef __cplusplus
extern "C" {
#endif

/* dtype: COLOC_STREAM_F64 / F32; arrays a=1, b=2, c=0 of n elements on
 * `dev`; `iterations` Listing-4 iterations; timings and validation in out. */
int stream_native_run(int dtype, int dev, uint64_t n, int iterations,
    coloc_stream_timing* out);
const char* stream_native_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* STREAM_NATIVE_H */
