/*
 * coloc_stream.h -- C ABI of the STREAM driver built on the C++ drop-in
 * layer (paper_2206_06302_b200/csrc/stream_driver.cpp).
 *
 * The reference does not ship a STREAM driver; it exists as the paper's
 * Listing 4 and the SPEC's stream_bench module
 * (run_stream 529-537, validate 539-547, bytes 516-520).
 * This ABI exposes that driver so harnesses (bench.py, tests) can run the
 * hot path exactly the way a C++ user of the drop-in API does:
 * coloc::vector over cuda::block_allocator, cuda_block_executor, and
 * coloc::copy / coloc::transform with par.on(exec).
 */
#ifndef COLOC_STREAM_H
#define COLOC_STREAM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum coloc_stream_dtype
{
    COLOC_STREAM_F64 = 0,
    COLOC_STREAM_F32 = 1
};

enum coloc_stream_reduction_mode
{
    COLOC_STREAM_REDUCE_AUTO = 0, /* NCCL when the blocks sit on distinct GPUs, else the host */
    COLOC_STREAM_REDUCE_HOST = 1, /* host sums in block order */
    COLOC_STREAM_REDUCE_NCCL = 2  /* always ncclAllReduce (needs one target per GPU) */
};

enum coloc_stream_init
{
    COLOC_STREAM_INIT_STREAM = 0, /* a=1, b=2, c=0 */
    COLOC_STREAM_INIT_RANDOM = 1  /* seeded splitmix64 in [-1,1) */
};

typedef struct coloc_stream_config
{
    int dtype;           /* coloc_stream_dtype */
    int init;            /* coloc_stream_init */
    int fma;             /* triad as fma(c, s, b) instead of b + (c*s) */
    int synchronous;     /* 1: each algorithm call blocks (reference semantics) */
    int ntargets;        /* targets (GPU + stream) in this process */
    const int* devices;  /* device ordinal of each target */
    uint64_t count;      /* elements held by this process, split over its targets */
    uint64_t first;      /* global index of this process's first element */
    uint64_t seed;       /* COLOC_STREAM_INIT_RANDOM */
    double scalar;       /* 3.0 in Listing 4 */
    double triad_scalar; /* scalar used by Triad; == scalar unless fault-injecting */
    int host_buffers;    /* host in/out arrays for e2e steps: 1 pinned, 2 pageable (new[]) */
    int reduction;       /* coloc_stream_reduction: how validation sums of this
                            process's blocks are combined */
    int chain;           /* 1: iterate_many chains its kernels tile by tile on each target
                            (coloc_cuda_chain_begin/end around the iterations); 2: only where
                            chains pay (per-target arrays of ~1-16 L2 sizes, and not with
                            events around every kernel); 0: never */
} coloc_stream_config;

/* Builds the three vectors (constructed on their owning GPUs). */
int coloc_stream_create(const coloc_stream_config* cfg, void** handle);
int coloc_stream_destroy(void* handle);
const char* coloc_stream_last_error(void);

/* One Listing-4 iteration: Copy c=a, Scale b=s*c, Add c=a+b, Triad a=b+s*c.
 * record 1 brackets each kernel with CUDA events on every target; record 2
 * brackets only the whole iteration (no event between the kernels, so
 * programmatic dependent launch can overlap consecutive kernels); record 3
 * times every kernel by completion stamps recorded on a per-target side
 * stream (coloc_cuda_stream_fork_timestamp): kernel k spans kernel k-1's
 * completion to its own, with no event node between the kernels; record 4
 * (iterate_many only) times every kernel from inside (earliest CTA start
 * to latest CTA end, %globaltimer, coloc_cuda_span_begin) -- no event at
 * all; coloc_stream_iteration_ms then returns the sum of the four. */
int coloc_stream_iterate(void* handle, int record);
/* `iterations` iterations at once; graph != 0 (stream-ordered config)
 * captures them -- with their timing events -- into one CUDA graph per
 * target and replays those, removing host launch overhead from the device
 * timeline for any number of targets and GPUs. */
int coloc_stream_iterate_many(void* handle, int iterations, int record, int graph);
/* Waits for all targets. */
int coloc_stream_sync(void* handle);
/* Recorded iterations so far, and per-kernel device time (ms) of recorded
 * iteration i: max over this process's targets.  Syncs. */
int coloc_stream_recorded(void* handle, int* count);
int coloc_stream_kernel_ms(void* handle, int i, double ms[4]);
/* Span of recorded iteration i (first kernel start to last kernel stop),
 * max over this process's targets; either record mode.  Syncs. */
int coloc_stream_iteration_ms(void* handle, int i, double* ms);
void coloc_stream_clear_records(void* handle);
/* Iterations executed since creation (recorded or not). */
int coloc_stream_iterations(void* handle, int* count);

/* End-to-end step through the public API from the host buffers
 * (cfg.host_buffers: pinned or pageable): copy host->device (a, b, c),
 * `ntimes` iterations, copy device->host (a, b, c); device time bracketed
 * by events on every target (max).  With pinned buffers and a
 * stream-ordered executor the step is captured into per-target CUDA graphs
 * before the timed region; pageable buffers go through the staging
 * workers, stream-ordered. */
int coloc_stream_e2e_step(void* handle, int ntimes, double* ms);

/* Validation: expected[3] from the recurrence for the
 * executed iteration count; sums[3] = sum |x - expected| over this
 * process's elements (fused kernel per block, f64).  If dev_out is
 * non-NULL it must be 3 doubles of device memory on the first target's
 * GPU and receives the sums too (for a cross-process allreduce). */
int coloc_stream_err_sums(void* handle, double expected[3], double sums[3],
    double* dev_out);
/* Position-sensitive checksums of a, b, c over this process's elements,
 * global indices from cfg.first (oracle_checksum_bits*). */
int coloc_stream_checksums(void* handle, uint64_t out[3]);
/* Copies elements [first, first+n) of array k (0=a, 1=b, 2=c; local
 * index) into host memory `out`. */
int coloc_stream_read(void* handle, int k, uint64_t first, uint64_t n, void* out);

/* One process per GPU: `comm` (coloc_cuda_nccl_init_rank) makes
 * coloc_stream_err_sums sum the per-process sums over all ranks with
 * NCCL, so every rank gets the job's totals.  NULL detaches.  The
 * communicator stays owned by the caller. */
int coloc_stream_set_comm(void* handle, void* comm);
/* How the last coloc_stream_err_sums combined its sums: "host", "nccl",
 * "host+ranks", "nccl+ranks" ("none" before the first call). */
const char* coloc_stream_reduction(void* handle);

/* ------------------------------------------------------------------ */
/* Abstraction vs native: the same   */
/* blocking, host-clock timing for the drop-in, the direct C-ABI calls   */
/* and the native CUDA STREAM (stream_native.h).                         */
/* ------------------------------------------------------------------ */

typedef struct coloc_stream_timing
{
    double min_s[4];    /* per kernel (copy, scale, add, triad), first iteration excluded */
    double avg_s[4];
    double max_s[4];
    double max_rel_err; /* max over a, b, c and elements of |x - e| / |e| (SPEC validate) */
    int validated;      /* max_rel_err <= 1e-8 (f64) / 1e-6 (f32) */
} coloc_stream_timing;

enum coloc_stream_arm
{
    COLOC_STREAM_ARM_DROPIN = 0, /* coloc::copy/transform(par.on(cuda_block_executor{synchronous}))
                                    over coloc::vector: the reference's blocking semantics */
    COLOC_STREAM_ARM_CABI = 1    /* coloc_cuda_<op>_<dtype> + coloc_cuda_stream_sync per call */
};

/* Listing 4 for `iterations` iterations on n elements per array (a=1,
 * b=2, c=0) on one GPU, every kernel call timed with the host's steady
 * clock around a call that returns only when the kernel has finished. */
int coloc_stream_blocking_run(int arm, int dtype, int dev, uint64_t n,
    int iterations, coloc_stream_timing* out);

/* Kernels launched by libcoloc_cuda so far (gpu_launches accounting). */
uint64_t coloc_stream_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* COLOC_STREAM_H */
