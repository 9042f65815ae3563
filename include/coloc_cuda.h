/*
 * coloc_cuda.h -- C ABI of the B200-native STREAM hot path.
 *
 * The reference library `coloc` (/root/reference/proj) has no FFI: its
 * boundary is a header-only C++ template API (algorithms.hpp, the
 * executor/allocator concepts).  Its "device" is an in-process mock whose
 * operations are host lambdas run by a FIFO worker thread
 * (device.hpp:43-96, src/device.cpp:44-68).  This header is the seam that
 * replaces that mock with real sm_100a work: every entry point below stands
 * in for one reference operation (cited per function), and the C++ drop-in
 * layer (paper_2206_06302_b200/include/coloc_b200/) calls nothing else.
 *
 * Conventions
 *   - Every function returns int status: COLOC_OK (0) or a COLOC_ERR_* code.
 *     A thread-local message is available from coloc_cuda_last_error().
 *     The C++ layer rethrows codes as the reference's exception types
 *     (error.hpp:11-57): ALLOCATION -> allocation_error, INVALID_TARGET ->
 *     invalid_target_error, SUBMISSION -> submission_error, INVALID_ARGUMENT
 *     -> std::invalid_argument, everything else -> coloc::error.
 *   - Every call names its device ordinal `dev` explicitly; streams and
 *     events are opaque handles (cudaStream_t / cudaEvent_t).  A NULL
 *     stream means the device's legacy default stream.
 *   - Element counts are size_t (N = 2^31 floats is a BASELINE config).
 *   - Kernels are asynchronous with respect to the host and ordered on the
 *     given stream, like enqueue() on the reference's fifo_queue
 *     (device.hpp:63-71).  n == 0 is a no-op (algorithms.hpp:369-371).
 *   - No entry point has a CPU fallback: without a usable GPU they fail with
 *     COLOC_ERR_INVALID_TARGET / COLOC_ERR_CUDA.
 */
#ifndef COLOC_CUDA_H
#define COLOC_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define COLOC_CUDA_ABI_VERSION 3

enum coloc_status
{
    COLOC_OK = 0,
    COLOC_ERR_INVALID_ARGUMENT = 1,
    COLOC_ERR_INVALID_TARGET = 2,
    COLOC_ERR_ALLOCATION = 3,
    COLOC_ERR_SUBMISSION = 4,
    COLOC_ERR_CUDA = 5,
    COLOC_ERR_NCCL = 6,
    COLOC_ERR_UNSUPPORTED = 7
};

/* Message of the last failing call on this thread ("" if none). */
const char* coloc_cuda_last_error(void);
int coloc_cuda_abi_version(void);

/* ------------------------------------------------------------------ */
/* Targets: one per GPU (+ stream).  Replaces device::target and the    */
/* mock registry (device.hpp:29-41, 148-180; src/device.cpp:133-177);   */
/* PAPER.md:456-460 defines a CUDA target as device int + CUDA stream.  */
/* ------------------------------------------------------------------ */

typedef struct coloc_cuda_device_info
{
    int ordinal;
    int sm_count;
    int cc_major;
    int cc_minor;
    int max_threads_per_sm;
    int sm_clock_khz;
    int mem_clock_khz;
    int mem_bus_width_bits;
    size_t l2_bytes;
    size_t hbm_bytes;
    char name[128];
} coloc_cuda_device_info;

int coloc_cuda_device_count(int* count);
int coloc_cuda_device_info_get(int dev, coloc_cuda_device_info* out);
/* Non-blocking stream on `dev` (a fresh queue: system::make_target,
 * src/device.cpp:173-177 / mock_device::new_queue 109-115). */
int coloc_cuda_stream_create(int dev, void** stream);
int coloc_cuda_stream_destroy(int dev, void* stream);
/* fifo_queue::wait_idle (device.hpp:73-74) / device_executor::drain. */
int coloc_cuda_stream_sync(int dev, void* stream);
/* 1 when all work on the stream has completed, else 0. */
int coloc_cuda_stream_query(int dev, void* stream, int* done);
int coloc_cuda_device_sync(int dev);

/* ------------------------------------------------------------------ */
/* Memory.  Replaces mock_device::arena_allocate/deallocate             */
/* (src/device.cpp:78-98) and block_allocator::allocate (106-113).      */
/* ------------------------------------------------------------------ */

int coloc_cuda_malloc(int dev, size_t bytes, void** ptr);
int coloc_cuda_free(int dev, void* ptr);
int coloc_cuda_mem_info(int dev, size_t* free_bytes, size_t* total_bytes);
/* Page-locked host memory for staged transfers. */
int coloc_cuda_host_alloc(size_t bytes, void** ptr);
int coloc_cuda_host_free(void* ptr);
/* Pin/unpin existing host memory (cudaHostRegister). */
int coloc_cuda_host_register(void* ptr, size_t bytes);
int coloc_cuda_host_unregister(void* ptr);
/* Staged copies (algorithms.hpp:388-437): direction inferred from the
 * pointers (cudaMemcpyDefault), ordered on `stream`. */
int coloc_cuda_memcpy_async(int dev, void* stream, void* dst, const void* src,
    size_t bytes);
/* The same copy fully ordered on `stream` for any kind of host memory:
 * returns at once, and the host buffer must stay valid (and, for
 * host->device, unmodified) until the stream has passed the copy -- the
 * contract cudaMemcpyAsync has for pinned memory, extended to pageable
 * memory (>= 4 MiB) by per-device staging workers whose pinned ring
 * chunks are gated on the stream with stream memory operations.  A
 * stream synchronize after a device->host copy means the data is in dst.
 * Used by coloc::copy with a stream-ordered executor
 * (executor_options::synchronous == false; algorithms.hpp:388-407). */
int coloc_cuda_memcpy_stream_ordered(int dev, void* stream, void* dst,
    const void* src, size_t bytes);
/* Returns the pinned staging rings to the system once their copies have
 * completed (leak-free shutdown; the next staged copy sets them up
 * again). */
int coloc_cuda_staging_release(void);
/* Cross-device copy over NVLink (replaces the host bounce buffer of
 * algorithms.hpp:420-436). */
int coloc_cuda_memcpy_peer_async(int dst_dev, void* dst, int src_dev,
    const void* src, size_t bytes, void* stream);
int coloc_cuda_enable_peer_access(int dev, int peer_dev);

/* ------------------------------------------------------------------ */
/* Events and completion callbacks (device_executor futures,            */
/* device_executor.hpp:94-120).                       */
/* ------------------------------------------------------------------ */

int coloc_cuda_event_create(int dev, void** event);
int coloc_cuda_event_destroy(int dev, void* event);
int coloc_cuda_event_record(int dev, void* event, void* stream);
int coloc_cuda_event_sync(void* event);
int coloc_cuda_event_query(void* event, int* done);
int coloc_cuda_event_elapsed_ms(void* start, void* stop, float* ms);
int coloc_cuda_stream_wait_event(int dev, void* stream, void* event);
/* Timestamps the completion of the work queued on `stream` so far into
 * `event`, recorded on `side` (a second stream of the same device) so
 * that later work on `stream` does not wait behind the timing record:
 * back-to-back kernels are timed by consecutive completion stamps without
 * an event node between them.  Capture-safe; join `side` back before the
 * capture ends. */
int coloc_cuda_stream_fork_timestamp(int dev, void* stream, void* side,
    void* event);
/* `stream` waits for everything queued on `side` so far. */
int coloc_cuda_stream_join(int dev, void* stream, void* side);
/* fn(user, status) runs on a CUDA runtime thread once prior work on the
 * stream completes; status is COLOC_OK, or the mapped error when that work
 * failed (a device fault), so futures settled from it carry the error.
 * fn must not call CUDA. */
typedef void (*coloc_cuda_host_fn)(void* user, int status);
int coloc_cuda_launch_host_func(int dev, void* stream, coloc_cuda_host_fn fn,
    void* user);

/* CUDA graphs: capture whatever is enqueued on `stream` (kernels, copies,
 * event records -- recorded as event-record nodes) between begin and end,
 * then replay it with one launch.  Used to take host launch overhead out
 * of launch-bound loops (small arrays, SURVEY.md section 7 hard part 6). */
int coloc_cuda_graph_capture_begin(int dev, void* stream);
int coloc_cuda_graph_capture_end(int dev, void* stream, void** graph_exec);
/* Ends the captures of n streams (captured together, one graph each) and
 * instantiates the graphs; all captures are ended before any
 * instantiation, which CUDA forbids while a stream of the calling thread
 * is still capturing.  On failure no graph is returned. */
int coloc_cuda_graph_capture_end_many(int n, const int* devs,
    void* const* streams, void** graph_execs);
int coloc_cuda_graph_launch(int dev, void* graph_exec, void* stream);
int coloc_cuda_graph_destroy(int dev, void* graph_exec);

/* ------------------------------------------------------------------ */
/* Elementwise kernels: the hot path.                                   */
/*   copy   algorithms.hpp:359-387  (bytewise fast path, memcpy 384-386) */
/*   scale  algorithms.hpp:452-468  dst[i] = src[i] * s                  */
/*   add    algorithms.hpp:486-507  dst[i] = a[i] + b[i]                 */
/*   triad  algorithms.hpp:486-507  dst[i] = b[i] + c[i] * s             */
/* Triad: fma == 0 rounds the product then the sum (bit-exact with the   */
/* reference built without contraction); fma != 0 computes fma(c,s,b).   */
/* Source and destination ranges must not partially overlap; exact       */
/* aliasing (dst == src) is allowed.                                     */
/* ------------------------------------------------------------------ */

int coloc_cuda_copy_bytes(int dev, void* stream, void* dst, const void* src,
    size_t bytes);
int coloc_cuda_copy_f64(int dev, void* stream, double* dst, const double* src,
    size_t n);
int coloc_cuda_copy_f32(int dev, void* stream, float* dst, const float* src,
    size_t n);
int coloc_cuda_scale_f64(int dev, void* stream, double* dst, const double* src,
    double s, size_t n);
int coloc_cuda_scale_f32(int dev, void* stream, float* dst, const float* src,
    float s, size_t n);
int coloc_cuda_add_f64(int dev, void* stream, double* dst, const double* a,
    const double* b, size_t n);
int coloc_cuda_add_f32(int dev, void* stream, float* dst, const float* a,
    const float* b, size_t n);
int coloc_cuda_triad_f64(int dev, void* stream, double* dst, const double* b,
    const double* c, double s, size_t n, int fma);
int coloc_cuda_triad_f32(int dev, void* stream, float* dst, const float* b,
    const float* c, float s, size_t n, int fma);
/* The same transforms on integer vectors (coloc::vector<int>, <long>,
 * <unsigned> ...): two's complement wrap-around, as the reference's x86-64
 * build computes them; unsigned types use the same entry points (identical
 * bits for + and *).  Triad has no contraction to choose. */
int coloc_cuda_scale_i32(int dev, void* stream, int32_t* dst, const int32_t* src,
    int32_t s, size_t n);
int coloc_cuda_scale_i64(int dev, void* stream, int64_t* dst, const int64_t* src,
    int64_t s, size_t n);
int coloc_cuda_add_i32(int dev, void* stream, int32_t* dst, const int32_t* a,
    const int32_t* b, size_t n);
int coloc_cuda_add_i64(int dev, void* stream, int64_t* dst, const int64_t* a,
    const int64_t* b, size_t n);
int coloc_cuda_triad_i32(int dev, void* stream, int32_t* dst, const int32_t* b,
    const int32_t* c, int32_t s, size_t n);
int coloc_cuda_triad_i64(int dev, void* stream, int64_t* dst, const int64_t* b,
    const int64_t* c, int64_t s, size_t n);
/* Listing 3: dst[i] = to_upper(src[i]) over bytes. */
int coloc_cuda_to_upper_u8(int dev, void* stream, unsigned char* dst,
    const unsigned char* src, size_t n);

/* Tile chains: between begin and end, the elementwise launches above on
 * `stream` are chained -- each launch after the first is a programmatic
 * dependent launch whose CTAs wait only for the previous launch's same
 * tile (per-tile flags, release/acquire), so a kernel's first tiles run
 * while its predecessor's last wave drains.  All launches must cover the
 * same index range with the same alignment (every op reads and writes
 * index i only); one that does not restarts the chain after a full
 * dependency.  Graph-capture safe: end clears the flags in stream order,
 * so captured chains may be replayed. */
int coloc_cuda_chain_begin(int dev, void* stream);
int coloc_cuda_chain_end(int dev, void* stream);
/* In-kernel spans (measurement): between span_begin and span_end every
 * elementwise launch on `stream` (up to `capacity`) records its earliest
 * CTA start and latest CTA end (after its stores are performed) with
 * %globaltimer (32 ns resolution on B200) -- kernel durations without any
 * event node between the kernels.  span_read (after span_end and once the
 * stream has run them) returns the first `count` durations in ms, in
 * launch order.  Capture-safe: replays overwrite the same slots. */
int coloc_cuda_span_begin(int dev, void* stream, int capacity);
int coloc_cuda_span_end(int dev, void* stream, int* count);
int coloc_cuda_span_read(int dev, void* stream, double* ms, int count);
/* Call before enqueueing any other kernel on a stream with an open chain
 * (device_lambda.cuh does for user lambdas): the chain restarts behind
 * it, so the next chained launch waits for that kernel in full.  Copies,
 * memsets and event records need no break.  No-op without a chain. */
int coloc_cuda_chain_break(int dev, void* stream);

/* ------------------------------------------------------------------ */
/* Construction on the owning device ("first touch"):                   */
/* block_allocator::bulk_construct (block_allocator.hpp:127-133) and     */
/* device_allocator::bulk_construct/bulk_generate (163-203).             */
/* ------------------------------------------------------------------ */

/* Fills n elements of elem_size bytes (1, 2, 4, 8, 16 or 32) with the
 * bit pattern at value (host memory). */
int coloc_cuda_fill(int dev, void* stream, void* dst, size_t n,
    const void* value, size_t elem_size);
int coloc_cuda_fill_f64(int dev, void* stream, double* dst, size_t n, double v);
int coloc_cuda_fill_f32(int dev, void* stream, float* dst, size_t n, float v);
/* dst[i] = u(seed, k, first + i): counter-based splitmix64 mapped to
 * [-1, 1) (oracle/coloc_oracle.c oracle_fill_random_*). */
int coloc_cuda_generate_random_f64(int dev, void* stream, double* dst,
    size_t n, uint64_t seed, uint32_t k, uint64_t first);
int coloc_cuda_generate_random_f32(int dev, void* stream, float* dst,
    size_t n, uint64_t seed, uint32_t k, uint64_t first);
/* dst[i] = first + i (as the element type). */
int coloc_cuda_iota_f64(int dev, void* stream, double* dst, size_t n,
    double first);

/* ------------------------------------------------------------------ */
/* Validation and parity checksums.                   */
/* Results are written to DEVICE memory so the reduction can be chained  */
/* with a collective on the same stream.                                 */
/* ------------------------------------------------------------------ */

/* out[j] = sum_i |x_j[i] - expected[j]| for the three STREAM arrays
 * (x_0=a, x_1=b, x_2=c), in f64, deterministic order.  out: 3 doubles
 * of device memory. */
int coloc_cuda_stream_err_sums_f64(int dev, void* stream, const double* a,
    const double* b, const double* c, size_t n, const double expected[3],
    double* out);
int coloc_cuda_stream_err_sums_f32(int dev, void* stream, const float* a,
    const float* b, const float* c, size_t n, const double expected[3],
    double* out);
/* *out += sum_i mix64(bits(x[i]) + (first+i)*GOLDEN) mod 2^64, with
 * elem_size 8 (bits = the 64-bit pattern) or 4 (zero-extended).  out: one
 * uint64 of device memory, accumulated (zero it first). */
int coloc_cuda_checksum(int dev, void* stream, const void* x, size_t n,
    size_t elem_size, uint64_t first, uint64_t* out);

/* ------------------------------------------------------------------ */
/* Launch tuning (process-wide; 0 fields = automatic per-size choice).  */
/* ------------------------------------------------------------------ */

typedef struct coloc_cuda_tuning
{
    int threads;        /* threads per CTA: 128, 256, 512, 1024; 0 = auto   */
    int unroll;         /* 32-byte packs per thread per tile: 1, 2, 4; 0 = auto */
    int ctas_per_sm;    /* persistent CTAs per SM; 0 = fill the SM          */
    int cache_hint;     /* 0 plain, 1 streaming (evict-first/no-allocate), 2 = 1 + L2::256B prefetch,
                           3 streaming loads + L2 evict-last stores, 4 plain loads + evict-last stores,
                           5 streaming loads + stores evict-last for a share of the lines;
                           -1 = auto (by destination size vs L2) */
    int exact_grid;     /* 1: one tile per CTA; 0: persistent grid stride; -1 = auto */
    int variant;        /* 0 auto, 1 LDG/STG 256-bit packs, 2 TMA bulk copies,
                           3 LDG loads + one bulk store per CTA,
                           4 persistent CTAs with the next tile's loads in flight
                             (exact_grid selects the tile order: 1 blocked, 0 interleaved) */
    int chunk_bytes;    /* TMA variant: bytes per input per pipeline stage; 0 = auto */
    int stages;         /* TMA variant: input ring depth 2..8; 0 = auto         */
    int schedule;       /* TMA variant: 1 round-robin chunks, 2 atomic counter; 0 = auto */
    int l2_keep_permille; /* hint 5: share of output lines kept in L2 (1..1000); 0 = auto */
    int pdl;            /* programmatic dependent launch of the LDG/STG kernels: 1 on, 0 off,
                           -1 auto (ABI 3) */
} coloc_cuda_tuning;

int coloc_cuda_set_tuning(const coloc_cuda_tuning* t);
int coloc_cuda_get_tuning(coloc_cuda_tuning* t);
/* Number of kernels this library has launched in this process. */
uint64_t coloc_cuda_launch_count(void);

/* ------------------------------------------------------------------ */
/* Measurement probes (bench.py --probe-hbm; no reference counterpart). */
/* ------------------------------------------------------------------ */

/* Reads `bytes` (32-byte aligned and sized) once with the STREAM kernels'
 * tile shape and evict-first hint; XOR-folds them into *dev_sink (device
 * memory).  The HBM read-only ceiling next to copy/scale/add/triad. */
int coloc_cuda_probe_read(int dev, void* stream, const void* x, size_t bytes,
    uint64_t* dev_sink);
/* An empty one-CTA kernel: the launch floor of a timed kernel. */
int coloc_cuda_probe_empty(int dev, void* stream);

/* ------------------------------------------------------------------ */
/* NCCL (validation checksum reduction only; never in the timed loop).  */
/* libnccl.so.2 is loaded at first use with dlopen.                      */
/* ------------------------------------------------------------------ */

/* One communicator per listed device in this process (ncclCommInitAll). */
int coloc_cuda_nccl_init_all(int ndev, const int* devs, void** comms_out);
/* Grouped in-place sum-allreduce of `count` doubles: bufs[i] lives on
 * devs[i] and is reduced on streams[i]. */
int coloc_cuda_nccl_allreduce_sum_f64(int ndev, void* const* comms,
    double* const* bufs, size_t count, void* const* streams);
int coloc_cuda_nccl_destroy(int ndev, void* const* comms);

/* One process per GPU (the torchrun / MPI form): rank 0 creates an id,
 * ships the COLOC_NCCL_ID_BYTES bytes to every rank by any means
 * (torch.distributed's store, MPI_Bcast, a file), and each rank calls
 * init_rank on its GPU.  The validation sums and the max-over-ranks of
 * the kernel times are then reduced with nccl_allreduce_f64 over NVLink. */
#define COLOC_NCCL_ID_BYTES 128
enum coloc_reduce_op
{
    COLOC_REDUCE_SUM = 0,
    COLOC_REDUCE_MAX = 1,
    COLOC_REDUCE_MIN = 2
};
int coloc_cuda_nccl_unique_id(void* id_out, size_t bytes);
int coloc_cuda_nccl_init_rank(int dev, int nranks, const void* id, int rank,
    void** comm_out);
/* recv[i] = op over ranks of send[i] (device memory on `dev`; in place
 * when send == recv), ordered on `stream`. */
int coloc_cuda_nccl_allreduce_f64(void* comm, int dev, void* stream,
    const double* send, double* recv, size_t count, int op);

#ifdef __cplusplus
}
#endif

#endif /* COLOC_CUDA_H */
