"""Multi-process plumbing for the STREAM bench (one process per GPU).

The north star partitions the arrays: partition_block(N_total, world)
(include/coloc/partition.hpp:55-76) gives rank r its contiguous block, the
rank's GPU constructs and processes only that block, and the timed loop has
no collective ("scaling": "weak").  Around it: a barrier before/after the
timed region, the max over ranks of each kernel's device time, and the
validation reduction.  On GPUs these run over the library's own NCCL
communicator (coloc_cuda_nccl_init_rank through the C ABI, NVLink);
torch.distributed only carries the 128-byte NCCL id from rank 0 to the
others (a gloo group: rendezvous, no device work).  The CPU tests run the
same plumbing over gloo alone.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

KERNELS = ("copy", "scale", "add", "triad")
WORDS = {"copy": 2, "scale": 2, "add": 3, "triad": 3}   # STREAM byte rule


def partition_block(n: int, k: int) -> list[tuple[int, int]]:
    """(offset, length) per block, ceil-first (partition.hpp:55-76)."""
    if k <= 0:
        raise ValueError("partition_block: empty target list")
    q, r = divmod(n, k)
    out, at = [], 0
    for i in range(k):
        ln = q + (1 if i < r else 0)
        out.append((at, ln))
        at += ln
    return out


class LibComm:
    """The library's NCCL communicator for one rank (one GPU): reductions of
    small float vectors in device memory, ordered on the rank's own stream
    (coloc_cuda_nccl_allreduce_f64)."""

    OPS = {"sum": 0, "max": 1, "min": 2}

    def __init__(self, dev: int, world: int, rank: int, uid: bytes):
        import ctypes as C
        from . import native as N
        self.N, self.dev = N, dev
        comm = C.c_void_p()
        N.check(N.cuda().coloc_cuda_nccl_init_rank(dev, world, uid, rank, C.byref(comm)),
                "nccl_init_rank")
        self.handle = comm.value
        self.stream = N.Stream(dev)
        self.buf = N.DeviceBuffer(8 * 4096, dev)

    @staticmethod
    def unique_id() -> bytes:
        import ctypes as C
        from . import native as N
        buf = C.create_string_buffer(128)
        N.check(N.cuda().coloc_cuda_nccl_unique_id(buf, 128), "nccl_unique_id")
        return buf.raw

    def all_reduce(self, values: list[float], op: str) -> list[float]:
        import ctypes as C
        import numpy as np
        N = self.N
        if not values:
            return []
        out = []
        for lo in range(0, len(values), 4096):
            chunk = np.ascontiguousarray(values[lo:lo + 4096], dtype=np.float64)
            lib = N.cuda()
            N.check(lib.coloc_cuda_memcpy_async(self.dev, self.stream.handle, self.buf.ptr,
                                                chunk.ctypes.data, chunk.nbytes), "upload")
            N.check(lib.coloc_cuda_nccl_allreduce_f64(self.handle, self.dev, self.stream.handle,
                                                      self.buf.ptr, self.buf.ptr, chunk.size,
                                                      self.OPS[op]), "ncclAllReduce")
            got = np.empty_like(chunk)
            N.check(lib.coloc_cuda_memcpy_async(self.dev, self.stream.handle, got.ctypes.data,
                                                self.buf.ptr, got.nbytes), "download")
            self.stream.sync()
            out += got.tolist()
        return out

    def close(self) -> None:
        import ctypes as C
        if self.handle:
            arr = (C.c_void_p * 1)(self.handle)
            self.N.cuda().coloc_cuda_nccl_destroy(1, arr)
            self.handle = None
        self.buf.close()
        self.stream.close()


@dataclass
class Dist:
    rank: int = 0
    world: int = 1
    local_rank: int = 0
    backend: str | None = None
    comm: LibComm | None = None     # the library's NCCL communicator (GPU runs)

    @property
    def active(self) -> bool:
        return self.backend is not None


def init_from_env(backend: str) -> Dist:
    """torchrun / torch.distributed.run environment -> process group.

    backend "nccl": a gloo group for the rendezvous, then the library's
    NCCL communicator on this rank's GPU (COLOC_DEVICE_MAP respected);
    backend "gloo": gloo only (CPU tests, several ranks on one GPU)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world <= 1:
        return Dist()
    import torch.distributed as dist
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group(backend="gloo", rank=rank, world_size=world)
    d = Dist(rank, world, local, backend)
    if backend == "nccl":
        ids = [LibComm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(ids, src=0)
        d.comm = LibComm(device_for(d), world, rank, ids[0])
    return d


def finalize(d: Dist) -> None:
    """Tear the communicators down (a barrier first, so no rank leaves
    while another still reduces)."""
    if d.active:
        import torch.distributed as dist
        if dist.is_initialized():
            barrier(d)
            if d.comm is not None:
                d.comm.close()
                d.comm = None
            dist.destroy_process_group()


def device_for(d: Dist) -> int:
    """GPU ordinal of this rank: its local rank, unless COLOC_DEVICE_MAP
    ("0,0,1,...", one entry per local rank) remaps it -- used to run the
    multi-rank path on a one-GPU box (with the gloo backend, since NCCL
    refuses two ranks on one GPU)."""
    m = os.environ.get("COLOC_DEVICE_MAP")
    if m:
        return int(m.split(",")[d.local_rank])
    return d.local_rank if d.active else 0


def barrier(d: Dist) -> None:
    """All ranks reach this point (with the library communicator: an
    allreduce on each rank's stream, synchronized)."""
    if not d.active:
        return
    if d.comm is not None:
        d.comm.all_reduce([0.0], "sum")
        return
    import torch.distributed as dist
    dist.barrier()


def all_reduce(values: list[float], d: Dist, op: str = "max") -> list[float]:
    """Elementwise max/sum/min of a float list over ranks (identity at
    world 1); over the library's NCCL communicator on GPUs."""
    if not d.active:
        return list(values)
    if d.comm is not None:
        return d.comm.all_reduce(list(values), op)
    import torch
    import torch.distributed as dist
    t = torch.tensor(values, dtype=torch.float64)
    dist.all_reduce(t, op={"max": dist.ReduceOp.MAX, "sum": dist.ReduceOp.SUM,
                           "min": dist.ReduceOp.MIN}[op])
    return [float(x) for x in t.tolist()]


def all_reduce_u64_sum(values: list[int], d: Dist) -> list[int]:
    """Sum mod 2^64 of uint64 checksums over ranks (exact: int64 wraps;
    a host-side gloo reduction -- checksums are test-only)."""
    if not d.active:
        return [v % (1 << 64) for v in values]
    import torch
    import torch.distributed as dist
    signed = [v - (1 << 64) if v >= (1 << 63) else v for v in values]
    t = torch.tensor(signed, dtype=torch.int64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [int(x) % (1 << 64) for x in t.tolist()]


def stream_stats(per_iter_ms: list[list[float]], n_total: int, elem: int) -> dict:
    """per_iter_ms[i][k]: device ms of kernel k in timed iteration i, already
    max over ranks.  Aggregate GB/s = all ranks' bytes / that time; best =
    min time (STREAM's best-of), avg = mean time."""
    out = {}
    for k, name in enumerate(KERNELS):
        ts = [row[k] for row in per_iter_ms]
        byts = WORDS[name] * n_total * elem
        tmin, tavg, tmax = min(ts), sum(ts) / len(ts), max(ts)
        out[name] = {
            "bytes": byts,
            "min_ms": tmin, "avg_ms": tavg, "max_ms": tmax,
            "best_gbs": byts / (tmin * 1e-3) / 1e9,
            "avg_gbs": byts / (tavg * 1e-3) / 1e9,
        }
    return out


def stream_expected(iterations: int, dtype: str = "f64", s: float = 3.0) -> tuple:
    """SPEC.md:542 recurrence from (1,2,0), in the element type."""
    import numpy as np
    t = np.float64 if dtype == "f64" else np.float32
    a, b, c, s = t(1), t(2), t(0), t(s)
    for _ in range(iterations):
        c = a
        b = s * c
        c = a + b
        a = b + s * c
    return float(a), float(b), float(c)
