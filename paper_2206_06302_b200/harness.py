"""Multi-process plumbing for the STREAM bench (one process per GPU).

The north star partitions the arrays: partition_block(N_total, world)
(include/coloc/partition.hpp:55-76) gives rank r its contiguous block, the
rank's GPU constructs and processes only that block, and the timed loop has
no collective ("scaling": "weak").  torch.distributed is used for the
plumbing around it: a barrier before/after the timed region, the max over
ranks of each kernel's device time, and the validation reduction (NCCL on
GPUs; gloo in the CPU tests).
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


@dataclass
class Dist:
    rank: int = 0
    world: int = 1
    local_rank: int = 0
    backend: str | None = None

    @property
    def active(self) -> bool:
        return self.backend is not None


def init_from_env(backend: str) -> Dist:
    """torchrun / torch.distributed.run environment -> process group."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world <= 1:
        return Dist()
    import torch.distributed as dist
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    kwargs = {}
    if backend == "nccl":
        import torch
        torch.cuda.set_device(local)
        kwargs["device_id"] = torch.device("cuda", local)
    dist.init_process_group(backend=backend, rank=rank, world_size=world, **kwargs)
    return Dist(rank, world, local, backend)


def finalize(d: Dist) -> None:
    """Tear the process group down (a barrier first, so no rank leaves
    while another still reduces)."""
    if d.active:
        import torch.distributed as dist
        if dist.is_initialized():
            barrier(d)
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


def _tensor(values, d: Dist, dtype):
    import torch
    dev = torch.device("cuda", d.local_rank) if d.backend == "nccl" else torch.device("cpu")
    return torch.tensor(values, dtype=dtype, device=dev)


def barrier(d: Dist) -> None:
    if d.active:
        import torch.distributed as dist
        if d.backend == "nccl":
            dist.barrier(device_ids=[d.local_rank])
        else:
            dist.barrier()


def all_reduce(values: list[float], d: Dist, op: str = "max") -> list[float]:
    """Elementwise max/sum of a float list over ranks (identity at world 1)."""
    if not d.active:
        return list(values)
    import torch
    import torch.distributed as dist
    t = _tensor(values, d, torch.float64)
    dist.all_reduce(t, op={"max": dist.ReduceOp.MAX, "sum": dist.ReduceOp.SUM,
                           "min": dist.ReduceOp.MIN}[op])
    return [float(x) for x in t.cpu().tolist()]


def all_reduce_u64_sum(values: list[int], d: Dist) -> list[int]:
    """Sum mod 2^64 of uint64 checksums over ranks (exact: int64 wraps)."""
    if not d.active:
        return [v % (1 << 64) for v in values]
    import torch
    import torch.distributed as dist
    signed = [v - (1 << 64) if v >= (1 << 63) else v for v in values]
    t = _tensor(signed, d, torch.int64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [int(x) % (1 << 64) for x in t.cpu().tolist()]


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
