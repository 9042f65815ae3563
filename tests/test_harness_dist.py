"""Multi-rank bench plumbing at world size 2 on CPU (gloo): block ownership
per rank, max-over-ranks kernel timing, validation and checksum reductions,
and that per-rank checksums of the oracle's blocks add up to the global one
(the property the GPU ranks rely on)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2206_06302_b200 import harness as H


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    import oracle_lib as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    try:
        d = H.init_from_env("gloo")
        n_total = 1_000_003
        first, count = H.partition_block(n_total, d.world)[d.rank]
        # per-iteration kernel times differ per rank; the max is reported
        times = [[1.0 + rank, 2.0, 3.0 - rank, 4.0]]
        mx = H.all_reduce([x for row in times for x in row], d, "max")
        # validation sums add up
        sums = H.all_reduce([0.5 * (rank + 1)] * 3, d, "sum")
        # checksums of each rank's block (global indices) add up mod 2^64
        cks = O.stream_random_checksums(np.float64, count, 2, first=first)
        tot = H.all_reduce_u64_sum(cks, d)
        H.barrier(d)
        q.put((rank, first, count, mx, sums, tot))
        H.finalize(d)
        import torch.distributed as dist
        assert not dist.is_initialized()
    except Exception as e:  # surface failures to the parent
        q.put((rank, "error", repr(e)))


@pytest.mark.timeout(300)
def test_two_rank_gloo_plumbing():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(60)
    for r in res:
        assert r[1] != "error", r
    import oracle_lib as O
    (_, f0, c0, mx0, s0, t0), (_, f1, c1, mx1, s1, t1) = res
    assert (f0, c0, f1, c1) == (0, 500_002, 500_002, 500_001)
    assert mx0 == mx1 == [2.0, 2.0, 3.0, 4.0]
    assert s0 == s1 == [1.5, 1.5, 1.5]
    assert t0 == t1 == O.stream_random_checksums(np.float64, 1_000_003, 2)


def test_partition_matches_oracle():
    import oracle_lib as O
    for n, k in [(10, 3), (2, 3), (1 << 33, 8), (7, 1)]:
        assert [(o, l) for _, o, l in O.partition_block(n, k)] == H.partition_block(n, k)
    with pytest.raises(ValueError):
        H.partition_block(5, 0)


def test_stream_stats_best_and_avg():
    st = H.stream_stats([[1.0, 1.0, 2.0, 2.0], [2.0, 2.0, 4.0, 1.0]], n_total=1_000_000, elem=8)
    assert st["triad"]["min_ms"] == 1.0 and st["triad"]["avg_ms"] == 1.5
    assert st["triad"]["best_gbs"] == pytest.approx(24e6 / 1e-3 / 1e9)
    assert st["copy"]["bytes"] == 16e6


def test_expected_recurrence():
    import oracle_lib as O
    for k in (0, 1, 10, 13):
        assert H.stream_expected(k) == O.stream_expected(k)
        assert H.stream_expected(k, "f32") == O.stream_expected(k, np.float32)
