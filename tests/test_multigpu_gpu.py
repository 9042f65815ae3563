"""The multi-GPU code paths, exercised on the one GPU a test box has
(VERDICT r01 "next" item 1):

- per-target CUDA graphs: the STREAM loop over several targets (streams)
  captured one graph per target equals eager launches;
- the e2e step captured into per-target graphs equals the eager step;
- the forced NCCL branch of the validation reduction (one target per GPU);
- the library's one-process-per-GPU NCCL path (coloc_cuda_nccl_unique_id /
  init_rank / allreduce_f64) at nranks = 1, alone and through the STREAM
  driver's cross-rank validation (coloc_stream_set_comm) and bench.py's
  validate().
"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O
from paper_2206_06302_b200 import harness as H
from paper_2206_06302_b200 import native as N

pytestmark = pytest.mark.gpu

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


@pytest.fixture(scope="module")
def dev(built):
    assert N.device_count() >= 1, "no GPU visible"
    return 0


def make(n, devices, dtype="f64", init=1, host_buffers=0, reduction=0, sync=0):
    devs = (C.c_int * len(devices))(*devices)
    cfg = N.StreamConfig(dtype=0 if dtype == "f64" else 1, init=init, fma=0, synchronous=sync,
                         ntargets=len(devices), devices=devs, count=n, first=0, seed=O.SEED,
                         scalar=3.0, triad_scalar=3.0, host_buffers=host_buffers,
                         reduction=reduction)
    h = C.c_void_p()
    N.check(N.stream().coloc_stream_create(C.byref(cfg), C.byref(h)), "create", "stream")
    return h


def checksums(h):
    out = (C.c_uint64 * 3)()
    N.check(N.stream().coloc_stream_checksums(h, out), "checksums", "stream")
    return list(out)


def err(h):
    e, s = (C.c_double * 3)(), (C.c_double * 3)()
    N.check(N.stream().coloc_stream_err_sums(h, e, s, None), "err", "stream")
    return list(e), list(s), N.stream().coloc_stream_reduction(h).decode()


@pytest.mark.parametrize("ntargets", [2, 5])
def test_per_target_graphs_equal_eager(dev, ntargets):
    """COLOC_DEVICE_MAP=0,0-style placement: several targets on GPU 0, one
    block each.  One graph per target (kernels + timing events) gives the
    same state as eager launches, and every kernel of every target is
    timed."""
    n = 3_000_017
    eager, graph = make(n, (0,) * ntargets), make(n, (0,) * ntargets)
    lib = N.stream()
    N.check(lib.coloc_stream_iterate_many(eager, 4, 1, 0), "eager", "stream")
    N.check(lib.coloc_stream_iterate_many(graph, 4, 1, 1), "graph", "stream")
    want = O.stream_random_checksums_parallel(np.float64, n, 4)
    assert checksums(eager) == checksums(graph) == want
    cnt = C.c_int()
    N.check(lib.coloc_stream_recorded(graph, C.byref(cnt)))
    assert cnt.value == 4
    for i in range(4):
        ms = (C.c_double * 4)()
        N.check(lib.coloc_stream_kernel_ms(graph, i, ms))
        assert all(0 < x < 100 for x in ms)
    # captured again on the same handle: still the same
    N.check(lib.coloc_stream_iterate_many(graph, 3, 0, 1), "graph2", "stream")
    N.check(lib.coloc_stream_iterate_many(eager, 3, 0, 0), "eager2", "stream")
    assert checksums(eager) == checksums(graph)
    lib.coloc_stream_destroy(eager)
    lib.coloc_stream_destroy(graph)


def test_e2e_graph_equals_eager_step(dev):
    """Pinned host buffers + stream-ordered executor: the e2e step is
    captured into per-target graphs; the synchronous executor runs the same
    step eagerly.  Both end in the exact STREAM state."""
    n = 4_000_037
    lib = N.stream()
    outs = []
    for sync in (0, 1):
        h = make(n, (0,) * 4, init=0, host_buffers=1, sync=sync)
        ms = C.c_double()
        for _ in range(2):
            N.check(lib.coloc_stream_e2e_step(h, 10, C.byref(ms)), "e2e", "stream")
            assert ms.value > 0
        e, s, _ = err(h)
        assert e == list(O.stream_expected(10)) and s == [0.0, 0.0, 0.0]
        outs.append(checksums(h))
        lib.coloc_stream_destroy(h)
    assert outs[0] == outs[1]


def test_forced_nccl_reduction_branch(dev):
    """reduction = NCCL with one target per GPU (here: one GPU) takes the
    ncclCommInitAll + grouped ncclAllReduce branch of err_sums; auto picks
    the host branch for one target; forcing NCCL over two targets on one
    GPU is refused (NCCL allows one rank per device)."""
    n = 1_000_003
    lib = N.stream()
    got = {}
    for mode in (0, 1, 2):
        h = make(n, (0,), init=0, reduction=mode)
        N.check(lib.coloc_stream_iterate_many(h, 10, 0, 1), "iterate", "stream")
        e, s, how = err(h)
        assert e == list(O.stream_expected(10)) and s == [0.0, 0.0, 0.0]
        got[mode] = how
        lib.coloc_stream_destroy(h)
    assert got == {0: "host", 1: "host", 2: "nccl"}
    # random init: the NCCL sum equals the host sum bit for bit (one rank)
    sums = []
    for mode in (1, 2):
        h = make(n, (0,), init=1, reduction=mode)
        N.check(lib.coloc_stream_iterate(h, 0), "iterate", "stream")
        sums.append(err(h)[1])
        lib.coloc_stream_destroy(h)
    assert sums[0] == sums[1] and all(x > 0 for x in sums[0])
    h = make(n, (0, 0), init=0, reduction=2)
    e, s = (C.c_double * 3)(), (C.c_double * 3)()
    assert lib.coloc_stream_err_sums(h, e, s, None) == N.INVALID_ARGUMENT
    lib.coloc_stream_destroy(h)


def test_nccl_rank_path_one_rank(dev):
    """coloc_cuda_nccl_unique_id + init_rank + allreduce_f64 at nranks = 1
    (the torchrun form's communicator): sum/max/min, in place and out of
    place, on the rank's stream."""
    uid = H.LibComm.unique_id()
    assert len(uid) == 128
    comm = H.LibComm(0, 1, 0, uid)
    try:
        vals = [1.5, -2.0, 3.25, 1e300]
        for op in ("sum", "max", "min"):
            assert comm.all_reduce(vals, op) == vals
        big = [float(i) for i in range(5000)]          # more than one device chunk
        assert comm.all_reduce(big, "max") == big
        assert comm.all_reduce([], "sum") == []
        lib = N.cuda()
        src, dst = N.DeviceBuffer(24), N.DeviceBuffer(24)
        src.upload(np.array([1.0, 2.0, 3.0]))
        st = N.Stream(0)
        N.check(lib.coloc_cuda_nccl_allreduce_f64(comm.handle, 0, st.handle, src.ptr, dst.ptr, 3, 0))
        st.sync()
        assert dst.download(np.float64, 3).tolist() == [1.0, 2.0, 3.0]
        assert lib.coloc_cuda_nccl_allreduce_f64(comm.handle, 0, st.handle, src.ptr, dst.ptr, 3, 7) \
            == N.INVALID_ARGUMENT
        st.close()
    finally:
        comm.close()


def test_stream_driver_cross_rank_validation(dev):
    """The driver's cross-rank reduction (coloc_stream_set_comm) and
    bench.py's validate() over the library communicator at nranks = 1."""
    import bench
    uid = H.LibComm.unique_id()
    comm = H.LibComm(0, 1, 0, uid)
    d = H.Dist(rank=0, world=1, local_rank=0, backend="nccl", comm=comm)
    try:
        n = 2_000_003
        run = bench.StreamRun(N, bench.stream_config(N, "f64", n, 0, 0))
        run.iterate_many(10, False, True)
        v = bench.validate(run, d, n, "f64")
        assert v["passed"] and v["reduction"] == "host+ranks"
        assert v["rel_err"] == [0.0, 0.0, 0.0]
        run.close()
        # the max-over-ranks of kernel times and the barrier
        assert H.all_reduce([1.0, 2.0], d, "max") == [1.0, 2.0]
        H.barrier(d)
    finally:
        comm.close()
