"""Parity of the sm_100a kernels (through the C ABI) with the CPU oracle.

Bit-exact for copy, scale, add and triad (no contraction); the FMA triad is
compared bit-exactly with the oracle's explicit fma() and held to 1 ulp of
max(|b|, |s*c|) against the uncontracted result.  Sizes cover the edge
cases: empty, single element, tails not divisible by the 32-byte pack,
misaligned sub-ranges and mutually misaligned operands."""
import ctypes as C

import numpy as np
import pytest

import oracle_lib as O
from paper_2206_06302_b200 import native as N

pytestmark = pytest.mark.gpu

SIZES = [0, 1, 7, 31, 1000, 100_000, 10_000_003]
DTYPES = [np.float64, np.float32]


def fn(name, dt):
    return getattr(N.cuda(), f"coloc_cuda_{name}_{'f64' if dt == np.float64 else 'f32'}")


@pytest.fixture(scope="module")
def dev(built):
    assert N.device_count() >= 1, "no GPU visible: the CUDA path cannot run"
    info = N.device_info(0)
    assert (info.cc_major, info.cc_minor) == (10, 0), info.name
    return 0


def put(x, extra=0, offset=0):
    buf = N.DeviceBuffer(max(x.nbytes + extra + offset, 1))
    if x.nbytes:
        buf.upload(x, offset)
    return buf


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("n", SIZES)
def test_elementwise_bit_exact(dev, dt, n):
    a, b, c = (O.random(dt, n, k) for k in range(3))
    da, db, dc = put(a), put(b), put(c)
    out = N.DeviceBuffer(max(a.nbytes, 1))
    item = a.itemsize
    cases = {
        "copy": (lambda: fn("copy", dt)(0, None, out.ptr, da.ptr, n), O.copy(a)),
        "scale": (lambda: fn("scale", dt)(0, None, out.ptr, dc.ptr, 3.0, n), O.scale(c, 3.0)),
        "add": (lambda: fn("add", dt)(0, None, out.ptr, da.ptr, db.ptr, n), O.add(a, b)),
        "triad": (lambda: fn("triad", dt)(0, None, out.ptr, db.ptr, dc.ptr, 3.0, n, 0),
                  O.triad(b, c, 3.0)),
        "triad_fma": (lambda: fn("triad", dt)(0, None, out.ptr, db.ptr, dc.ptr, 3.0, n, 1),
                      O.triad(b, c, 3.0, fma=True)),
    }
    for name, (run, want) in cases.items():
        N.check(run(), name)
        got = out.download(dt, n)
        assert got.tobytes() == want.tobytes(), f"{name} n={n} differs at " \
            f"{np.flatnonzero(got.view(np.uint8) != want.view(np.uint8))[:4]}"
    assert item in (4, 8)


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("shift", [1, 3, 5])
def test_misaligned_subranges(dev, dt, shift):
    """Sub-range views at element offsets (shared misalignment -> pack path
    with head/tail) and mutually misaligned operands (element path)."""
    n = 100_003
    a, b, c = (O.random(dt, n, k) for k in range(3))
    it = a.itemsize
    # same offset for every operand
    da, db, dc = put(a, offset=shift * it), put(b, offset=shift * it), put(c, offset=shift * it)
    out = N.DeviceBuffer(a.nbytes + 64)
    N.check(fn("triad", dt)(0, None, out.ptr + shift * it, db.ptr + shift * it,
                            dc.ptr + shift * it, 3.0, n, 0))
    assert out.download(dt, n, shift * it).tobytes() == O.triad(b, c, 3.0).tobytes()
    # destination aligned, sources shifted differently
    db2, dc2 = put(b, offset=it), put(c, offset=2 * it)
    N.check(fn("triad", dt)(0, None, out.ptr, db2.ptr + it, dc2.ptr + 2 * it, 3.0, n, 0))
    assert out.download(dt, n).tobytes() == O.triad(b, c, 3.0).tobytes()
    N.check(fn("add", dt)(0, None, out.ptr + it, da.ptr + shift * it, db2.ptr + it, n))
    assert out.download(dt, n, it).tobytes() == O.add(a, b).tobytes()


@pytest.mark.parametrize("n", [0, 1, 31, 32, 33, 4097, 1_000_001])
@pytest.mark.parametrize("src_off,dst_off", [(0, 0), (3, 3), (1, 0), (0, 7), (8, 16)])
def test_copy_bytes_any_alignment(dev, n, src_off, dst_off):
    x = np.frombuffer(np.random.default_rng(n).bytes(n), dtype=np.uint8)
    src = put(x, offset=src_off)
    dst = N.DeviceBuffer(n + dst_off + 8)
    N.check(N.cuda().coloc_cuda_copy_bytes(0, None, dst.ptr + dst_off, src.ptr + src_off, n))
    assert dst.download(np.uint8, n, dst_off).tobytes() == x.tobytes()


def test_overlapping_copy_rejected(dev):
    buf = N.DeviceBuffer(4096)
    with pytest.raises(ValueError):
        N.check(N.cuda().coloc_cuda_copy_bytes(0, None, buf.ptr + 8, buf.ptr, 1024))
    # exact aliasing is an identity copy
    N.check(N.cuda().coloc_cuda_copy_bytes(0, None, buf.ptr, buf.ptr, 1024))


@pytest.mark.parametrize("dt", DTYPES)
def test_in_place_scale(dev, dt):
    c = O.random(dt, 12345, 2)
    d = put(c)
    N.check(fn("scale", dt)(0, None, d.ptr, d.ptr, 3.0, c.size))
    assert d.download(dt, c.size).tobytes() == O.scale(c, 3.0).tobytes()


def test_to_upper_listing3(dev):
    for text in (b"helloworld", b"Hello, World! abc xyz {|}` 09" * 1001):
        x = np.frombuffer(text, dtype=np.uint8)
        d = put(x)
        out = N.DeviceBuffer(x.nbytes)
        N.check(N.cuda().coloc_cuda_to_upper_u8(0, None, out.ptr, d.ptr, x.size))
        assert out.download(np.uint8, x.size).tobytes() == O.to_upper(x).tobytes()
    assert O.to_upper(np.frombuffer(b"helloworld", np.uint8)).tobytes() == b"HELLOWORLD"


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("n,first", [(1, 0), (33, 5), (1_000_003, 987654321)])
def test_generators_match_oracle(dev, dt, n, first):
    out = N.DeviceBuffer(n * np.dtype(dt).itemsize + 64)
    for k in range(3):
        N.check(fn("generate_random", dt)(0, None, out.ptr, n, O.SEED, k, first))
        assert out.download(dt, n).tobytes() == O.random(dt, n, k, first=first).tobytes()
    N.check(fn("fill", dt)(0, None, out.ptr, n, 2.5))
    assert (out.download(dt, n) == 2.5).all()


def test_fill_patterns(dev):
    out = N.DeviceBuffer(4096)
    for size, val in ((1, b"\x7f"), (2, b"\x01\x02"), (4, b"\x01\x02\x03\x04"),
                      (8, bytes(range(8)))):
        n = 1001 // size
        N.check(N.cuda().coloc_cuda_fill(0, None, out.ptr + 3 * (size == 1), n, val, size))
        got = out.download(np.uint8, n * size, 3 * (size == 1)).tobytes()
        assert got == val * n


@pytest.mark.parametrize("dt", DTYPES)
def test_checksum_and_err_sums(dev, dt):
    n = 1_000_003
    x = O.random(dt, n, 0, first=77)
    d = put(x)
    acc = N.DeviceBuffer(8)
    acc.upload(np.zeros(1, np.uint64))
    N.check(N.cuda().coloc_cuda_checksum(0, None, d.ptr, n, x.itemsize, 77, acc.ptr))
    assert int(acc.download(np.uint64, 1)[0]) == O.checksum(x, 77)
    # STREAM error sums: fused over three arrays, matches the oracle to
    # summation-order rounding
    y, z = O.random(dt, n, 1), O.random(dt, n, 2)
    dy, dz = put(y), put(z)
    out = N.DeviceBuffer(24)
    exp = (C.c_double * 3)(0.25, -0.5, 0.0)
    f = N.cuda().coloc_cuda_stream_err_sums_f64 if dt == np.float64 else N.cuda().coloc_cuda_stream_err_sums_f32
    N.check(f(0, None, d.ptr, dy.ptr, dz.ptr, n, exp, out.ptr))
    got = out.download(np.float64, 3)
    want = [O.abs_err_sum(x, 0.25), O.abs_err_sum(y, -0.5), O.abs_err_sum(z, 0.0)]
    np.testing.assert_allclose(got, want, rtol=1e-12)
    # deterministic run to run
    N.check(f(0, None, d.ptr, dy.ptr, dz.ptr, n, exp, out.ptr))
    assert out.download(np.float64, 3).tobytes() == got.tobytes()


@pytest.mark.parametrize("dt,n", [(np.float64, 1 << 30), (np.float32, 1 << 31),
                                  (np.float32, (1 << 32) + 7)])    # > 2^32 elements: 64-bit indexing
def test_full_size_kernel_checksums(dev, dt, n):
    """BASELINE configs 2 and 3 at full size: every kernel's output,
    checksummed on the GPU, equals the oracle's streaming checksum."""
    it = np.dtype(dt).itemsize
    bufs = [N.DeviceBuffer(n * it) for _ in range(4)]
    a, b, c, out = bufs
    gen = fn("generate_random", dt)
    for k, buf in enumerate((a, b, c)):
        N.check(gen(0, None, buf.ptr, n, O.SEED, k, 0))
    acc = N.DeviceBuffer(8)

    def cks():
        acc.upload(np.zeros(1, np.uint64))
        N.check(N.cuda().coloc_cuda_checksum(0, None, out.ptr, n, it, 0, acc.ptr))
        return int(acc.download(np.uint64, 1)[0])

    got = []
    N.check(fn("copy", dt)(0, None, out.ptr, a.ptr, n)); got.append(cks())
    N.check(fn("scale", dt)(0, None, out.ptr, c.ptr, 3.0, n)); got.append(cks())
    N.check(fn("add", dt)(0, None, out.ptr, a.ptr, b.ptr, n)); got.append(cks())
    N.check(fn("triad", dt)(0, None, out.ptr, b.ptr, c.ptr, 3.0, n, 0)); got.append(cks())
    N.check(fn("triad", dt)(0, None, out.ptr, b.ptr, c.ptr, 3.0, n, 1)); got.append(cks())
    for buf in bufs:
        buf.close()
    assert got == O.kernel_checksums_parallel(dt, n)


def test_tuning_shapes_stay_exact(dev):
    n = 3_000_017
    b, c = O.random(np.float64, n, 1), O.random(np.float64, n, 2)
    db, dc, out = put(b), put(c), N.DeviceBuffer(b.nbytes)
    want = O.triad(b, c, 3.0).tobytes()
    try:
        for threads in (128, 256, 512, 1024):
            for unroll in (1, 2, 4):
                for hint in (0, 1, 3, 4, 5):
                    for exact in (0, 1):
                        N.set_tuning(threads=threads, unroll=unroll, cache_hint=hint,
                                     exact_grid=exact)
                        N.check(N.cuda().coloc_cuda_triad_f64(0, None, out.ptr, db.ptr,
                                                              dc.ptr, 3.0, n, 0))
                        assert out.download(np.float64, n).tobytes() == want, \
                            (threads, unroll, hint, exact)
    finally:
        N.cuda().coloc_cuda_set_tuning(None)


@pytest.mark.parametrize("variant,threads", [(1, 32), (1, 64), (2, 64), (3, 32), (4, 32)])
def test_small_ctas_cover_byte_head_and_tail(dev, variant, threads):
    """Byte element types have up to 31 + 31 elements outside the 32-byte
    packs; a CTA of 32 threads must still write all of them (strided
    fix-up), for copy_bytes and Listing 3's to_upper, in every variant."""
    try:
        N.set_tuning(variant=variant, threads=threads)
        for n in (62, 63, 1000, 4133):
            for off in (1, 17, 31):
                x = np.frombuffer(np.random.default_rng(n + off).bytes(n), dtype=np.uint8)
                src = put(x, offset=off)
                dst = N.DeviceBuffer(n + 64)
                N.check(N.cuda().coloc_cuda_copy_bytes(0, None, dst.ptr + off, src.ptr + off, n))
                assert dst.download(np.uint8, n, off).tobytes() == x.tobytes(), (n, off)
                N.check(N.cuda().coloc_cuda_to_upper_u8(0, None, dst.ptr + off, src.ptr + off, n))
                assert dst.download(np.uint8, n, off).tobytes() == O.to_upper(x).tobytes(), (n, off)
    finally:
        N.cuda().coloc_cuda_set_tuning(None)


def test_errors_map_to_reference_types(dev):
    p = C.c_void_p()
    st = N.cuda().coloc_cuda_malloc(0, 1 << 50, C.byref(p))
    assert st == N.ALLOCATION and not p.value
    st = N.cuda().coloc_cuda_malloc(97, 1024, C.byref(p))
    assert st == N.INVALID_TARGET
    assert N.cuda().coloc_cuda_triad_f64(0, None, None, None, None, 3.0, 5, 0) == N.INVALID_ARGUMENT


@pytest.mark.parametrize("chunk,stages,schedule", [(4096, 0, 0), (16384, 0, 0), (32768, 0, 0),
                                                   (4096, 2, 2), (8192, 3, 1), (8192, 8, 2),
                                                   (12288, 6, 1), (4096, 8, 1)])
@pytest.mark.parametrize("dt", DTYPES)
def test_tma_bulk_variant_bit_exact(dev, dt, chunk, stages, schedule):
    """The cp.async.bulk (TMA) variant: same results for every op, size
    and alignment, ring depth and chunk schedule (round robin / atomic
    counter); repeated launches on one stream reuse the atomic scheduler."""
    try:
        N.set_tuning(variant=2, chunk_bytes=chunk, stages=stages, schedule=schedule)
        for n in (1, 7, 1000, 100_003, 3_000_017):
            for shift in (0, 1):
                a, b, c = (O.random(dt, n, k) for k in range(3))
                it = a.itemsize
                da, db, dc = (put(x, offset=shift * it) for x in (a, b, c))
                out = N.DeviceBuffer(a.nbytes + 64)
                o = out.ptr + shift * it
                for _ in range(2):
                    N.check(fn("triad", dt)(0, None, o, db.ptr + shift * it, dc.ptr + shift * it, 3.0, n, 0))
                    assert out.download(dt, n, shift * it).tobytes() == O.triad(b, c, 3.0).tobytes()
                N.check(fn("add", dt)(0, None, o, da.ptr + shift * it, db.ptr + shift * it, n))
                assert out.download(dt, n, shift * it).tobytes() == O.add(a, b).tobytes()
                N.check(fn("scale", dt)(0, None, o, dc.ptr + shift * it, 3.0, n))
                assert out.download(dt, n, shift * it).tobytes() == O.scale(c, 3.0).tobytes()
                N.check(fn("copy", dt)(0, None, o, da.ptr + shift * it, n))
                assert out.download(dt, n, shift * it).tobytes() == a.tobytes()
                N.check(fn("fill", dt)(0, None, o, n, 1.5))
                assert (out.download(dt, n, shift * it) == 1.5).all()
    finally:
        N.cuda().coloc_cuda_set_tuning(None)


@pytest.mark.parametrize("variant,threads,unroll,exact", [
    (3, 1024, 1, -1), (3, 1024, 2, -1), (3, 256, 2, -1), (3, 128, 1, -1),
    (4, 512, 1, 1), (4, 512, 2, 0), (4, 256, 2, 1), (4, 128, 1, 0)])
@pytest.mark.parametrize("dt", DTYPES)
def test_experimental_variants_bit_exact(dev, dt, variant, threads, unroll, exact):
    """Variant 3 (LDG loads, one bulk store per CTA) and variant 4
    (persistent, next tile's loads in flight; blocked or interleaved tile
    order): every op, size and alignment, bit for bit."""
    try:
        N.set_tuning(variant=variant, threads=threads, unroll=unroll, exact_grid=exact)
        for n in (1, 7, 1000, 100_003, 3_000_017):
            for shift in (0, 1):
                a, b, c = (O.random(dt, n, k) for k in range(3))
                it = a.itemsize
                da, db, dc = (put(x, offset=shift * it) for x in (a, b, c))
                out = N.DeviceBuffer(a.nbytes + 64)
                o = out.ptr + shift * it
                N.check(fn("triad", dt)(0, None, o, db.ptr + shift * it, dc.ptr + shift * it, 3.0, n, 0))
                assert out.download(dt, n, shift * it).tobytes() == O.triad(b, c, 3.0).tobytes()
                N.check(fn("add", dt)(0, None, o, da.ptr + shift * it, db.ptr + shift * it, n))
                assert out.download(dt, n, shift * it).tobytes() == O.add(a, b).tobytes()
                N.check(fn("scale", dt)(0, None, o, dc.ptr + shift * it, 3.0, n))
                assert out.download(dt, n, shift * it).tobytes() == O.scale(c, 3.0).tobytes()
                N.check(fn("copy", dt)(0, None, o, da.ptr + shift * it, n))
                assert out.download(dt, n, shift * it).tobytes() == a.tobytes()
                N.check(fn("fill", dt)(0, None, o, n, 1.5))
                assert (out.download(dt, n, shift * it) == 1.5).all()
    finally:
        N.cuda().coloc_cuda_set_tuning(None)


def test_nccl_validation_reduction(dev):
    """The validation collective through the C ABI (dlopen'ed NCCL): a
    communicator per listed GPU, in-place sum over the per-GPU error sums
    on each GPU's stream.  One GPU here; the same call runs G GPUs."""
    ndev = min(N.device_count(), 8)
    devs = (C.c_int * ndev)(*range(ndev))
    comms = (C.c_void_p * ndev)()
    N.check(N.cuda().coloc_cuda_nccl_init_all(ndev, devs, comms), "nccl_init_all")
    bufs, streams = [], []
    for d in range(ndev):
        b = N.DeviceBuffer(24, d)
        b.upload(np.array([1.0 + d, 2.0, 0.5], dtype=np.float64))
        bufs.append(b)
        streams.append(N.Stream(d))
    ptrs = (C.c_void_p * ndev)(*[b.ptr for b in bufs])
    sts = (C.c_void_p * ndev)(*[s.handle for s in streams])
    N.check(N.cuda().coloc_cuda_nccl_allreduce_sum_f64(ndev, comms, ptrs, 3, sts), "allreduce")
    for s in streams:
        s.sync()
    want = [sum(1.0 + d for d in range(ndev)), 2.0 * ndev, 0.5 * ndev]
    for b in bufs:
        assert list(b.download(np.float64, 3)) == want
    N.check(N.cuda().coloc_cuda_nccl_destroy(ndev, comms))


def test_measurement_probes(dev):
    """probe_read reads without writing (its sink only changes on an
    impossible fold value); the empty kernel launches; bad arguments fail."""
    x = put(O.random(np.float64, 1 << 16, 0))
    sink = N.DeviceBuffer(8)
    sink.upload(np.array([12345], dtype=np.uint64))
    launches = N.launch_count()
    N.check(N.cuda().coloc_cuda_probe_read(0, None, x.ptr, 8 << 16, sink.ptr))
    N.check(N.cuda().coloc_cuda_probe_empty(0, None))
    N.check(N.cuda().coloc_cuda_device_sync(0))
    assert N.launch_count() - launches == 2
    assert int(sink.download(np.uint64, 1)[0]) == 12345
    assert N.cuda().coloc_cuda_probe_read(0, None, x.ptr + 8, 64, sink.ptr) == N.INVALID_ARGUMENT
    assert N.cuda().coloc_cuda_probe_read(0, None, x.ptr, 0, sink.ptr) == N.OK


@pytest.mark.parametrize("nbytes", [4096, (64 << 20) + 4096])
def test_pinned_host_buffers_round_trip(dev, nbytes):
    """coloc_cuda_host_alloc (cudaHostAlloc for small buffers, THP-backed
    registered memory from 64 MiB) round-trips data through the GPU."""
    lib = N.cuda()
    h = C.c_void_p()
    N.check(lib.coloc_cuda_host_alloc(nbytes, C.byref(h)))
    try:
        n = nbytes // 8
        src = O.random(np.float64, n, 5)
        C.memmove(h.value, src.ctypes.data, nbytes)
        d = N.DeviceBuffer(nbytes)
        N.check(lib.coloc_cuda_memcpy_async(0, None, d.ptr, h.value, nbytes))
        N.check(lib.coloc_cuda_device_sync(0))
        C.memset(h.value, 0, nbytes)
        N.check(lib.coloc_cuda_memcpy_async(0, None, h.value, d.ptr, nbytes))
        N.check(lib.coloc_cuda_device_sync(0))
        back = np.frombuffer((C.c_char * nbytes).from_address(h.value), dtype=np.float64)
        assert back.tobytes() == src.tobytes()
    finally:
        N.check(lib.coloc_cuda_host_free(h))


@pytest.mark.parametrize("nbytes,offset", [(4 << 20, 0), ((100 << 20) + 7, 3), ((96 << 20), 8)])
def test_pageable_host_copies_through_staging(dev, nbytes, offset):
    """Pageable (numpy) host buffers of >= 4 MiB go through the pinned
    staging ring both ways; results are byte-identical, at odd sizes and
    offsets, and ordered with kernels on the same stream."""
    lib = N.cuda()
    src = np.frombuffer(np.random.default_rng(7).bytes(nbytes + offset), dtype=np.uint8)
    d = N.DeviceBuffer(nbytes + 64)
    s = N.Stream(0)
    N.check(lib.coloc_cuda_memcpy_async(0, s.handle, d.ptr + offset, src.ctypes.data + offset, nbytes))
    back = np.zeros(nbytes + offset, dtype=np.uint8)
    N.check(lib.coloc_cuda_memcpy_async(0, s.handle, back.ctypes.data + offset, d.ptr + offset, nbytes))
    assert back[offset:].tobytes() == src[offset:].tobytes()
    # stream order: a kernel writing the device buffer, then a staged D2H
    if nbytes % 8 == 0 and offset % 8 == 0:
        n = nbytes // 8
        N.check(lib.coloc_cuda_fill_f64(0, s.handle, d.ptr + offset, n, 2.5))
        out = np.zeros(n)
        N.check(lib.coloc_cuda_memcpy_async(0, s.handle, out.ctypes.data, d.ptr + offset, nbytes))
        assert (out == 2.5).all()
        # and a staged H2D followed by a kernel reading it
        h = np.full(n, 1.25)
        N.check(lib.coloc_cuda_memcpy_async(0, s.handle, d.ptr + offset, h.ctypes.data, nbytes))
        N.check(lib.coloc_cuda_scale_f64(0, s.handle, d.ptr + offset, d.ptr + offset, 2.0, n))
        N.check(lib.coloc_cuda_memcpy_async(0, s.handle, out.ctypes.data, d.ptr + offset, nbytes))
        assert (out == 2.5).all()
    s.close()


@pytest.mark.parametrize("nbytes,offset", [((4 << 20) - 1, 0), (4 << 20, 5), (32 << 20, 0),
                                           ((32 << 20) + 1, 0), ((200 << 20) + 13, 7)])
def test_stream_ordered_staging_sizes(dev, nbytes, offset):
    """coloc_cuda_memcpy_stream_ordered with pageable buffers across the
    staging thresholds: below 4 MiB (driver path), exactly one chunk, one
    byte over a chunk, and more chunks than the ring has slots (slot reuse
    gated by the flags); a kernel in between reads what the H2D wrote and
    the D2H returns what the kernel wrote once the stream is synced."""
    lib = N.cuda()
    src = np.frombuffer(np.random.default_rng(nbytes).bytes(nbytes + offset), dtype=np.uint8)
    d1, d2 = N.DeviceBuffer(nbytes + 64), N.DeviceBuffer(nbytes + 64)
    s = N.Stream(0)
    back = np.zeros(nbytes + offset, dtype=np.uint8)
    N.check(lib.coloc_cuda_memcpy_stream_ordered(0, s.handle, d1.ptr + offset, src.ctypes.data + offset, nbytes))
    N.check(lib.coloc_cuda_copy_bytes(0, s.handle, d2.ptr + offset, d1.ptr + offset, nbytes))
    N.check(lib.coloc_cuda_memcpy_stream_ordered(0, s.handle, back.ctypes.data + offset, d2.ptr + offset, nbytes))
    s.sync()
    assert back[offset:].tobytes() == src[offset:].tobytes()
    s.close()
    d1.close()
    d2.close()


@pytest.mark.parametrize("dt", [np.int32, np.int64])
@pytest.mark.parametrize("n,shift", [(1, 0), (7, 1), (1000, 0), (100_003, 1), (3_000_017, 0)])
def test_integer_transforms_wrap_like_the_reference(dev, dt, n, shift):
    """scale / add / triad on integer vectors: two's complement wrap-around
    (the reference's x86-64 arithmetic), values chosen to overflow; misaligned
    sub-ranges included."""
    rng = np.random.default_rng(n)
    info = np.iinfo(dt)
    a, b, c = (rng.integers(info.min, info.max, size=n, dtype=dt, endpoint=True) for _ in range(3))
    s = dt(info.max // 3 + 7)
    sfx = "i32" if dt == np.int32 else "i64"
    it = a.itemsize
    da, db, dc = (put(x, offset=shift * it) for x in (a, b, c))
    out = N.DeviceBuffer(a.nbytes + 64)
    o = out.ptr + shift * it
    lib = N.cuda()
    with np.errstate(over="ignore"):
        want_scale = (c * s).astype(dt)
        want_add = (a + b).astype(dt)
        want_triad = (b + c * s).astype(dt)
    N.check(getattr(lib, f"coloc_cuda_scale_{sfx}")(0, None, o, dc.ptr + shift * it, int(s), n))
    assert out.download(dt, n, shift * it).tobytes() == want_scale.tobytes()
    N.check(getattr(lib, f"coloc_cuda_add_{sfx}")(0, None, o, da.ptr + shift * it, db.ptr + shift * it, n))
    assert out.download(dt, n, shift * it).tobytes() == want_add.tobytes()
    N.check(getattr(lib, f"coloc_cuda_triad_{sfx}")(0, None, o, db.ptr + shift * it, dc.ptr + shift * it, int(s), n))
    assert out.download(dt, n, shift * it).tobytes() == want_triad.tobytes()


def test_staging_release_and_reuse(dev):
    """coloc_cuda_staging_release frees the rings once idle; the next staged
    copies set them up again (tickets restart with the zeroed flags), in
    both directions, more chunks than ring slots."""
    lib = N.cuda()
    n = (160 << 20) // 8 + 5
    src = O.random(np.float64, n, 3)
    d = N.DeviceBuffer(src.nbytes)
    s = N.Stream(0)
    for _ in range(2):
        back = np.zeros(n)
        N.check(lib.coloc_cuda_memcpy_stream_ordered(0, s.handle, d.ptr, src.ctypes.data, src.nbytes))
        N.check(lib.coloc_cuda_memcpy_stream_ordered(0, s.handle, back.ctypes.data, d.ptr, src.nbytes))
        s.sync()
        assert back.tobytes() == src.tobytes()
        N.check(lib.coloc_cuda_staging_release())
    s.close()
    d.close()
