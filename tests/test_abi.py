"""CPU-side checks of the drop-in boundary: both C-ABI libraries load and
export every function their headers declare, and without a GPU they fail
loudly instead of computing anything on the host."""
import ctypes as C

import pytest

from paper_2206_06302_b200 import native as N


@pytest.mark.parametrize("lib_name", sorted(N.HEADERS))
def test_library_exports_every_declared_symbol(built, lib_name):
    lib = C.CDLL(str(N.LIB_DIR / lib_name))
    declared = N.declared_functions(N.HEADERS[lib_name])
    assert len(declared) >= (2 if lib_name == "libstream_native.so" else 10)
    missing = [f for f in declared if not hasattr(lib, f)]
    assert not missing, missing


def test_bindings_cover_headers(built):
    assert sorted(N._CUDA_SIGS) == N.declared_functions(N.HEADERS["libcoloc_cuda.so"])
    assert sorted(N._STREAM_SIGS) == N.declared_functions(N.HEADERS["libcoloc_stream.so"])
    assert sorted(N._NATIVE_SIGS) == N.declared_functions(N.HEADERS["libstream_native.so"])


def test_abi_version(built):
    assert N.cuda().coloc_cuda_abi_version() == 3


def _has_gpu():
    try:
        return N.device_count() > 0
    except Exception:
        return False


def test_no_gpu_means_errors_not_fallback(built):
    if _has_gpu():
        pytest.skip("a GPU is present")
    assert N.device_count() == 0
    p = C.c_void_p()
    st = N.cuda().coloc_cuda_malloc(0, 1024, C.byref(p))
    assert st != N.OK and not p.value
    st = N.cuda().coloc_cuda_triad_f64(0, None, 16, 32, 48, 3.0, 1, 0)
    assert st in (N.INVALID_TARGET, N.CUDA)
    assert N.launch_count() == 0
    cfg = N.StreamConfig(dtype=0, init=0, fma=0, synchronous=1, ntargets=1,
                         devices=(C.c_int * 1)(0), count=10, first=0, seed=0,
                         scalar=3.0, triad_scalar=3.0, host_buffers=0)
    h = C.c_void_p()
    st = N.stream().coloc_stream_create(C.byref(cfg), C.byref(h))
    assert st == N.INVALID_TARGET
    assert b"cuda" in N.stream().coloc_stream_last_error()


def test_tuning_validation(built):
    with pytest.raises(ValueError):
        N.set_tuning(threads=100)
    with pytest.raises(ValueError):
        N.set_tuning(unroll=3)
    with pytest.raises(ValueError):
        N.set_tuning(stages=9)
    with pytest.raises(ValueError):
        N.set_tuning(schedule=3)
    N.set_tuning(threads=512, unroll=2, cache_hint=0, stages=6, schedule=2)
    t = N.Tuning()
    N.check(N.cuda().coloc_cuda_get_tuning(C.byref(t)))
    assert (t.threads, t.unroll, t.cache_hint, t.stages, t.schedule) == (512, 2, 0, 6, 2)
    N.check(N.cuda().coloc_cuda_set_tuning(None))
    N.check(N.cuda().coloc_cuda_get_tuning(C.byref(t)))
    assert (t.threads, t.unroll, t.cache_hint) == (0, 0, -1)


def test_zero_length_calls_are_noops(built):
    # algorithms.hpp:369-371: n == 0 returns at once, even without a GPU
    assert N.cuda().coloc_cuda_copy_bytes(0, None, None, None, 0) == N.OK
    assert N.cuda().coloc_cuda_triad_f64(0, None, None, None, None, 3.0, 0, 0) == N.OK


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    """No silent fallback: without the built libraries the bindings raise
    instead of computing anything on the host."""
    monkeypatch.setattr(N, "LIB_DIR", tmp_path)
    monkeypatch.setattr(N, "_libs", {})
    with pytest.raises(ImportError, match="no CPU fallback"):
        N.cuda()
    with pytest.raises(ImportError):
        N.stream()
    with pytest.raises(ImportError):
        N.native_baseline()
