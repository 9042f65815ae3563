"""ctypes bindings of the two C ABIs (include/coloc_cuda.h, include/coloc_stream.h).

The libraries are built in-tree by `_build.py` (``__graft_entry__.build()``)
and loaded from ``paper_2206_06302_b200/lib``.  There is no fallback: if a
library is missing, or no GPU is usable, calls raise.
"""
from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_DIR = PKG / "lib"
REPO = PKG.parent
HEADERS = {
    "libcoloc_cuda.so": REPO / "include" / "coloc_cuda.h",
    "libcoloc_stream.so": REPO / "include" / "coloc_stream.h",
    "libstream_native.so": REPO / "include" / "stream_native.h",
}

OK, INVALID_ARGUMENT, INVALID_TARGET, ALLOCATION, SUBMISSION, CUDA, NCCL, UNSUPPORTED = range(8)


class ColocError(RuntimeError):
    """coloc::error"""


class InvalidTargetError(ColocError):
    """coloc::invalid_target_error"""


class AllocationError(ColocError):
    """coloc::allocation_error"""


class SubmissionError(ColocError):
    """coloc::submission_error"""


_STATUS_EXC = {INVALID_ARGUMENT: ValueError, INVALID_TARGET: InvalidTargetError,
               ALLOCATION: AllocationError, SUBMISSION: SubmissionError}


class DeviceInfo(C.Structure):
    _fields_ = [("ordinal", C.c_int), ("sm_count", C.c_int), ("cc_major", C.c_int),
                ("cc_minor", C.c_int), ("max_threads_per_sm", C.c_int),
                ("sm_clock_khz", C.c_int), ("mem_clock_khz", C.c_int),
                ("mem_bus_width_bits", C.c_int), ("l2_bytes", C.c_size_t),
                ("hbm_bytes", C.c_size_t), ("name", C.c_char * 128)]


class Tuning(C.Structure):
    _fields_ = [("threads", C.c_int), ("unroll", C.c_int), ("ctas_per_sm", C.c_int),
                ("cache_hint", C.c_int), ("exact_grid", C.c_int), ("variant", C.c_int),
                ("chunk_bytes", C.c_int), ("stages", C.c_int), ("schedule", C.c_int),
                ("l2_keep_permille", C.c_int), ("pdl", C.c_int)]


class StreamConfig(C.Structure):
    _fields_ = [("dtype", C.c_int), ("init", C.c_int), ("fma", C.c_int),
                ("synchronous", C.c_int), ("ntargets", C.c_int),
                ("devices", C.POINTER(C.c_int)), ("count", C.c_uint64),
                ("first", C.c_uint64), ("seed", C.c_uint64), ("scalar", C.c_double),
                ("triad_scalar", C.c_double), ("host_buffers", C.c_int),
                ("reduction", C.c_int), ("chain", C.c_int)]


class Timing(C.Structure):
    _fields_ = [("min_s", C.c_double * 4), ("avg_s", C.c_double * 4), ("max_s", C.c_double * 4),
                ("max_rel_err", C.c_double), ("validated", C.c_int)]


VP, I, SZ, U64, U32, D, F = C.c_void_p, C.c_int, C.c_size_t, C.c_uint64, C.c_uint32, C.c_double, C.c_float
PI = C.POINTER(C.c_int)

_CUDA_SIGS = {
    "coloc_cuda_last_error": (C.c_char_p, []),
    "coloc_cuda_abi_version": (I, []),
    "coloc_cuda_device_count": (I, [PI]),
    "coloc_cuda_device_info_get": (I, [I, C.POINTER(DeviceInfo)]),
    "coloc_cuda_stream_create": (I, [I, C.POINTER(VP)]),
    "coloc_cuda_stream_destroy": (I, [I, VP]),
    "coloc_cuda_stream_sync": (I, [I, VP]),
    "coloc_cuda_stream_query": (I, [I, VP, PI]),
    "coloc_cuda_device_sync": (I, [I]),
    "coloc_cuda_malloc": (I, [I, SZ, C.POINTER(VP)]),
    "coloc_cuda_free": (I, [I, VP]),
    "coloc_cuda_mem_info": (I, [I, C.POINTER(SZ), C.POINTER(SZ)]),
    "coloc_cuda_host_alloc": (I, [SZ, C.POINTER(VP)]),
    "coloc_cuda_host_free": (I, [VP]),
    "coloc_cuda_host_register": (I, [VP, SZ]),
    "coloc_cuda_host_unregister": (I, [VP]),
    "coloc_cuda_memcpy_async": (I, [I, VP, VP, VP, SZ]),
    "coloc_cuda_memcpy_stream_ordered": (I, [I, VP, VP, VP, SZ]),
    "coloc_cuda_staging_release": (I, []),
    "coloc_cuda_memcpy_peer_async": (I, [I, VP, I, VP, SZ, VP]),
    "coloc_cuda_enable_peer_access": (I, [I, I]),
    "coloc_cuda_event_create": (I, [I, C.POINTER(VP)]),
    "coloc_cuda_event_destroy": (I, [I, VP]),
    "coloc_cuda_event_record": (I, [I, VP, VP]),
    "coloc_cuda_event_sync": (I, [VP]),
    "coloc_cuda_event_query": (I, [VP, PI]),
    "coloc_cuda_event_elapsed_ms": (I, [VP, VP, C.POINTER(F)]),
    "coloc_cuda_stream_wait_event": (I, [I, VP, VP]),
    "coloc_cuda_stream_fork_timestamp": (I, [I, VP, VP, VP]),
    "coloc_cuda_stream_join": (I, [I, VP, VP]),
    "coloc_cuda_launch_host_func": (I, [I, VP, VP, VP]),
    "coloc_cuda_graph_capture_begin": (I, [I, VP]),
    "coloc_cuda_graph_capture_end": (I, [I, VP, C.POINTER(VP)]),
    "coloc_cuda_graph_capture_end_many": (I, [I, PI, C.POINTER(VP), C.POINTER(VP)]),
    "coloc_cuda_graph_launch": (I, [I, VP, VP]),
    "coloc_cuda_graph_destroy": (I, [I, VP]),
    "coloc_cuda_copy_bytes": (I, [I, VP, VP, VP, SZ]),
    "coloc_cuda_copy_f64": (I, [I, VP, VP, VP, SZ]),
    "coloc_cuda_copy_f32": (I, [I, VP, VP, VP, SZ]),
    "coloc_cuda_scale_f64": (I, [I, VP, VP, VP, D, SZ]),
    "coloc_cuda_scale_f32": (I, [I, VP, VP, VP, F, SZ]),
    "coloc_cuda_add_f64": (I, [I, VP, VP, VP, VP, SZ]),
    "coloc_cuda_add_f32": (I, [I, VP, VP, VP, VP, SZ]),
    "coloc_cuda_triad_f64": (I, [I, VP, VP, VP, VP, D, SZ, I]),
    "coloc_cuda_triad_f32": (I, [I, VP, VP, VP, VP, F, SZ, I]),
    "coloc_cuda_scale_i32": (I, [I, VP, VP, VP, C.c_int32, SZ]),
    "coloc_cuda_scale_i64": (I, [I, VP, VP, VP, C.c_int64, SZ]),
    "coloc_cuda_add_i32": (I, [I, VP, VP, VP, VP, SZ]),
    "coloc_cuda_add_i64": (I, [I, VP, VP, VP, VP, SZ]),
    "coloc_cuda_triad_i32": (I, [I, VP, VP, VP, VP, C.c_int32, SZ]),
    "coloc_cuda_triad_i64": (I, [I, VP, VP, VP, VP, C.c_int64, SZ]),
    "coloc_cuda_to_upper_u8": (I, [I, VP, VP, VP, SZ]),
    "coloc_cuda_chain_begin": (I, [I, VP]),
    "coloc_cuda_chain_end": (I, [I, VP]),
    "coloc_cuda_chain_break": (I, [I, VP]),
    "coloc_cuda_span_begin": (I, [I, VP, I]),
    "coloc_cuda_span_end": (I, [I, VP, PI]),
    "coloc_cuda_span_read": (I, [I, VP, C.POINTER(D), I]),
    "coloc_cuda_fill": (I, [I, VP, VP, SZ, VP, SZ]),
    "coloc_cuda_fill_f64": (I, [I, VP, VP, SZ, D]),
    "coloc_cuda_fill_f32": (I, [I, VP, VP, SZ, F]),
    "coloc_cuda_generate_random_f64": (I, [I, VP, VP, SZ, U64, U32, U64]),
    "coloc_cuda_generate_random_f32": (I, [I, VP, VP, SZ, U64, U32, U64]),
    "coloc_cuda_iota_f64": (I, [I, VP, VP, SZ, D]),
    "coloc_cuda_stream_err_sums_f64": (I, [I, VP, VP, VP, VP, SZ, C.POINTER(D), VP]),
    "coloc_cuda_stream_err_sums_f32": (I, [I, VP, VP, VP, VP, SZ, C.POINTER(D), VP]),
    "coloc_cuda_checksum": (I, [I, VP, VP, SZ, SZ, U64, VP]),
    "coloc_cuda_set_tuning": (I, [C.POINTER(Tuning)]),
    "coloc_cuda_get_tuning": (I, [C.POINTER(Tuning)]),
    "coloc_cuda_launch_count": (U64, []),
    "coloc_cuda_probe_read": (I, [I, VP, VP, SZ, VP]),
    "coloc_cuda_probe_empty": (I, [I, VP]),
    "coloc_cuda_nccl_init_all": (I, [I, PI, C.POINTER(VP)]),
    "coloc_cuda_nccl_allreduce_sum_f64": (I, [I, C.POINTER(VP), C.POINTER(VP), SZ, C.POINTER(VP)]),
    "coloc_cuda_nccl_destroy": (I, [I, C.POINTER(VP)]),
    "coloc_cuda_nccl_unique_id": (I, [VP, SZ]),
    "coloc_cuda_nccl_init_rank": (I, [I, I, VP, I, C.POINTER(VP)]),
    "coloc_cuda_nccl_allreduce_f64": (I, [VP, I, VP, VP, VP, SZ, I]),
}

_STREAM_SIGS = {
    "coloc_stream_create": (I, [C.POINTER(StreamConfig), C.POINTER(VP)]),
    "coloc_stream_destroy": (I, [VP]),
    "coloc_stream_last_error": (C.c_char_p, []),
    "coloc_stream_iterate": (I, [VP, I]),
    "coloc_stream_iterate_many": (I, [VP, I, I, I]),
    "coloc_stream_sync": (I, [VP]),
    "coloc_stream_recorded": (I, [VP, PI]),
    "coloc_stream_kernel_ms": (I, [VP, I, C.POINTER(D)]),
    "coloc_stream_iteration_ms": (I, [VP, I, C.POINTER(D)]),
    "coloc_stream_clear_records": (None, [VP]),
    "coloc_stream_iterations": (I, [VP, PI]),
    "coloc_stream_e2e_step": (I, [VP, I, C.POINTER(D)]),
    "coloc_stream_err_sums": (I, [VP, C.POINTER(D), C.POINTER(D), VP]),
    "coloc_stream_checksums": (I, [VP, C.POINTER(U64)]),
    "coloc_stream_read": (I, [VP, I, U64, U64, VP]),
    "coloc_stream_launch_count": (U64, []),
    "coloc_stream_set_comm": (I, [VP, VP]),
    "coloc_stream_blocking_run": (I, [I, I, I, U64, I, C.POINTER(Timing)]),
    "coloc_stream_reduction": (C.c_char_p, [VP]),
}

_NATIVE_SIGS = {
    "stream_native_run": (I, [I, I, U64, I, C.POINTER(Timing)]),
    "stream_native_last_error": (C.c_char_p, []),
}

_libs: dict[str, C.CDLL] = {}


def _load(name: str, sigs: dict) -> C.CDLL:
    if name in _libs:
        return _libs[name]
    path = LIB_DIR / name
    if not path.exists():
        raise ImportError(f"{path} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    if name == "libcoloc_stream.so":
        _load("libcoloc_cuda.so", _CUDA_SIGS)
    lib = C.CDLL(str(path), mode=C.RTLD_GLOBAL)
    for fn, (res, args) in sigs.items():
        f = getattr(lib, fn)
        f.restype = res
        f.argtypes = args
    _libs[name] = lib
    return lib


def cuda() -> C.CDLL:
    return _load("libcoloc_cuda.so", _CUDA_SIGS)


def stream() -> C.CDLL:
    return _load("libcoloc_stream.so", _STREAM_SIGS)


def native_baseline() -> C.CDLL:
    """The hand-written native CUDA STREAM (measurement baseline only)."""
    return _load("libstream_native.so", _NATIVE_SIGS)


def declared_functions(header: Path) -> list[str]:
    """Function names a C header declares (for the export check)."""
    text = re.sub(r"/\*.*?\*/", "", header.read_text(), flags=re.S)
    text = re.sub(r"typedef[^;]*;", "", text)
    return sorted(set(re.findall(r"\b((?:coloc|stream_native)_[a-z0-9_]+)\s*\(", text)))


def check(status: int, what: str = "", lib: str = "cuda") -> None:
    if status == OK:
        return
    msg_fn = stream().coloc_stream_last_error if lib == "stream" else cuda().coloc_cuda_last_error
    msg = (msg_fn() or b"").decode(errors="replace")
    raise _STATUS_EXC.get(status, ColocError)(f"{what}: status {status}: {msg}")


def device_count() -> int:
    n = C.c_int(0)
    check(cuda().coloc_cuda_device_count(C.byref(n)), "device_count")
    return n.value


def device_info(dev: int = 0) -> DeviceInfo:
    info = DeviceInfo()
    check(cuda().coloc_cuda_device_info_get(dev, C.byref(info)), "device_info")
    return info


def set_tuning(threads=0, unroll=0, ctas_per_sm=0, cache_hint=-1, exact_grid=-1,
               variant=0, chunk_bytes=0, stages=0, schedule=0, l2_keep_permille=0, pdl=-1) -> None:
    t = Tuning(threads, unroll, ctas_per_sm, cache_hint, exact_grid, variant, chunk_bytes,
               stages, schedule, l2_keep_permille, pdl)
    check(cuda().coloc_cuda_set_tuning(C.byref(t)), "set_tuning")


def launch_count() -> int:
    return int(cuda().coloc_cuda_launch_count())


class DeviceBuffer:
    """cudaMalloc'd bytes on one device (freed on close/GC)."""

    def __init__(self, nbytes: int, dev: int = 0):
        self.dev, self.nbytes = dev, nbytes
        p = C.c_void_p()
        check(cuda().coloc_cuda_malloc(dev, nbytes, C.byref(p)), f"malloc({nbytes})")
        self.ptr = p.value or 0

    def close(self) -> None:
        if self.ptr:
            cuda().coloc_cuda_free(self.dev, self.ptr)
            self.ptr = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def upload(self, host, offset: int = 0) -> None:
        import numpy as np
        a = np.ascontiguousarray(host)
        check(cuda().coloc_cuda_memcpy_async(self.dev, None, self.ptr + offset,
                                             a.ctypes.data, a.nbytes), "upload")
        check(cuda().coloc_cuda_stream_sync(self.dev, None), "sync")

    def download(self, dtype, count: int, offset: int = 0):
        import numpy as np
        out = np.empty(count, dtype=dtype)
        if out.nbytes:
            check(cuda().coloc_cuda_memcpy_async(self.dev, None, out.ctypes.data,
                                                 self.ptr + offset, out.nbytes), "download")
            check(cuda().coloc_cuda_stream_sync(self.dev, None), "sync")
        return out


class Stream:
    def __init__(self, dev: int = 0):
        self.dev = dev
        s = C.c_void_p()
        check(cuda().coloc_cuda_stream_create(dev, C.byref(s)), "stream_create")
        self.handle = s.value

    def sync(self) -> None:
        check(cuda().coloc_cuda_stream_sync(self.dev, self.handle), "stream_sync")

    def close(self) -> None:
        if self.handle:
            cuda().coloc_cuda_stream_destroy(self.dev, self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
