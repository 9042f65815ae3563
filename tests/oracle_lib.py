"""ctypes access to the CPU oracle (oracle/liboracle.so) -- the checker.

Test infrastructure only (see oracle/coloc_oracle.c).  Builds the library
with gcc on first use if it is missing (gcc is available here and on the
GPU box; /root/reference is not needed for it).
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[1]
ORACLE_DIR = REPO / "oracle"
LIB = ORACLE_DIR / "liboracle.so"
REF_BIN = ORACLE_DIR / "_ref" / "ref_stream_cpu"
SEED = 0x220606302

_lib = None
U64, SZ, D, F, I = C.c_uint64, C.c_size_t, C.c_double, C.c_float, C.c_int
VP = C.c_void_p


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            subprocess.run(["make", "-s", "-C", str(ORACLE_DIR), "oracle"], check=True)
        L = C.CDLL(str(LIB))
        sigs = {
            "oracle_mix64": (U64, [U64]),
            "oracle_random_bits": (U64, [U64, C.c_uint32, U64]),
            "oracle_fill_random_f64": (None, [VP, SZ, U64, C.c_uint32, U64]),
            "oracle_fill_random_f32": (None, [VP, SZ, U64, C.c_uint32, U64]),
            "oracle_partition_block": (I, [SZ, SZ, VP, VP]),
            "oracle_chunk_range": (SZ, [SZ, SZ, SZ, VP, VP]),
            "oracle_copy_bytes": (None, [VP, VP, SZ]),
            "oracle_scale_f64": (None, [VP, VP, D, SZ]),
            "oracle_add_f64": (None, [VP, VP, VP, SZ]),
            "oracle_triad_f64": (None, [VP, VP, VP, D, SZ]),
            "oracle_triad_fma_f64": (None, [VP, VP, VP, D, SZ]),
            "oracle_scale_f32": (None, [VP, VP, F, SZ]),
            "oracle_add_f32": (None, [VP, VP, VP, SZ]),
            "oracle_triad_f32": (None, [VP, VP, VP, F, SZ]),
            "oracle_triad_fma_f32": (None, [VP, VP, VP, F, SZ]),
            "oracle_to_upper_u8": (None, [VP, VP, SZ]),
            "oracle_stream_iteration_f64": (None, [VP, VP, VP, SZ, D, I]),
            "oracle_stream_iteration_f32": (None, [VP, VP, VP, SZ, F, I]),
            "oracle_stream_expected_f64": (None, [I, D, VP]),
            "oracle_stream_expected_f32": (None, [I, F, VP]),
            "oracle_abs_err_sum_f64": (D, [VP, SZ, D]),
            "oracle_abs_err_sum_f32": (D, [VP, SZ, D]),
            "oracle_checksum_bits64": (U64, [VP, SZ, U64]),
            "oracle_checksum_bits32": (U64, [VP, SZ, U64]),
            "oracle_kernel_checksums_f64": (None, [U64, U64, SZ, D, VP]),
            "oracle_kernel_checksums_f32": (None, [U64, U64, SZ, F, VP]),
            "oracle_stream_random_checksums_f64": (None, [U64, U64, SZ, D, I, I, VP]),
            "oracle_stream_random_checksums_f32": (None, [U64, U64, SZ, F, I, I, VP]),
        }
        for name, (res, args) in sigs.items():
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args
        _lib = L
    return _lib


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


def random(dtype, n: int, k: int, seed: int = SEED, first: int = 0) -> np.ndarray:
    out = np.empty(n, dtype=dtype)
    if dtype == np.float64:
        lib().oracle_fill_random_f64(_p(out), n, seed, k, first)
    else:
        lib().oracle_fill_random_f32(_p(out), n, seed, k, first)
    return out


def partition_block(n: int, k: int):
    off = np.zeros(max(k, 1), dtype=np.uint64)
    ln = np.zeros(max(k, 1), dtype=np.uint64)
    if lib().oracle_partition_block(n, k, _p(off), _p(ln)) != 0:
        raise ValueError("partition_block: empty target list")
    return [(i, int(off[i]), int(ln[i])) for i in range(k)]


def chunk_range(begin: int, end: int, parts: int):
    cap = max(end - begin, 1)
    b = np.zeros(cap, dtype=np.uint64)
    e = np.zeros(cap, dtype=np.uint64)
    m = lib().oracle_chunk_range(begin, end, parts, _p(b), _p(e))
    return [(int(b[i]), int(e[i])) for i in range(m)]


def copy(src: np.ndarray) -> np.ndarray:
    dst = np.empty_like(src)
    lib().oracle_copy_bytes(_p(dst), _p(src), src.nbytes)
    return dst


def scale(src: np.ndarray, s: float) -> np.ndarray:
    dst = np.empty_like(src)
    fn = lib().oracle_scale_f64 if src.dtype == np.float64 else lib().oracle_scale_f32
    fn(_p(dst), _p(src), s, src.size)
    return dst


def add(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    dst = np.empty_like(a)
    fn = lib().oracle_add_f64 if a.dtype == np.float64 else lib().oracle_add_f32
    fn(_p(dst), _p(a), _p(b), a.size)
    return dst


def triad(b: np.ndarray, c: np.ndarray, s: float, fma: bool = False) -> np.ndarray:
    dst = np.empty_like(b)
    if b.dtype == np.float64:
        fn = lib().oracle_triad_fma_f64 if fma else lib().oracle_triad_f64
    else:
        fn = lib().oracle_triad_fma_f32 if fma else lib().oracle_triad_f32
    fn(_p(dst), _p(b), _p(c), s, b.size)
    return dst


def to_upper(src: np.ndarray) -> np.ndarray:
    dst = np.empty_like(src)
    lib().oracle_to_upper_u8(_p(dst), _p(src), src.size)
    return dst


def stream_iteration(a, b, c, s=3.0, fma=False) -> None:
    fn = lib().oracle_stream_iteration_f64 if a.dtype == np.float64 else lib().oracle_stream_iteration_f32
    fn(_p(a), _p(b), _p(c), a.size, s, int(fma))


def stream_expected(iterations: int, dtype=np.float64, s: float = 3.0):
    out = np.zeros(3, dtype=np.float64)
    fn = lib().oracle_stream_expected_f64 if dtype == np.float64 else lib().oracle_stream_expected_f32
    fn(iterations, s, _p(out))
    return tuple(float(x) for x in out)


def abs_err_sum(x: np.ndarray, expected: float) -> float:
    fn = lib().oracle_abs_err_sum_f64 if x.dtype == np.float64 else lib().oracle_abs_err_sum_f32
    return float(fn(_p(x), x.size, expected))


def checksum(x: np.ndarray, first: int = 0) -> int:
    if x.dtype.itemsize == 8:
        return int(lib().oracle_checksum_bits64(_p(x.view(np.uint64)), x.size, first))
    return int(lib().oracle_checksum_bits32(_p(x.view(np.uint32)), x.size, first))


def kernel_checksums(dtype, n: int, first: int = 0, seed: int = SEED, s: float = 3.0):
    """Checksums of copy(a), scale(c), add(a,b), triad(b,c), triad_fma(b,c)
    over random inputs, O(1) memory (full BASELINE sizes)."""
    out = np.zeros(5, dtype=np.uint64)
    fn = lib().oracle_kernel_checksums_f64 if dtype == np.float64 else lib().oracle_kernel_checksums_f32
    fn(seed, first, n, s, _p(out))
    return [int(x) for x in out]


def stream_random_checksums(dtype, n: int, iterations: int, fma: bool = False,
                            first: int = 0, seed: int = SEED, s: float = 3.0):
    out = np.zeros(3, dtype=np.uint64)
    fn = (lib().oracle_stream_random_checksums_f64 if dtype == np.float64
          else lib().oracle_stream_random_checksums_f32)
    fn(seed, first, n, s, iterations, int(fma), _p(out))
    return [int(x) for x in out]


def _parallel_sum(fn, n: int, width: int, parts: int | None = None):
    """Runs fn(first, count) -> list[int] over chunks on threads (ctypes
    drops the GIL) and adds the results mod 2^64 (the checksums are sums)."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    parts = parts or max(1, min(64, os.cpu_count() or 1))
    step = -(-n // parts)
    chunks = [(s, min(step, n - s)) for s in range(0, n, step)] or [(0, 0)]
    with ThreadPoolExecutor(len(chunks)) as ex:
        res = list(ex.map(lambda c: fn(*c), chunks))
    return [sum(r[i] for r in res) % (1 << 64) for i in range(width)]


def kernel_checksums_parallel(dtype, n: int, first: int = 0, seed: int = SEED, s: float = 3.0):
    return _parallel_sum(lambda f, m: kernel_checksums(dtype, m, first + f, seed, s), n, 5)


def stream_random_checksums_parallel(dtype, n: int, iterations: int, fma: bool = False,
                                     first: int = 0, seed: int = SEED, s: float = 3.0):
    return _parallel_sum(lambda f, m: stream_random_checksums(dtype, m, iterations, fma,
                                                              first + f, seed, s), n, 3)
