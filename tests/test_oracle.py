"""Pins the CPU oracle (oracle/coloc_oracle.c) before anything trusts it:
against the SPEC examples and against outputs of the unmodified reference
library committed under tests/golden (tests/golden/make_golden.py)."""
import json
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O

GOLDEN = Path(__file__).resolve().parent / "golden"
REF = json.loads((GOLDEN / "reference.json").read_text())


# --- SPEC examples (the only results the reference pins itself) -------------

def test_spec_partition_examples():
    # SPEC.md:173-175
    assert O.partition_block(10, 2) == [(0, 0, 5), (1, 5, 5)]
    assert O.partition_block(10, 3) == [(0, 0, 4), (1, 4, 3), (2, 7, 3)]
    assert O.partition_block(2, 3) == [(0, 0, 1), (1, 1, 1), (2, 2, 0)]
    with pytest.raises(ValueError):
        O.partition_block(10, 0)


def test_spec_kernel_examples():
    # SPEC.md:461, 471-472
    np.testing.assert_array_equal(O.scale(np.array([1.0, 2.0, 3.0]), 3.0), [3.0, 6.0, 9.0])
    np.testing.assert_array_equal(O.add(np.array([1.0, 1.0]), np.array([2.0, 2.0])), [3.0, 3.0])
    np.testing.assert_array_equal(O.triad(np.array([2.0]), np.array([1.0]), 3.0), [5.0])
    s = np.frombuffer(b"helloworld", dtype=np.uint8)
    assert O.to_upper(s).tobytes() == b"HELLOWORLD"


def test_spec_stream_one_iteration():
    # (1,2,0) -> a=15, b=3, c=4 for every element
    for dt in (np.float64, np.float32):
        a, b, c = (np.full(7, v, dtype=dt) for v in (1.0, 2.0, 0.0))
        O.stream_iteration(a, b, c)
        assert (a == 15).all() and (b == 3).all() and (c == 4).all()
    assert O.stream_expected(1) == (15.0, 3.0, 4.0)


def test_stream_recurrence_closed_form():
    # a = 15^k, b = 3*15^(k-1), c = 4*15^(k-1): exact in f64 up to k = 13
    for k in range(1, 14):
        assert O.stream_expected(k) == (15.0 ** k, 3.0 * 15.0 ** (k - 1), 4.0 * 15.0 ** (k - 1))


def test_partition_exhaustive_properties():
    # SPEC.md:218, 606 (n <= 10^4 sampled densely, all k <= 16)
    for k in range(1, 17):
        for n in list(range(0, 300)) + [997, 1000, 4096, 9999, 10000]:
            blocks = O.partition_block(n, k)
            assert blocks[0][1] == 0
            for (i, off, ln), nxt in zip(blocks, blocks[1:] + [None]):
                if nxt is not None:
                    assert nxt[1] == off + ln
            assert sum(b[2] for b in blocks) == n
            lens = [b[2] for b in blocks]
            assert max(lens) - min(lens) <= 1
            assert lens == sorted(lens, reverse=True)


def test_chunk_range_rules():
    assert O.chunk_range(0, 10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert O.chunk_range(5, 7, 10) == [(5, 6), (6, 7)]
    assert O.chunk_range(3, 3, 4) == []
    assert O.chunk_range(0, 5, 0) == [(0, 5)]


# --- golden vectors from the reference itself --------------------------------

@pytest.mark.parametrize("key", sorted(REF["partition"]))
def test_partition_matches_reference(key):
    n, k = (int(x) for x in key.split(","))
    want = REF["partition"][key]
    if isinstance(want, dict):
        with pytest.raises(ValueError):
            O.partition_block(n, k)
    else:
        assert [list(b) for b in O.partition_block(n, k)] == want


@pytest.mark.parametrize("key", sorted(REF["shape"]))
def test_algorithm_shape_matches_reference(key):
    """algorithm_shape (algorithms.hpp:210-234) = per destination block,
    chunk_range into 4 x workers pieces (workers = |cpuset|)."""
    n, doms, off, ln = key.split("|")
    n, off, ln = int(n), int(off), int(ln)
    sizes = []
    for d in doms.split(";"):
        cnt = 0
        for part in d.split(","):
            lo, _, hi = part.partition("-")
            cnt += int(hi or lo) - int(lo) + 1
        sizes.append(cnt)
    got = []
    for b, (_, boff, blen) in enumerate(O.partition_block(n, len(sizes))):
        lo, hi = max(boff, off), min(boff + blen, off + ln)
        if lo < hi:
            got += [[x - off, y - off, b] for x, y in O.chunk_range(lo, hi, 4 * sizes[b])]
    assert got == REF["shape"][key]


def test_helloworld_matches_reference():
    assert REF["helloworld"] == "HELLOWORLD"
    assert O.to_upper(np.frombuffer(b"helloworld", np.uint8)).tobytes().decode() == REF["helloworld"]


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_kernels_bit_exact_vs_reference(dtype):
    g = np.load(GOLDEN / f"kernels_{dtype}.npz")
    dt = np.float64 if dtype == "f64" else np.float32
    n = g["a"].size
    a, b, c = (O.random(dt, n, k) for k in range(3))
    # the generator restatement reproduces the reference's inputs bit for bit
    for name, x in zip("abc", (a, b, c)):
        assert x.tobytes() == g[name].tobytes(), name
    assert O.copy(a).tobytes() == g["copy"].tobytes()
    assert O.scale(c, 3.0).tobytes() == g["scale"].tobytes()
    assert O.add(a, b).tobytes() == g["add"].tobytes()
    assert O.triad(b, c, 3.0).tobytes() == g["triad"].tobytes()


@pytest.mark.parametrize("key", sorted(REF["stream_expected"]))
def test_stream_validation_expectations_match_reference(key):
    dtype, nt = key.split(",")
    dt = np.float64 if dtype == "f64" else np.float32
    want = REF["stream_expected"][key]
    assert list(O.stream_expected(int(nt), dt)) == want["expected"]
    assert want["passed"] is True


@pytest.mark.parametrize("key", sorted(REF["stream_random"]))
def test_chained_stream_checksums_match_reference(key):
    dtype, n, nt = key.split(",")
    dt = np.float64 if dtype == "f64" else np.float32
    want = [int(x, 16) for x in REF["stream_random"][key]]
    assert O.stream_random_checksums(dt, int(n), int(nt)) == want
    # and the array-based iteration agrees with the streaming form
    a, b, c = (O.random(dt, int(n), k) for k in range(3))
    for _ in range(int(nt)):
        O.stream_iteration(a, b, c)
    assert [O.checksum(a), O.checksum(b), O.checksum(c)] == want


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_streaming_kernel_checksums_agree_with_arrays(dtype):
    n, first = 5003, 1234567
    a, b, c = (O.random(dtype, n, k, first=first) for k in range(3))
    want = [O.checksum(a, first), O.checksum(O.scale(c, 3.0), first),
            O.checksum(O.add(a, b), first), O.checksum(O.triad(b, c, 3.0), first),
            O.checksum(O.triad(b, c, 3.0, fma=True), first)]
    assert O.kernel_checksums(dtype, n, first) == want


def test_fma_variant_differs_and_stays_close():
    b = O.random(np.float64, 100000, 1)
    c = O.random(np.float64, 100000, 2)
    t0, t1 = O.triad(b, c, 3.0), O.triad(b, c, 3.0, fma=True)
    assert (t0 != t1).any()
    # |fma - rounded| <= 1 ulp of max(|b|, |3c|) (the FMA build's bound)
    bound = np.spacing(np.maximum(np.abs(b), np.abs(3.0 * c)))
    assert (np.abs(t0 - t1) <= bound).all()


def test_reference_binary_agrees_when_present():
    if not O.REF_BIN.exists():
        pytest.skip("oracle/_ref not built here")
    import subprocess
    out = subprocess.run([str(O.REF_BIN), "stream", "--n", "1001", "--ntimes", "3"],
                         capture_output=True, text=True, check=True).stdout
    js = json.loads(out)
    assert js["validation"]["expected"] == list(O.stream_expected(3))


def test_f32_recurrence_overflow_is_exact_infinity():
    """f32 STREAM at 100 iterations: 15^33 > FLT_MAX, so the
    recurrence reaches +inf after 32 iterations and stays there (inf + 3*inf
    never makes NaN); an array equal to it has zero error (equal infinities
    count as 0), and a finite array against an infinite expectation does
    not validate."""
    finite = O.stream_expected(32, np.float32)
    assert all(np.isfinite(finite))
    e = O.stream_expected(33, np.float32)
    assert np.isinf(e[0]) and e[0] > 0
    e100 = O.stream_expected(100, np.float32)
    assert all(np.isinf(v) and v > 0 for v in e100)
    x = np.full(1000, np.inf, dtype=np.float32)
    assert O.abs_err_sum(x, e100[0]) == 0.0
    assert O.abs_err_sum(np.ones(10, np.float32), e100[0]) == np.inf
    # f64 stays finite and exact at 100 iterations (15^100 < DBL_MAX)
    a, b, c = O.stream_expected(100, np.float64)
    assert np.isfinite(a) and abs(a / 15 ** 100 - 1) < 1e-13
