"""Runs the C++ drop-in API tests (tests/cpp/test_api.cpp): host-side logic
on CPU, the full API on the GPU."""
import subprocess

import pytest


def _run(built, flag):
    res = subprocess.run([str(built / "test_api"), flag], capture_output=True, text=True,
                         timeout=900)
    print(res.stdout, res.stderr)
    return res


def test_cpp_api_host_logic(built):
    res = _run(built, "--cpu")
    assert res.returncode == 0, res.stdout + res.stderr
    assert "FAIL" not in res.stdout


@pytest.mark.gpu
def test_cpp_api_on_gpu(built):
    res = _run(built, "--gpu")
    assert res.returncode == 0, res.stdout + res.stderr
    assert "FAIL" not in res.stdout


@pytest.mark.gpu
def test_device_fault_settles_future_with_error(built):
    """A kernel fault before a bulk_async_execute completion callback makes
    the future throw (first error wins at launch granularity, reference
    detail/bulk.hpp:67-91) instead of settling as a success."""
    res = _run(built, "--fault")
    assert res.returncode == 0, res.stdout + res.stderr
    assert "FAIL" not in res.stdout


@pytest.mark.gpu
def test_listing4_with_device_lambdas(built):
    """nvcc-compiled user code: Listing 4's lambdas (with __device__) run as
    sm_100a kernels and equal the named-op path bit for bit."""
    res = subprocess.run([str(built / "test_lambda")], capture_output=True, text=True, timeout=600)
    print(res.stdout, res.stderr)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "all lambda checks passed" in res.stdout
    # the lambda path's seeded STREAM state against the CPU oracle
    import numpy as np
    import oracle_lib as O
    line = next(l for l in res.stdout.splitlines() if l.startswith("LAMBDA_CHECKSUMS"))
    n, iters, *cks = (int(x) for x in line.split()[1:])
    assert cks == O.stream_random_checksums_parallel(np.float64, n, iters)


def test_launch_policy_host_checks(built):
    """Shape and cache-policy choices per array size (kernels/launch.cuh),
    host-only: no GPU needed."""
    res = subprocess.run([str(built / "test_launch_policy")], capture_output=True, text=True,
                         timeout=120)
    print(res.stdout, res.stderr)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "launch policy checks passed" in res.stdout
