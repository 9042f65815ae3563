"""bench.py end to end on the GPU: the contract line's keys, the multi-rank
path (two torchrun ranks sharing the one GPU through COLOC_DEVICE_MAP and
the gloo backend, so partitioning, max-over-ranks timing and the
validation reduction all run for real), and the reference arm."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu

KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
        "gpu_launches", "clocks"}


def _line(stdout: str) -> dict:
    lines = [l for l in stdout.splitlines() if l.startswith("{")]
    assert lines, stdout
    return json.loads(lines[-1])


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_contract_line(built):
    res = subprocess.run([sys.executable, "bench.py", "--config", "c1", "--steps", "4", "--warmup", "3",
                          "--e2e-steps", "1"], cwd=REPO, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]
    line = _line(res.stdout)
    assert KEYS <= set(line)
    assert line["n_gpus"] == 1 and line["gpu_launches"] == 4 * 4
    assert line["validation"]["passed"] and line["e2e"]["validation_passed"]
    assert line["roofline"]["bound"] == "hbm" and line["roofline"]["achieved"] > 1000
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 3 * 8 * 10_000_000
    assert line["e2e"]["pageable"]["validation_passed"] and line["e2e"]["pageable"]["value"] > 0
    assert line["abstraction_vs_native"]["validated"]
    assert line["ceilings"]["kernel_fixed_cost"]["in_graph_us"] > 0
    assert line["iteration"]["back_to_back_median_gbs"] > 0
    it = line["iteration"]
    assert it["bytes"] == 10 * 8 * 10_000_000 and 0 < it["avg_gbs"] <= it["best_gbs"]
    ce = line["ceilings"]
    assert ce["read_only_gbs"] > 1000 and ce["write_only_gbs"] > 1000
    assert 0 < ce["timed_kernel_floor_us"] < 100


def test_probe_hbm_mode(built):
    res = subprocess.run([sys.executable, "bench.py", "--probe-hbm", "--config", "c1", "--steps", "3"],
                         cwd=REPO, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    rows = [json.loads(l) for l in res.stdout.splitlines() if l.startswith("{")]
    assert [r["probe"] for r in rows] == ["read_1array", "read_3arrays", "write_fill", "copy", "scale",
                                          "add", "triad", "empty_kernel"]
    assert all(r["best_gbs"] > 500 for r in rows if r["bytes"])


def test_bench_two_ranks(built):
    env = dict(os.environ, COLOC_DEVICE_MAP="0,0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--config", "c1", "--steps", "3", "--warmup", "3", "--dist-backend", "gloo",
           "--e2e-steps", "1", "--e2e-blocks", "2"]
    res = subprocess.run(cmd, cwd=REPO, env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]
    line = _line(res.stdout)
    assert line["n_gpus"] == 2 and line["scaling"] == "weak"
    assert line["config"]["n_total"] == 2 * 10_000_000
    assert line["gpu_launches"] == 2 * 3 * 4        # summed over ranks
    assert line["validation"]["passed"] and line["e2e"]["validation_passed"]
    assert line["cpu_baseline"] is None               # rank 0 at N=1 only


def test_bench_single_process_partitioned_vector(built):
    """C4's single-process form: one vector block-partitioned over two
    targets (mapped onto the one GPU here), per-kernel max over targets."""
    env = dict(os.environ, COLOC_DEVICE_MAP="0,0")
    res = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--config", "c1", "--steps", "3",
                          "--warmup", "3", "--e2e-steps", "1", "--e2e-blocks", "2"], cwd=REPO,
                         env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]
    line = _line(res.stdout)
    assert line["n_gpus"] == 2 and "one process" in line["setup"]["parallelism"]
    assert line["config"]["n_total"] == 2 * 10_000_000
    assert line["gpu_launches"] == 3 * 4 * 2        # one launch per block per kernel
    assert line["validation"]["passed"] and line["e2e"]["validation_passed"]
    assert line["cpu_baseline"] is None


def test_reference_arm(built):
    res = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "c1",
                          "--steps", "3", "--warmup", "3"], cwd=REPO, capture_output=True,
                         text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]
    line = _line(res.stdout)
    assert line["impl"] == "reference" and line["validation"]["passed"]
    assert line["e2e"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "reference"


def test_sweep_two_ranks_and_two_targets(built):
    """C5 on several GPUs: both launch forms, blocks mapped onto the one GPU."""
    env = dict(os.environ, COLOC_DEVICE_MAP="0,0")
    common = ["--sweep", "--sweep-max-log2", "2", "--config", "c2"]
    runs = [
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
         "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
         "--dist-backend", "gloo", *common],
        [sys.executable, "bench.py", "--gpus", "2", *common],
    ]
    for cmd in runs:
        res = subprocess.run(cmd, cwd=REPO, env=env, capture_output=True, text=True, timeout=900)
        assert res.returncode == 0, res.stderr[-3000:]
        rows = [json.loads(l) for l in res.stdout.splitlines() if l.startswith("{")]
        assert [r["bytes_per_array_per_gpu"] for r in rows] == [1 << 20, 2 << 20, 4 << 20]
        assert all(r["n_gpus"] == 2 and r["validated"] and r["triad_best_gbs"] > 10 for r in rows)


def test_compare_baseline_mode(built):
    res = subprocess.run([sys.executable, "bench.py", "--compare-baseline", "--compare-sizes", "10,40",
                          "--compare-reps", "1"], cwd=REPO, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    rows = [json.loads(l) for l in res.stdout.splitlines() if l.startswith("{")]
    summary = rows[-1]["summary"]
    assert summary["sizes_mb"] == [10, 40] and summary["validated"]
    for r in rows[:-1]:
        assert set(r["avg_gbs"]) == {"dropin", "cabi", "native"}
        assert all(v > 0 for v in r["ratio_dropin_vs_native"].values())
