"""CPU checks of bench.py's host-side helpers (no GPU): the L2-regime label,
the whole-iteration rate, the clock sampler's GPU list and the config
table's sizes."""
import bench
from paper_2206_06302_b200 import harness as H

L2 = 133 * 1000 * 1000


def test_l2_regime_labels():
    assert "streams from HBM" in bench.l2_regime(8 << 30, L2)
    assert "L2-assisted" in bench.l2_regime(80_000_000, L2)
    assert "partly L2-resident" in bench.l2_regime(200_000_000, L2)


def test_step_rate_is_bytes_over_summed_time():
    # equal rates give that rate; a slow kernel drags the step down by its byte share
    assert abs(bench.step_gbs({k: 7000.0 for k in H.KERNELS}) - 7000.0) < 1e-9
    slow = dict({k: 7000.0 for k in H.KERNELS}, copy=3500.0)
    want = 10 / (2 / 3500 + 2 / 7000 + 3 / 7000 + 3 / 7000)
    assert abs(bench.step_gbs(slow) - want) < 1e-9


def test_sampled_gpus(monkeypatch):
    monkeypatch.delenv("COLOC_DEVICE_MAP", raising=False)
    monkeypatch.delenv("LOCAL_WORLD_SIZE", raising=False)
    assert bench.sampled_gpus(True, [2, 0, 2], H.Dist()) == "0,2"
    assert bench.sampled_gpus(False, 3, H.Dist()) == "3"
    assert bench.sampled_gpus(False, 0, H.Dist(0, 4, 0, "nccl")) == "0,1,2,3"
    monkeypatch.setenv("COLOC_DEVICE_MAP", "0,0")
    monkeypatch.setenv("LOCAL_WORLD_SIZE", "2")
    assert bench.sampled_gpus(False, 0, H.Dist(0, 2, 0, "gloo")) == "0"


def test_configs_match_baseline_sizes():
    assert bench.CONFIGS["c1"]["n_per_gpu"] == 10_000_000
    assert bench.CONFIGS["c2"]["n_per_gpu"] == 1 << 30 and bench.CONFIGS["c2"]["dtype"] == "f64"
    assert bench.CONFIGS["c3"]["n_per_gpu"] == 1 << 31 and bench.CONFIGS["c3"]["dtype"] == "f32"


def test_reference_sample_fits_host_ram(monkeypatch):
    monkeypatch.setattr(bench, "mem_available_bytes", lambda: 16 << 30)
    n = bench.reference_sample_n("f64", 1 << 30)
    assert 3 * 8 * n <= 8 << 30 and n >= 1 << 20


def test_arm_configs_are_identical_dicts():
    """Both arms print arm_config(): the driver's same_config compares the
    workload, not how each arm ran it (that goes under `setup`)."""
    for c in bench.CONFIGS.values():
        a, b = bench.arm_config(c, 1), bench.arm_config(dict(c), 1)
        assert a == b and a["n_total"] == c["n_per_gpu"]
    assert bench.arm_config(bench.CONFIGS["c2"], 8)["n_total"] == 8 << 30


def test_e2e_window_rule():
    # 10-iteration windows: best = least total time
    its = [1.0] * 5 + [0.5] * 10 + [2.0]
    gbs, s = bench.best_window_gbs(its, 10 ** 9, 10)
    assert s == 5.0 and abs(gbs - 10 * 1e9 / 5.0 / 1e9) < 1e-12
    # fewer iterations than the window: all of them
    gbs, s = bench.best_window_gbs([1.0, 3.0], 10 ** 9, 10)
    assert s == 4.0 and abs(gbs - 0.5) < 1e-12


def test_reference_arm_line_on_cpu():
    """--impl reference at C1 runs the unmodified reference (oracle/_ref) on
    this host: same config dict as the GPU arm, e2e by the GPU arm's rule."""
    import json
    import subprocess
    import sys
    import pytest
    if not bench.REF_BIN.exists():
        pytest.skip("oracle/_ref not built")
    res = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "c1",
                          "--steps", "10", "--warmup", "3"], capture_output=True, text=True,
                         timeout=600, cwd=str(bench.REPO))
    assert res.returncode == 0, res.stderr
    line = json.loads(res.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["config"] == bench.arm_config(bench.CONFIGS["c1"], 1)
    assert line["e2e"]["value"] > 0 and "e2e rule" in line["e2e"]["definition"]
    assert line["cpu_baseline"]["kind"] == "reference" and line["validation"]["passed"]


def test_compare_summary_claims():
    """The paper's two claims as compare_summary computes them: parity at
    100 MB (>= 0.95 per kernel vs the native arm) and convergence (suite
    ratio at the largest size >= at the smallest)."""
    def row(mb, dn, dc):
        k = ("copy", "scale", "add", "triad")
        return {"mb_per_array": mb, "validated": True,
                "ratio_dropin_vs_native": {x: dn for x in k},
                "ratio_dropin_vs_cabi": {x: dc for x in k},
                "suite_ratio_dropin_vs_native": dn, "suite_ratio_dropin_vs_cabi": dc}
    rows = [row(10, 0.97, 0.96), row(100, 1.5, 0.99), row(400, 1.4, 0.996)]
    s = bench.compare_summary(rows)
    assert s["at_mb"] == 100 and s["parity_ge_0_95"] and s["converges"] and s["validated"]
    assert s["suite_ratio_dropin_vs_cabi_by_size"] == {10: 0.96, 100: 0.99, 400: 0.996}
    bad = bench.compare_summary([row(10, 0.97, 0.9), row(100, 0.9, 0.9), row(400, 0.8, 0.9)])
    assert not bad["parity_ge_0_95"] and not bad["converges"]


def test_harness_partition_equals_the_oracle_property():
    """harness.partition_block (rank blocks of the multi-GPU bench) is the
    reference's partition_block: equal to the C oracle's restatement for
    random n, k (hypothesis), contiguous, covering, ceil-first."""
    from hypothesis import given, settings, strategies as st
    import oracle_lib as O

    @settings(max_examples=300, deadline=None)
    @given(st.integers(0, 10 ** 12), st.integers(1, 64))
    def check(n, k):
        mine = H.partition_block(n, k)
        ref = [(int(off), int(ln)) for _, off, ln in O.partition_block(n, k)]
        assert mine == ref
        assert sum(ln for _, ln in mine) == n
        assert max(ln for _, ln in mine) - min(ln for _, ln in mine) <= 1

    check()
