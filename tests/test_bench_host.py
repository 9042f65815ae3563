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
