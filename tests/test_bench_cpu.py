"""bench.py's host-side pieces (no GPU): the workload table matches
BASELINE.json's configs, the CPU-sample budget keeps full RRS where a query is
affordable and scales otherwise, and `--impl reference` runs on CPU-only
hosts for a tiny workload."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_workloads_match_baseline():
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert "config4" in bench.WORKLOADS
    notion, n, d, k, r, alpha, dist, B = bench.WORKLOADS["config4"]
    assert (notion, n, d, k, r, alpha) == ("halfspace", 100_000, 50, 20_000, 20, 0.9)
    assert base["metric"].startswith("query-depths/sec")


@pytest.mark.parametrize("wl,expect_full", [("config1", True), ("config2", True), ("config3", True),
                                            ("config4", True), ("config5", False), ("config5p", False)])
def test_cpu_sample_budget(wl, expect_full):
    notion, n, d, k, r, alpha, dist, B = bench.WORKLOADS[wl]
    r_s, m_s = bench.cpu_sample_budget(n, d, k, r)
    m = -(-k // r)
    assert (r_s, m_s) == (r, m) if expect_full else (r_s * m_s < r * m)
    assert 2.0 * n * d * m_s * r_s <= 2.5e11 or expect_full


def test_reference_arm_runs_on_cpu():
    """--impl reference is the oracle port on host cores: it must not need a GPU."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload",
                          "config1", "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["cpu_baseline"]["kind"] == "port"
