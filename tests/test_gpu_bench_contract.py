"""The bench.py JSON-line contract (the driver parses it): one line, the required keys and their
types, the roofline / cpu_baseline / e2e / clocks objects, for the default workload and the
reference arm.  Short runs (few steps) -- this checks the shape, not the numbers."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    out = subprocess.check_output([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                                  cwd=ROOT, timeout=900, stderr=subprocess.DEVNULL).decode()
    lines = [l for l in out.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out
    return json.loads(lines[0])


def test_default_line():
    d = _run("--steps", "5", "--warmup", "3", "--cpu-seconds", "1")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "clocks", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] >= 3
    assert d["config"]["workload"].startswith("cfg2") and d["scaling"] == "strong"
    # the other metric sizes, timed the same way (N=16, N=64, N=32 LDL)
    per = d["per_config"]
    assert set(per) == {"cfg3", "cfg4", "cfg5"}
    for k, r in per.items():
        assert r["workload"].startswith(k) and r["n_gpus"] == 1 and r["steps"] == 5
        assert r["value"] > 0 and r["kernel_ms"] > 0 and r["info_nonzero"] == 0
        assert 0 < r["roofline"]["frac"] <= 1.5 and "sm_mhz" in r["clocks"]
        assert r["global_batch"] == r["batch_per_rank"]
    assert d["gpu_launches"] == 5 + sum(r["gpu_launches"] for r in per.values())
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor", "alu") and r["unit"] in ("GB/s", "TFLOP/s")
    assert 0 < r["frac"] <= 1.5 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["matches_device_run"] is True
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    assert d["info_nonzero"] == 0


def test_reference_arm():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "0")
    assert d["impl"] == "reference" and d["value"] > 0
    ours = _run("--steps", "3", "--warmup", "3", "--per-config", "", "--no-e2e", "--no-library",
                "--no-cpu-baseline")
    assert d["config"] == ours["config"]          # the driver compares the two arms' configs
    assert d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
