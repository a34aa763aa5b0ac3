"""The driver's bench.py contract on a real GPU: one JSON line with the tier's
keys (roofline of the dominant kernel, end-to-end leg with its host copies,
launch count, clocks), timed on the small c1 layer so the test takes seconds."""

import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_bench_line_has_contract_keys():
    out = subprocess.run([sys.executable, "bench.py", "--config", "c1", "--steps", "5", "--warmup", "3",
                          "--no-others", "--no-cpu"], cwd=REPO, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3 and d["config"]["workload"] == "c1"
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    # the end-to-end leg moves the step's inputs over PCIe: it cannot beat the device-resident layer
    assert e["us_per_layer"] >= d["ms_per_step"] * 1e3 * 0.9
    assert d["clocks"]["sm_mhz"] > 0
