"""bench.py keeps the driver's JSON contract (one line on rank 0: metric,
value, unit, steps, warmup, ms_per_step, roofline, e2e, gpu_launches,
clocks, ...) for the headline config and the config-5 driver; and the
reference arm prints its line."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=900):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_line_contract():
    d = _run("--steps", "3", "--warmup", "3", "--no-cpu", "--no-others")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "e2e", "gpu_launches", "clocks", "dropin_e2e"):
        assert k in d, k
    assert d["steps"] == 3 and d["warmup"] >= 3 and d["n_gpus"] == 1
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["gpu_launches"] > 0
    assert d["config"]["workload"].startswith("3D 1025^3 fp32")
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] < 1.0 and r["achieved"] > 0 and r["peak"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["roundtrip_rel_err"] < 1e-5
    for pol in ("exact", "fast"):
        assert d["dropin_e2e"][pol]["value"] > 0


def test_bench_config5_line():
    d = _run("--config", "5", "--steps", "3", "--warmup", "3")
    assert d["config"]["blocks"] == 8 and d["scaling"] == "strong"
    assert d["value"] > 0 and d["roundtrip_rel_err"] < 1e-12


def test_bench_reference_arm_line():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "0")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0
