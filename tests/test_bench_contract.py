"""bench.py's output contract (-m gpu): one JSON line on stdout with the keys the driver
reads -- metric / value / unit / timing fields, roofline, cpu_baseline, e2e, clocks,
gpu_launches -- for our arm (configs[3], the short complex128 workload) and for the
reference arm (the oracle; it must not load the product library)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=900):
    r = subprocess.run([sys.executable, "bench.py"] + args, capture_output=True, text=True, cwd=ROOT,
                       timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_line_ours():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = _run(["--config", "3", "--steps", "3", "--warmup", "3", "--cpu-budget", "3"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["higher_is_better"] is True and d["scaling"] == "weak" and d["dtype"] == "c128"
    assert "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] in ("tensor", "hbm") and r["peak"] > 0 and r["achieved"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) <= 1e-9 * r["frac"]
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["check"]["max_rel_diff_vs_graph_path"] == 0.0


def test_bench_line_reference():
    d = _run(["--impl", "reference", "--config", "3", "--steps", "1", "--warmup", "3"])
    assert d["impl"] == "reference" and d["value"] > 0 and d["dtype"] == "c128"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0
    ours_cfg = _run(["--config", "3", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"])["config"]
    assert d["config"] == ours_cfg           # same workload, metric and unit as our arm
