"""The bench line's contract (the driver parses it): every required key, on the
committed round-2 lines (profiles/r02_bench_c3.json, profiles/r02_bench_c3_reference.json)
and on a live reference-arm run on the host (config 1, a 2-second sample).  CPU only."""

import json
import os
import subprocess
import sys

from conftest import ROOT

REQUIRED = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "e2e", "gpu_launches", "cpu_baseline"}


def _line(name):
    return json.load(open(os.path.join(ROOT, "profiles", name)))


def test_b200_bench_line_contract():
    d = _line("r02_bench_c3.json")
    assert REQUIRED <= set(d), REQUIRED - set(d)
    assert d["unit"] == "Gentries/s" and d["higher_is_better"] is True and d["scaling"] == "weak"
    assert "workload" in d["config"] and "model" not in d["config"] and d["config"]["workload"].startswith("config3")
    assert d["state_check"] is True and d["deterministic_steps"] is True
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r) and r["bound"] in ("hbm", "tensor")
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9 and r["frac"] <= 1.2
    e = d["e2e"]
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(e) and e["h2d_bytes_per_step"] > 0
    assert e["unit"] == d["unit"] and e["same_decisions"] is True
    c = d["cpu_baseline"]
    assert {"value", "unit", "cores", "kind", "sample"} <= set(c) and c["kind"] in ("port", "reference")
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["gpu_launches"] > 0 and d["warmup"] >= 3
    k = d["kernel_microbench"]["roofline"]
    assert k["bound"] == "hbm" and 0 < k["frac"] <= 1.0


def test_reference_arm_line_contract():
    d = _line("r02_bench_c3_reference.json")
    assert d["impl"] == "reference" and d["unit"] == "Gentries/s"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert {"value", "cores", "kind", "sample"} <= set(d["cpu_baseline"]) and d["cpu_baseline"]["kind"] == "reference"
    assert d["ms_per_step"] * d["steps"] <= 1.01e3 * d["consistency"]["timed_seconds"]


def test_reference_arm_runs_on_the_host():
    """`bench.py --impl reference` (the unmodified numpy reference from baseline/_ref)
    prints a contract line without any GPU, or `unavailable` if it is not installed."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                          "--steps", "1", "--warmup", "0", "--ref-seconds", "2"], capture_output=True, text=True,
                         timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference"
    if "unavailable" in d:
        return
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"] and d["cpu_baseline"]["cores"] >= 1
