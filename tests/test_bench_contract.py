"""bench.py output contract (the driver parses one JSON line): required keys, types and the
self-consistency of the reported numbers, on a short run."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
            "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
            "roofline", "gpu_launches", "clocks", "e2e", "cpu_baseline")


def _run(args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "0",
              "--cpu-seconds", "1"])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "steps/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


@pytest.mark.gpu
def test_bench_line_contract():
    d = _run(["--steps", "3", "--warmup", "3", "--layers", "4", "--cpu-seconds", "1"])
    for k in REQUIRED:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and abs(d["value"] * d["ms_per_step"] - 1e3) < 1e-6 * d["value"] * d["ms_per_step"] + 1e-3
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] < 1.2 and abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-9
    assert d["gpu_launches"] > 0 and d["config"]["workload"].startswith("c2")
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle"


@pytest.mark.gpu
def test_bench_c4_trace_replay_contract():
    """--config c4: a (shortened) trace replay reports steps/s per load regime, and its
    timed replay re-derived the first pass's admission bit for bit (asserted inside)."""
    d = _run(["--config", "c4", "--c4-steps", "700", "--layers", "2", "--warmup", "3"])
    assert d["config"]["workload"].startswith("c4") and d["steps"] == 700
    regs = d["regimes"]
    assert len(regs) == 3 and all(v["steps_per_s"] > 0 for v in regs.values())
    rates = [v["opportunistic_admission_rate"] for v in regs.values()]
    assert rates[0] > rates[1]  # low load admits more than the stress regime (P206-210)
    assert d["gpu_launches"] > 0 and 0 < d["roofline"]["frac"] < 1.3
