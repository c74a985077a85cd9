"""bench.py's one-line JSON contract (the driver parses it): the reference arm runs here on the CPU (it
is the oracle on host cores), our arm on the GPU, both on the tiny config so that they finish fast."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_contract_on_cpu():
    d = _run(["--impl", "reference", "--config", "tiny", "--steps", "2", "--warmup", "1"], 300)
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["unit"] == "TFLOPS" and d["higher_is_better"] is True
    assert d["steps"] == 2 and d["warmup"] == 1 and d["n_gpus"] == 1
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert "workload" in d["config"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_our_arm_contract_on_gpu():
    d = _run(["--config", "tiny", "--steps", "3", "--warmup", "3", "--no-dense", "--cpu-seconds", "2"], 600)
    assert BASE_KEYS <= set(d)
    assert d["metric"].startswith("block-sparse attn fwd") and d["unit"] == "TFLOPS" and d["value"] > 0
    assert d["steps"] == 3 and d["warmup"] == 3 and d["scaling"] in ("weak", "strong")
    assert d["config"]["workload"].startswith("tiny")
    roof = d["roofline"]
    assert roof["bound"] == "tensor" and roof["unit"] == "TFLOP/s" and roof["peak"] > 0
    assert abs(roof["frac"] - roof["achieved"] / roof["peak"]) < 1e-3
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 3 * 2 * 256 * 64 * 2 and e["d2h_bytes_per_step"] == 2 * 256 * 64 * 2
    assert d["gpu_launches"] > 0
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0
    assert "libmoddit.so" in d["library"]
