"""bench.py's reference arm runs on host cores only (the oracle port of the
reference kernel), so its JSON contract is checked here without a GPU: one
line, the headline metric, `impl: reference`, a cpu_baseline describing the
run and an e2e block with no host<->device bytes."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_json_contract():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "3", "--ref-sample", "1024")
    assert d["impl"] == "reference"
    assert d["metric"].startswith("projected points/sec")
    assert d["unit"] == "points/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] >= 3
    assert d["dtype"] == "f64" and d["data"] == "synthetic"
    assert d["config"]["workload"].startswith("cfg2")
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["sample"]
    assert cb["value"] == d["value"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


def test_reference_arm_surface_config():
    d = _run("--impl", "reference", "--config", "cfg4", "--steps", "1", "--warmup", "3",
             "--ref-sample", "1024")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["config"]["workload"].startswith("cfg4")
