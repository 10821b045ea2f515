"""bench.py keeps the driver's JSON contract: one line, the required keys (the GPU arm on a B200,
the reference (oracle) arm on the CPU)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def run(args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         cwd=ROOT, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = run(["--impl", "reference", "--config", "C1", "--steps", "1", "--warmup", "0"])
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["value"] > 0 and d["higher_is_better"] is True


@pytest.mark.gpu
def test_gpu_arm_contract():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    d = run(["--config", "C1", "--steps", "3", "--warmup", "3"])
    assert BASE_KEYS <= set(d) and {"roofline", "gpu_launches", "clocks"} <= set(d)
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r) and r["bound"] == "alu"
    assert 0 < r["frac"] < 1.2 and abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-9
    assert {"value", "unit", "cores", "kind", "sample"} <= set(d["cpu_baseline"])
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] == 1000 * 3 * 8 * 2 and e["d2h_bytes_per_step"] == 1000 * 3 * 8
    assert d["gpu_launches"] > 0 and d["n_gpus"] == 1 and d["warmup"] >= 3
    assert d["check"]["E_vs_gpu_direct"] < 1e-2
