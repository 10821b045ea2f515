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


def run(args, env=None):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         cwd=ROOT, timeout=900, env=env)
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


def test_reference_arm_same_config_string():
    # both arms name the workload identically (the driver compares them)
    import bench
    d = run(["--impl", "reference", "--config", "C1", "--steps", "1", "--warmup", "0"])
    assert d["config"] == {"workload": bench.workload("C1")}
    m = d["cpu_baseline"]["measured_per_step"]
    assert m["sample_wall_s"] > 0 and m["eval_scale"] >= 1.0


def test_launcher_starts_n_ranks():
    # --gpus N without a torch.distributed environment re-runs the bench under
    # torch.distributed.run with N ranks (dry run: gloo on the CPU, one all-reduce)
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    d = run(["--gpus", "2", "--dry-run"], env=env)
    assert d == {"dry_run": True, "n_gpus": 2, "ranks_seen": 2, "gpus_arg": 2}
    d = run(["--gpus", "1", "--dry-run"], env=env)
    assert d["n_gpus"] == 1


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, cwd=ROOT, timeout=300, env=env)
    assert out.returncode != 0 and "one rank per GPU" in out.stderr


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
    import bench
    assert d["config"] == {"workload": bench.workload("C1")} and "A19" in d["precision"]
    assert r["peak_measured"] is None or 20 < r["peak_measured"] < 40


@pytest.mark.gpu
def test_gpu_arm_explicit_gpus_1():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    d = run(["--gpus", "1", "--config", "C1", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-e2e"])
    assert d["n_gpus"] == 1 and d["value"] > 0
