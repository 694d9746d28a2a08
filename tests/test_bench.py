"""bench.py keeps the driver's JSON-line contract.

- CPU: the reference arm (`--impl reference`), on C0.
- GPU: our arm, on C1, with e2e, cpu_baseline, roofline, clocks and
  gpu_launches.
"""

import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config"}


def _run(*args, env=None):
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args], cwd=REPO, env=env,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_json_line(oracle_mod):
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    d = _run("--impl", "reference", "--workload", "C0", "--steps", "2", "--warmup", "1", env=env)
    assert BASE_KEYS <= d.keys()
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["workload"] == "C0"
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["cores"] >= 1
    if os.path.isdir(os.path.join(REPO, "baseline", "_ref", "hbproxy")):
        # the unmodified reference (numba run_case) with the C port beside it
        assert cb["kind"] == "reference" and "run_case" in cb["sample"]
        assert cb["port"]["value"] > 0
    else:
        assert cb["kind"] == "port"
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_our_arm_json_line(cuda):
    d = _run("--workload", "C1", "--steps", "4", "--warmup", "3", "--cpu-sample-iters", "1")
    assert BASE_KEYS <= d.keys()
    assert d["n_gpus"] == 1 and d["steps"] == 4 and d["warmup"] == 3 and d["value"] > 0
    assert d["dtype"] == "f64" and d["config"]["workload"] == "C1"
    assert d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["bound"] in ("fp64", "hbm") and 0 < r["frac"] < 1.5 and r["peak"] > 0
    assert d["cpu_baseline"]["value"] > 0 and d["cpu_baseline"]["cores"] >= 1
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


def test_our_arm_refuses_library_knobs():
    """A bench line is never taken with a libhbgpu test knob set unknowingly
    (HBGPU_GRID_LIMIT, HBGPU_FUSED, ...): the arm exits before touching a GPU."""
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0", HBGPU_GRID_LIMIT="3")
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--workload", "C0"], cwd=REPO,
                         env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode != 0 and "refusing to benchmark" in out.stderr
