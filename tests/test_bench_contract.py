"""bench.py keeps the driver's JSON contract (one line, required keys), for
the reference arm on CPU and for our arm on a B200 (tiny configs)."""

import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout):
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args], cwd=REPO,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "1", "--n-sites", "20000",
              "--width", "64", "--height", "48"], 900)
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_our_arm_contract(cuda_ok):
    d = _run(["--steps", "3", "--warmup", "3", "--n-sites", "20000", "--width", "256",
              "--height", "128", "--no-cpu-baseline"], 900)
    assert BASE_KEYS <= set(d)
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["gpu_launches"] > 0
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r)
    assert d["e2e"]["value"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["fwd_bwd"]["value"] > 0
    assert d["adjacency_rebuild"]["csr_equals_fixture"] is True
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
