"""bench.py on the GPU: the JSON line carries every contract key (-m gpu)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_bench_json_contract_tiny():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "tiny",
                        "--steps", "5", "--warmup", "3", "--e2e-steps", "1", "--no-cpu"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "clocks", "gpu_launches", "e2e"):
        assert k in d, k
    assert d["steps"] == 5 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["gpu_launches"] == 5                      # one fused kernel per round
    assert d["config"]["workload"] == "tiny"
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["achieved"] > 0 and rf["peak"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-3
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["clocks"]["sm_mhz"] is None or d["clocks"]["sm_mhz"] > 0


def test_c_example_runs():
    import runpy
    b = runpy.run_path(os.path.join(ROOT, "paper_1805_07891_b200", "build.py"))
    exe = b["build_example"]()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 mismatches" in r.stdout
