"""bench.py contract pieces that run without a GPU (-m "not gpu")."""
import json
import os
import subprocess
import sys

from conftest import ROOT


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--config", "tiny", "--steps", "2", "--warmup", "1"],
                       capture_output=True, text=True, timeout=300,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["value"] > 0
    assert d["config"]["E"] == 288768 and "full" in d["cpu_baseline"]["sample"]   # no sampling


def test_reference_arm_nonzero_rank_is_silent():
    env = dict(os.environ, RANK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--config", "tiny", "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_results_csv_schema(tmp_path):
    """scripts/results_csv.py: fixed header, one row per bench.py JSON line."""
    d = tmp_path / "p"
    d.mkdir()
    (d / "a.json").write_text('noise\n{"metric": "m", "value": 1.5, "n_gpus": 2, "config": '
                              '{"workload": "vgg19", "workers": 8}, "roofline": {"frac": 0.9}}\n')
    (d / "b.json").write_text('{"not": "a bench line"}\n')
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "results_csv.py"), str(d)],
                       capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert lines[0].split(",")[:4] == ["file", "impl", "workload", "n_gpus"]
    assert len(lines) == 2 and ",vgg19,2,8," in lines[1] and ",0.9," in lines[1]
