"""bench.py contract pieces that run without a GPU: the reference arm (the fp64 oracle on
a bounded sample) prints one JSON line with the required keys."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert "workload" in line["config"]


def test_oracle_timing_tool_c1():
    """tools/oracle_timing.py (SURVEY §8(d) oracle timing): one JSON line per (config, cores),
    the 1-core line really pinned to one BLAS thread."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "oracle_timing.py"), "--configs", "C1", "--steps", "1"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(s) for s in r.stdout.strip().splitlines()]
    assert len(lines) == 2 and all(l["config"] == "C1" for l in lines)
    assert lines[0]["cores"] >= 1 and lines[1]["cores"] == 1
    for l in lines:
        assert l["frames_per_s"] > 0 and l["steps"] == 1 and l["kind"].startswith("oracle")
