"""Regression test for the intermittent stream-K attention hang (profiles/r02_hang.md): before
mbar_wait_warp, a C3 step graph replayed a few thousand times hung with probability ~0.3-0.5
(a softmax warp's lanes fell a barrier phase apart).  The replays run in a subprocess under a
watchdog, so a hang fails the test instead of stalling the suite."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_c3_step_replays_do_not_hang():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "stress_step.py"), "C3", "6000", "0", "20"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, f"stress exit {r.returncode}:\n{r.stdout[-2000:]}\n{r.stderr[-2000:]}"
    assert "done 6000 steps" in r.stdout
