"""The warp-per-token unfold (patch.cu, default; soft split and the F3N unfold) against the
per-vector gather unfold (VI_PATCH_V=0): bitwise equal soft split tokens, F3N hidden g of every
block, block outputs and soft composite of two steps, at C3 and C3S."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["C3", "C3S"])
def test_patch_variants_bitwise(tmp_path, name):
    outs = []
    for v in ("0", "1"):
        f = tmp_path / f"v{v}.npz"
        env = dict(os.environ, VI_PATCH_V=v)
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", "patch_dump.py"), name, str(f)], env=env,
                       check=True, cwd=ROOT, timeout=600)
        outs.append(np.load(f))
    a, b = outs
    assert sorted(a.files) == sorted(b.files)
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k
