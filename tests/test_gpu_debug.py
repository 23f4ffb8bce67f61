"""The PRK_DEBUG build (in-kernel shared/global index checks that trap) runs every
kernel family without a violation and gives the release build's bits."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def digest(lib):
    env = dict(os.environ)
    if lib:
        env["PR_LIB"] = lib
    res = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "debug_check.py")], capture_output=True,
                         text=True, timeout=900, cwd=ROOT, env=env)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-3000:]
    return [l for l in res.stdout.splitlines() if l.startswith("digest")][-1]


def test_debug_build_checks_and_bits():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    sys.path.insert(0, ROOT)
    from paper_1409_8563_b200 import build as b
    dbg = b.build(debug=True)
    assert digest(dbg) == digest(None)
