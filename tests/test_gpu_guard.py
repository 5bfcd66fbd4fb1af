"""Out-of-bounds check without compute-sanitizer, which is closed on this
GPU pool: tools/guard_check.py runs every kernel family with WRMG_GUARD=1 (4 KB guard
bands of 0xFF around every device allocation of the library: out-of-bounds reads
poison the oracle comparisons with NaN / -1 indices, out-of-bounds writes are
detected when the bands are freed) in a fresh process."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_guard_bands_clean():
    env = dict(os.environ, WRMG_GUARD="1")
    p = subprocess.run([sys.executable, "tools/guard_check.py"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=1200)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert "guard violations 0" in p.stdout
