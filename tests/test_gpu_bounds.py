"""Out-of-bounds write check of every kernel family (compute-sanitizer is closed on this pool:
"runs under it have left GPUs needing a reset"). tools/canary_small.py runs small cases of K1
(direct and binned scatter), K2 (call, put, FP32, r < 0, sigma = 0, streamed windows), K3, K4, the
European kernel, the exports and a device group with QMCG_CANARY=1: every device buffer is
bracketed by 4 KB guard regions that qmcg_check_canaries() verifies after each call."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_no_out_of_bounds_writes(qmcg):
    env = dict(os.environ, QMCG_CANARY="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "canary_small.py")], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=900)
    text = out.stdout + out.stderr
    assert out.returncode == 0, text[-3000:]
    assert "canary_small ok" in text
