"""The table build's 64-bit-magic digit division and endpoint clamp (otherwise reached only near
n = 2^32) bit-identical to the 32-bit path, and the range-checked walk (large m * sigma, the SLOW
pricing-kernel instantiation) within the parity bar of the oracle."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, json
sys.path.insert(0, %r)
import numpy as np
import paper_1205_0106_b200 as q
ctx = q.Context(0)
out = []
for (s, kind, m, n, kw) in %r:
    r = ctx.price_american(q.OptionSpec(*s, kind=q.OptionKind(kind)), m, n, 42, **kw)
    out.append([r.price.hex(), r.std_error.hex()])
u = ctx.uniform_rows(70001, 42, 0, 40)
out.append(int(np.frombuffer(u.tobytes(), dtype=np.uint64).sum(dtype=np.uint64)))
print(json.dumps(out))
"""
CASES = [((100.0, 100.0, 0.05, 0.2, 1.0), 0, 64, 70001, {}),
         ((100.0, 100.0, 0.05, 0.2, 1.0), 1, 40, 4097, {"allow_put": True}),
         ((100.0, 100.0, 0.05, 0.2, 1.0), 0, 48, 65536, {"fp32": True}),
         ((100.0, 95.0, -0.02, 0.3, 1.0), 0, 20, 3001, {})]


def _run(force):
    env = dict(os.environ, QMCG_FORCE_WIDE="1" if force else "0")
    out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, CASES)], env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return out.stdout.strip().splitlines()[-1]


def test_wide_magic_and_clamp_paths_bit_identical(qmcg):
    assert _run(True) == _run(False)


def test_range_checked_walk_vs_oracle(ctx, qmcg, oracle_lib):
    # |X0| + m (|a| + 7.05 b) > 700: the walk checks S against exp's range every date (SLOW)
    for spec, m, n in (((100.0, 100.0, 0.05, 3.0, 10.0), 200, 4097), ((50.0, 60.0, 0.02, 2.5, 8.0), 150, 3001)):
        r = ctx.price_american(qmcg.OptionSpec(*spec), m, n, 42)
        p, se = oracle_lib.price_american(*spec, m, n, 42)
        assert abs(r.price - p) <= 1e-9 * abs(p), (spec, r.price, p)
        assert abs(r.std_error - se) <= 1e-9 * se
