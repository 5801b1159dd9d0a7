"""The C++ drop-in (qmc::price_american with the reference's signature) built
against include/qmc_b200/qmc.hpp and libqmcg.so, running the reference's own
price_american test cases (tests/cpp/dropin_test.cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_dropin(qmcg, tmp_path):
    libdir = os.path.dirname(qmcg.qmcg.LIB_PATH)
    exe = tmp_path / "dropin_test"
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp"), "-L", libdir, "-l:libqmcg.so",
                    f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "PASSED" in out.stdout
