"""The drop-in boundary without a GPU: libqmcg.so loads, exports every symbol
include/qmcg.h declares (and the C++ drop-in of include/qmc_b200/qmc.hpp), the
headers compile as C and C++, and the host-only parts of the ABI (tree node
ranges, the fixed-order combine) reproduce the reference's pairwise tree."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INC = os.path.join(ROOT, "include")


def declared_symbols():
    text = open(os.path.join(INC, "qmcg.h")).read()
    return sorted(set(re.findall(r"\b(qmcg_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_header(qmcg):
    lib = qmcg.load_library()
    names = declared_symbols()
    assert len(names) >= 18
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(qmcg.qmcg.EXPORTS)
    nm = subprocess.run(["nm", "-D", "--defined-only", qmcg.qmcg.LIB_PATH], capture_output=True, text=True).stdout
    for sym in ("_ZN3qmc14price_americanERKNS_10OptionSpecEllmRKNS_10ExecPolicyE",
                "_ZN3qmc17convergence_curveERKNS_10OptionSpecERKSt6vectorIlSaIlEElmRKNS_10ExecPolicyE"):
        assert sym in nm, sym
    assert lib.qmcg_version().startswith(b"qmcg")


def test_headers_compile(tmp_path):
    c = tmp_path / "t.c"
    c.write_text('#include "qmcg.h"\nint main(void){qmcg_option_spec s={100,100,0.05,0.2,1,QMCG_CALL};'
                 "return s.kind;}\n")
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", INC, "-c", str(c), "-o", str(tmp_path / "t.o")],
                   check=True)
    cpp = tmp_path / "t.cpp"
    cpp.write_text('#include "qmc_b200/qmc.hpp"\nint main(){qmc::OptionSpec s; qmc::ExecPolicy e;'
                   " (void)e; return s.kind == qmc::OptionKind::Call ? 0 : 1;}\n")
    subprocess.run(["g++", "-std=c++17", "-Wall", "-Werror", "-I", INC, "-c", str(cpp), "-o",
                    str(tmp_path / "u.o")], check=True)


def test_no_gpu_fails_loudly(qmcg):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError):
        qmcg.Context(0)


def test_tree_nodes_partition(qmcg):
    for n in (2, 65, 129, 1000, 1 << 16, 1_000_003):
        for depth in range(0, 6):
            if (n >> max(depth - 1, 0)) <= 64 and depth > 0:
                continue
            prev = 0
            for node in range(1 << depth):
                b, e = qmcg.tree_node_range(n, depth, node)
                assert b == prev and e > b
                prev = e
            assert prev == n


def test_combine_matches_reference_tree(qmcg, oracle_lib):
    """Node sums folded by qmcg_combine_nodes == pairwise_sum over all values, bit for bit."""
    from paper_1205_0106_b200 import distributed
    rng = np.random.default_rng(3)
    for n in (2, 100, 129, 4096, 65537, 1 << 18):
        v = np.abs(rng.standard_normal(n)) * 7
        mean_ref, se_ref = oracle_lib.reduce_stats(v)
        for world in (1, 2, 3, 4, 8):
            depth = distributed.tree_depth(n, world)
            table = np.zeros((1 << depth, 2))
            for node in range(1 << depth):
                b, e = qmcg.tree_node_range(n, depth, node)
                table[node] = [oracle_lib.pairwise_sum(v[b:e]), oracle_lib.pairwise_sum(v[b:e] * v[b:e])]
            assert distributed.combine(n, depth, table) == (mean_ref, se_ref), (n, world)
