"""The CPU oracle (plain-C restatement, oracle/qmc_oracle.c) pinned against the
reference's own outputs: committed golden fixtures produced by oracle/_ref
(oracle/gen_golden.py) and, where the reference tree is present, the compiled
reference itself. Bit-exact throughout: the restatement keeps the reference's
IEEE operation order and links the same glibc libm."""
import numpy as np
import pytest

import oracle as O
from oracle.gen_golden import fnv1a64_c

REF = (100.0, 100.0, 0.05, 0.2, 1.0)


def fx(h):
    return float.fromhex(h)


def test_permutation_small(golden, oracle_lib):
    g = golden["permutations"]
    assert list(oracle_lib.permutation_indices(8, 42)) == g["perm_8_42"] == [6, 7, 0, 5, 3, 2, 1, 4]
    for d, v in g["dimension_seed"].items():
        assert oracle_lib.dimension_seed(42, int(d)) == int(v)


def test_permutation_tables(golden, oracle_lib):
    for t in golden["permutations"]["tables"]:
        p = oracle_lib.permutation_indices(t["n"], int(t["seed64"]))[: t["n"]]
        assert fnv1a64_c(p) == t["fnv1a64"], t
        assert [int(x) for x in p[:4]] == t["head"][: min(4, t["n"])]
        assert np.array_equal(np.sort(p), np.arange(t["n"], dtype=np.uint32))  # a bijection


def test_permutation_errors(oracle_lib):
    with pytest.raises(O.OracleError) as e:
        oracle_lib.permutation_indices(0, 1)
    assert e.value.code == O.INVALID_ARGUMENT


def test_uniforms(golden, oracle_lib):
    for c in golden["uniforms"]["cases"]:
        u = oracle_lib.uniform_dim(c["dim"] + 1, c["n"], c["seed"], c["dim"])
        assert fnv1a64_c(u) == c["fnv1a64"], c
        assert [x.hex() for x in u[:4]] == c["head_hex"]
        assert u.min() > 0.0 and u.max() < 1.0


def test_analytic(golden, oracle_lib):
    a = golden["analytic"]
    for u, z in a["moro"]:
        assert oracle_lib.moro_inv_cnd(fx(u)).hex() == z
    for d, v in a["cnd"]:
        assert oracle_lib.cnd(fx(d)).hex() == v
    for spec, kind, v in a["bs_price"]:
        assert oracle_lib.bs_price(*spec, kind=kind).hex() == v
    for i, b, v in a["radical_inverse"]:
        assert oracle_lib.radical_inverse(i, b).hex() == v
    with pytest.raises(O.OracleError):
        oracle_lib.moro_inv_cnd(1.0)


def test_prices(golden, oracle_lib):
    done = 0
    for c in golden["prices"]["cases"]:
        if c["n"] * c["m"] > (1 << 22) + 1:
            continue  # the large configs are pinned on the GPU box and by test_oracle_vs_reference
        p, se = oracle_lib.price_american(*c["spec"], c["m"], c["n"], c["seed"])
        assert p.hex() == c["price"] and se.hex() == c["std_error"], c
        done += 1
    assert done >= 20


def test_path_values(golden, oracle_lib):
    g = golden["path_values"]
    _, _, vals = oracle_lib.price_american(*g["spec"], g["m"], g["n"], g["seed"], want_values=True)
    assert [v.hex() for v in vals] == g["values_hex"]


def test_published_numbers(golden):
    """proj/test_output.txt:32-33 (6 significant digits) against the full-precision goldens."""
    published = {(1, 1 << 18): 10.4504, (2, 1 << 18): 11.3072, (5, 1 << 18): 13.3644, (10, 1 << 18): 14.9485,
                 (20, 1 << 18): 16.2522, (50, 1 << 18): 17.4148, (10, 1_000_000): 14.9587}
    seen = 0
    for c in golden["prices"]["cases"]:
        key = (c["m"], c["n"])
        if tuple(c["spec"]) == REF and key in published:
            assert float(f"{fx(c['price']):.6g}") == published[key]
            seen += 1
    assert seen == len(published)


def test_reduce_stats_and_pairwise(oracle_lib, reference_lib):
    rng = np.random.default_rng(7)
    for n in (1, 2, 63, 64, 65, 127, 128, 1000, 4097, 1 << 16, 100003):
        v = rng.standard_normal(n) * 10 + 3
        assert oracle_lib.pairwise_sum(v) == reference_lib.tree_reduce(v)
        if n >= 2:
            assert oracle_lib.reduce_stats(v) == reference_lib.reduce_stats(v)
            assert reference_lib.reduce_stats(v, lanes=8) == reference_lib.reduce_stats(v, lanes=1)


def test_oracle_vs_reference(oracle_lib, reference_lib):
    rng = np.random.default_rng(11)
    for _ in range(12):
        spec = (float(rng.uniform(60, 140)), float(rng.uniform(60, 140)), float(rng.uniform(-0.03, 0.1)),
                float(rng.uniform(0.05, 0.6)), float(rng.uniform(0.1, 3.0)))
        m = int(rng.integers(1, 70))
        n = int(rng.integers(2, 5000))
        seed = int(rng.integers(0, 2**63))
        p, se = oracle_lib.price_american(*spec, m, n, seed)
        pr, ser, _ = reference_lib.price_american(*spec, m, n, seed, lanes=3, chunk=777)
        assert (p, se) == (pr, ser)


def test_oracle_errors_match_reference(oracle_lib, reference_lib):
    bad = [((100, 100, 0.05, 0.2, 1.0), 1, 10, 1, "put"),
           ((100, 100, 0.05, 0.2, 1.0), 10, 1, 0, "n"),
           ((100, 100, 0.05, 0.2, 1.0), 0, 10, 0, "m"),
           ((100, 100, 0.05, 0.2, 0.0), 10, 10, 0, "T"),
           ((-1, 100, 0.05, 0.2, 1.0), 10, 10, 0, "spot"),
           ((100, 100, float("nan"), 0.2, 1.0), 10, 10, 0, "nan")]
    for spec, m, n, kind, _ in bad:
        with pytest.raises(O.OracleError) as eo:
            oracle_lib.price_american(*spec, m, n, 42, kind=kind)
        with pytest.raises(O.OracleError) as er:
            reference_lib.price_american(*spec, m, n, 42, kind=kind)
        assert str(eo.value) == str(er.value) and eo.value.code == er.value.code


def test_put_extension_properties(oracle_lib, reference_lib):
    """Puts are an opt-in extension (the reference throws): parity is UNPINNED, so
    only the reference's own property tests apply (test_american.cpp:127-135)."""
    for spec in [(100, 100, 0.05, 0.2, 1.0), (90, 100, 0.03, 0.3, 0.5), (110, 100, 0.08, 0.15, 2.0)]:
        p, se = oracle_lib.price_american(*spec, 20, 1 << 14, 42, kind=O.PUT, allow_put=True)
        assert p >= reference_lib.bs_price(*spec, kind=O.PUT) - 3 * se
        assert p >= reference_lib.crr_price(*spec, 512, True, kind=O.PUT) - 3 * se


def test_crr_dominance(golden, oracle_lib):
    """Acceptance criterion 5 (acceptance.cpp:118-154) on the oracle."""
    for c in golden["crr"]:
        p, se = oracle_lib.price_american(*c["spec"], 20, 1 << 15, 42)
        assert p >= c["american_call"] - 3 * se
        assert p >= c["bs_call"] - 3 * se
