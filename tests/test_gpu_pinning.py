"""Reference-pinned bit-level parity of the pricing path itself (not only the D1 exports).

* The uniforms the pricing kernels read -- the resident uniform table, built by K1 +
  uniforms_kernel and exported with qmcg_uniform_rows -- are bit-identical to the reference's
  uniform_at (proj/src/quasi_rng.cpp:71-83,96-101) for every column the config-2 and config-3
  pricings read: FNV-1a-64 of each column against hashes produced by the reference itself
  (oracle/gen_golden.py --only-columns).
* The GPU pairwise tree (K3) returns exactly the reference's reduce_stats
  (proj/src/path_engine.cpp:39-47,191-205) of the GPU's own per-path values, with `==`,
  for ragged and power-of-two n.
* Config 4 at its full size (1024 contracts, 2^18 paths x 128 dates) against the
  reference's price_american on 8 grid calls (tests/golden/config4.json).
* The put extension at the headline size (2^24 x 256) satisfies the reference's own lower
  bounds (acceptance.cpp:118-154 applied to puts): >= BS put - 3 se and >= CRR American put
  (2048 steps) - 3 se.
"""
import numpy as np
import pytest

from oracle.gen_golden import fnv1a64_c

pytestmark = pytest.mark.gpu

REF = (100.0, 100.0, 0.05, 0.2, 1.0)


def fx(h):
    return float.fromhex(h)


@pytest.fixture(scope="module")
def reducer(oracle_lib):
    """The reference's reduce_stats where oracle/_ref is present (it travels to the GPU box),
    else the C restatement, which is pinned bit-exact to it (tests/test_oracle.py)."""
    import oracle
    if oracle.reference_available():
        R = oracle.Reference()
        return lambda v: R.reduce_stats(np.ascontiguousarray(v), lanes=1)
    return lambda v: oracle_lib.reduce_stats(np.ascontiguousarray(v))


@pytest.mark.parametrize("which", [0, 1], ids=["c2_2^20x100", "c3_2^24x256"])
def test_pricing_generator_uniforms_match_reference_columns(ctx, golden, which):
    sets = golden["uniform_columns"]["sets"][which]
    n, dims, hashes = sets["n"], sets["dims"], sets["fnv1a64"]
    step = 100 if n <= 1 << 20 else 16
    bad = []
    for d0 in range(0, dims, step):
        cnt = min(step, dims - d0)
        rows = ctx.uniform_rows(n, 42, d0, cnt)
        for k in range(cnt):
            if fnv1a64_c(rows[k]) != hashes[d0 + k]:
                bad.append(d0 + k)
    assert not bad, f"columns differing from the reference at n={n}: {bad}"


def test_pricing_generator_uniforms_vs_oracle_small(ctx, oracle_lib):
    # ragged n (partial last block / chunk), bases with 2..7 digits and the base-2 reversal
    for n, dims in ((1000, 40), (4097, 33), (70001, 20)):
        rows = ctx.uniform_rows(n, 7, 0, dims)
        for d in range(dims):
            ref = oracle_lib.uniform_dim(dims, n, 7, d)
            assert np.array_equal(rows[d].view(np.uint64), ref.view(np.uint64)), (n, d)
    # a window that does not start at dimension 0
    rows = ctx.uniform_rows(5000, 42, 37, 11)
    for k in range(11):
        ref = oracle_lib.uniform_dim(48, 5000, 42, 37 + k)
        assert np.array_equal(rows[k].view(np.uint64), ref.view(np.uint64)), 37 + k


@pytest.mark.parametrize("n", [2, 3, 63, 64, 65, 127, 129, 4097, 16461, 100003, 1 << 20, 1 << 24])
def test_gpu_tree_equals_reference_reduce_stats(ctx, qmcg, reducer, n):
    m = 256 if n == 1 << 24 else 33
    spec = qmcg.OptionSpec(*REF)
    r = ctx.price_american(spec, m, n, 42)
    v = ctx.path_values(spec, m, n, 42)
    mean, se = reducer(v)
    assert r.price == mean and r.std_error == se, (n, r.price, mean, r.std_error, se)


def test_gpu_tree_equals_reference_reduce_stats_put_and_fp32(ctx, qmcg, reducer):
    for kw, kind in (({"allow_put": True}, 1), ({"fp32": True}, 0)):
        spec = qmcg.OptionSpec(*REF, kind=qmcg.OptionKind(kind))
        for n in (129, 100003):
            r = ctx.price_american(spec, 40, n, 42, **kw)
            v = ctx.path_values(spec, 40, n, 42, **kw)
            assert (r.price, r.std_error) == reducer(v), (kw, n)


def test_config4_full_size_vs_reference(ctx, qmcg, golden):
    """The whole 1024-contract grid in one batch call; the 8 reference-priced calls must match."""
    gi, gj = np.meshgrid(np.arange(32), np.arange(32), indexing="ij")
    strike, vol, kind = 80 + 40 * gi.ravel() / 31, 0.10 + 0.40 * gj.ravel() / 31, (gi + gj).ravel() % 2
    res = ctx.price_american_batch_arrays(100.0, strike, 0.05, vol, 1.0, kind, 128, 1 << 18, 42, allow_put=True)
    for c in golden["config4"]["cases"]:
        idx = c["i"] * 32 + c["j"]
        assert strike[idx] == c["spec"][1] and vol[idx] == c["spec"][3] and kind[idx] == 0
        p, se = fx(c["price"]), fx(c["std_error"])
        assert abs(res[idx, 0] - p) <= 1e-9 * p, (c, res[idx])
        assert abs(res[idx, 1] - se) <= 1e-9 * se, (c, res[idx])


def test_put_headline_bounds(ctx, qmcg, golden):
    """The put at 2^24 x 256 (the metric's option) against the reference's own lower bounds."""
    for c in golden["put_bounds"]["cases"]:
        spec = qmcg.OptionSpec(*c["spec"], kind=qmcg.OptionKind.Put)
        r = ctx.price_american(spec, 256, 1 << 24, 42, allow_put=True)
        assert r.price >= c["bs_put"] - 3 * r.std_error, (c, r)
        assert r.price >= c["american_put"] - 3 * r.std_error, (c, r)
        assert 0 < r.std_error < 0.01 * r.price


@pytest.mark.parametrize("n", [1 << 14, 1 << 18, 100003, 4097])
def test_batch_tree_equals_reference_reduce_stats(ctx, qmcg, reducer, n):
    """The batch's tree (the batched leaves kernel + perfect levels over every contract's values)
    equals the reference's reduce_stats of the same launch's per-path values, for power-of-two
    and ragged n, including a contract priced by the single-contract kernel (r < 0)."""
    specs = [qmcg.OptionSpec(100.0, 80 + 40 * i / 5, 0.05, 0.1 + 0.4 * j / 5, 1.0, qmcg.OptionKind((i + j) % 2))
             for i in range(6) for j in range(6)]
    specs.append(qmcg.OptionSpec(100.0, 95.0, -0.01, 0.3, 1.0))  # r < 0: the single-contract kernel
    res, vals = ctx.price_american_batch_values(specs, 24, n, 42, allow_put=True)
    plain = ctx.price_american_batch(specs, 24, n, 42, allow_put=True)
    for i, r in enumerate(res):
        assert (r.price, r.std_error) == reducer(vals[i]), (n, i)
        assert (plain[i].price, plain[i].std_error) == (r.price, r.std_error), (n, i)
        one = ctx.price_american(specs[i], 24, n, 42, allow_put=True)
        assert abs(one.price - r.price) <= 1e-12 * one.price, (n, i)
