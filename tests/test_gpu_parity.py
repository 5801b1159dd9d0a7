"""Parity of the CUDA path (through the C ABI) with the reference.

Bit-exact: permutation tables (K1), uniforms (D1 / the radical inverse inside
K2), the pairwise reduction tree (K3, across any node decomposition).
Tolerance: prices, standard errors and per-path values agree with the
reference to |rel| <= 1e-9 (north star: <= 1e-6 in FP64); the only
differences are CUDA vs glibc exp/log last-ulp and the log-space GBM walk.
Normals: within 1e-12 relative of the reference's moro_inv_cnd."""
import numpy as np
import pytest

import oracle as O
from oracle.gen_golden import fnv1a64_c

pytestmark = pytest.mark.gpu

REF = (100.0, 100.0, 0.05, 0.2, 1.0)
PRICE_RTOL = 1e-9   # measured ~3e-15; north-star bar is 1e-6
NORTH_STAR_RTOL = 1e-6


def fx(h):
    return float.fromhex(h)


def spec_of(q, s, kind=0):
    return q.OptionSpec(*s, kind=q.OptionKind(kind))


def test_permutations_bit_exact(ctx, golden, oracle_lib):
    for t in golden["permutations"]["tables"]:
        p = ctx.permutation(t["n"], int(t["seed64"]))[: t["n"]]
        assert fnv1a64_c(p) == t["fnv1a64"], t
    assert list(ctx.permutation(8, 42)) == golden["permutations"]["perm_8_42"]
    rng = np.random.default_rng(5)
    for n in (1, 2, 3, 31, 32, 33, 255, 256, 257, 1023, 4099, 65537, 300007):
        s = int(rng.integers(0, 2**64 - 1, dtype=np.uint64))
        assert np.array_equal(ctx.permutation(n, s)[:n], oracle_lib.permutation_indices(n, s)[:n]), n


def test_uniforms_bit_exact(ctx, golden, oracle_lib):
    for c in golden["uniforms"]["cases"]:
        u = ctx.uniforms(c["n"], c["seed"], c["dim"])
        assert fnv1a64_c(u) == c["fnv1a64"], c
    for n, dim in ((4097, 0), (4097, 7), (50000, 29), (50000, 255), (1 << 18, 364), (3000, 1500)):
        g = ctx.uniforms(n, 42, dim)
        r = oracle_lib.uniform_dim(dim + 1, n, 42, dim)
        assert np.array_equal(g.view(np.uint64), r.view(np.uint64)), (n, dim)


def test_normals_close(ctx, oracle_lib):
    for n, dim in ((1 << 16, 0), (1 << 16, 3), (1 << 16, 200)):
        u = oracle_lib.uniform_dim(dim + 1, n, 42, dim)
        z_ref = np.array([oracle_lib.moro_inv_cnd(x) for x in u])
        z = ctx.normals(n, 42, dim)
        assert np.max(np.abs(z - z_ref) / np.maximum(np.abs(z_ref), 1e-3)) < 1e-12


def test_prices_match_reference_goldens(ctx, golden, qmcg):
    for c in golden["prices"]["cases"]:
        r = ctx.price_american(spec_of(qmcg, c["spec"]), c["m"], c["n"], c["seed"])
        p, se = fx(c["price"]), fx(c["std_error"])
        tol = PRICE_RTOL * max(abs(p), 1e-12)
        assert abs(r.price - p) <= tol, (c, r.price)
        # se = sqrt((sum v^2 - n mean^2) / (n - 1) / n) cancels catastrophically when the paths
        # agree (sigma = 0): allow that cancellation floor, sqrt(1e-13 p^2 / n), besides the relative bar
        se_tol = PRICE_RTOL * se + (1e-13 * p * p / c["n"]) ** 0.5
        assert abs(r.std_error - se) <= se_tol, (c, r.std_error)
        assert abs(r.price - p) <= NORTH_STAR_RTOL * abs(p)
        assert r.n_paths == c["n"] and r.seed == c["seed"] and r.method == qmcg.Method.AmericanUpperBound


def test_path_values(ctx, golden, qmcg):
    g = golden["path_values"]
    v = ctx.path_values(spec_of(qmcg, g["spec"]), g["m"], g["n"], g["seed"])
    ref = np.array([fx(h) for h in g["values_hex"]])
    assert np.max(np.abs(v - ref) / np.maximum(np.abs(ref), 1e-300)) < 1e-9


@pytest.mark.parametrize("n,m", [(2, 1), (3, 2), (255, 9), (257, 17), (1000, 8), (4097, 33), (20000, 7)])
def test_edge_sizes_vs_oracle(ctx, qmcg, oracle_lib, n, m):
    for s in (REF, (95.0, 100.0, 0.0, 0.35, 2.0), (100.0, 90.0, -0.01, 0.25, 0.5)):
        p, se, vals = oracle_lib.price_american(*s, m, n, 42, want_values=True)
        v = ctx.path_values(spec_of(qmcg, s), m, n, 42)
        assert np.max(np.abs(v - vals) / np.maximum(np.abs(vals), 1e-300)) < 1e-9
        r = ctx.price_american(spec_of(qmcg, s), m, n, 42)
        assert abs(r.price - p) <= PRICE_RTOL * max(p, 1e-12)


def test_put_extension_vs_oracle(ctx, qmcg, oracle_lib):
    """Opt-in puts: parity with the C restatement of the mirrored rule; UNPINNED vs the reference."""
    for s in (REF, (90.0, 100.0, 0.03, 0.3, 0.5), (100.0, 110.0, -0.02, 0.3, 1.0), (100.0, 100.0, 0.05, 0.0, 1.0)):
        p, se = oracle_lib.price_american(*s, 25, 1 << 13, 42, kind=O.PUT, allow_put=True)
        r = ctx.price_american(spec_of(qmcg, s, 1), 25, 1 << 13, 42, allow_put=True)
        assert abs(r.price - p) <= PRICE_RTOL * max(p, 1e-12), (s, r.price, p)


def test_reference_error_behaviour(ctx, qmcg):
    cases = [((100, 100, 0.05, 0.2, 1.0), 1, 10, 1,
              "price_american: not implemented for puts; the foresight algorithm is call-only"),
             ((100, 100, 0.05, 0.2, 1.0), 10, 1, 0, "price_american: n_paths must be >= 2"),
             ((100, 100, 0.05, 0.2, 1.0), 0, 10, 0, "make_schedule: m must be >= 1"),
             ((100, 100, 0.05, 0.2, 0.0), 10, 10, 0, "make_schedule: maturity must be > 0"),
             ((-1, 100, 0.05, 0.2, 1.0), 10, 10, 0, "OptionSpec: spot must be > 0"),
             ((100, 0, 0.05, 0.2, 1.0), 10, 10, 0, "OptionSpec: strike must be > 0"),
             ((100, 100, 0.05, -0.2, 1.0), 10, 10, 0, "OptionSpec: volatility must be >= 0"),
             ((100, 100, float("inf"), 0.2, 1.0), 10, 10, 0, "OptionSpec: all fields must be finite")]
    for s, m, n, kind, msg in cases:
        with pytest.raises(ValueError) as e:
            ctx.price_american(spec_of(qmcg, s, kind), m, n, 42)
        assert str(e.value) == msg
    with pytest.raises(OverflowError):
        ctx.price_american(spec_of(qmcg, REF), 1, 1 << 32, 42)
    with pytest.raises(ValueError):
        ctx.price_american(spec_of(qmcg, REF), 1, 10, 42, exec=qmcg.ExecPolicy(lanes=0))


def test_deterministic_and_cache_invariant(ctx, qmcg):
    s = spec_of(qmcg, REF)
    a = ctx.price_american(s, 37, 100003, 9)
    b = ctx.price_american(s, 37, 100003, 9)
    c = ctx.price_american(s, 37, 100003, 9, no_cache=True)
    ctx.clear_cache()
    ctx.price_american(s, 11, 100003, 9)  # table grows from 11 to 37 dates below
    d = ctx.price_american(s, 37, 100003, 9)
    assert (a.price, a.std_error) == (b.price, b.std_error) == (c.price, c.std_error) == (d.price, d.std_error)


def test_node_decomposition_bit_identical(ctx, qmcg):
    """The multi-GPU decomposition (one tree node per rank) on one GPU: every depth
    gives the same bits as the single call (reference: bit-identical across lanes)."""
    from paper_1205_0106_b200 import distributed
    s = spec_of(qmcg, REF)
    for n in (1 << 16, 100003):
        full = ctx.price_american(s, 40, n, 42)
        for world in (2, 3, 4, 8):
            depth = distributed.tree_depth(n, world)
            table = np.stack([ctx.price_american_node(s, 40, n, 42, depth, node) for node in range(1 << depth)])
            assert distributed.combine(n, depth, table) == (full.price, full.std_error)
        ctx.clear_cache()


def test_batch_matches_single(ctx, qmcg):
    """Batch pricing (shared normal table generated once + multi-contract walk) against
    single calls: the same numbers up to the order of the log-price additions."""
    specs = [spec_of(qmcg, (100.0, 80 + 4 * i, 0.05, 0.1 + 0.05 * i, 1.0), kind=i % 2) for i in range(6)]
    specs.append(spec_of(qmcg, (100.0, 100.0, -0.01, 0.2, 1.0)))   # r < 0: fused path inside the batch
    specs.append(spec_of(qmcg, (100.0, 100.0, 0.05, 0.0, 1.0)))    # sigma = 0: fused path inside the batch
    batch = ctx.price_american_batch(specs, 24, (1 << 14) + 77, 42, allow_put=True)
    for s, r in zip(specs, batch):
        one = ctx.price_american(s, 24, (1 << 14) + 77, 42, allow_put=True)
        assert abs(one.price - r.price) <= 1e-12 * max(one.price, 1e-300), (s, one.price, r.price)
        assert abs(one.std_error - r.std_error) <= 1e-9 * one.std_error + 1e-12


@pytest.mark.parametrize("layout", ["one_plain_first", "plain_after_fused", "rates_interleaved"])
def test_batch_host_ordering(ctx, qmcg, layout):
    """The batch enqueues the shared prefix sums before planning the other contracts (speculatively
    when the first is plain) and uploads one discount chain per distinct discount factor: results
    must not depend on which contract comes first or how the rates interleave."""
    plain = spec_of(qmcg, (100.0, 95.0, 0.05, 0.25, 1.0))
    flat = spec_of(qmcg, (100.0, 100.0, 0.05, 0.0, 1.0))        # sigma = 0: fused path
    if layout == "one_plain_first":  # speculative prefix sums, then no shared walk at all
        specs = [plain, flat]
    elif layout == "plain_after_fused":
        specs = [flat, plain, spec_of(qmcg, (100.0, 110.0, 0.05, 0.25, 1.0), kind=1)]
    else:
        specs = [spec_of(qmcg, (100.0, 90 + 5 * i, (0.01, 0.07, 0.03)[i % 3], 0.2, 1.0), kind=i % 2) for i in range(9)]
    n, m = (1 << 13) + 5, 20
    batch = ctx.price_american_batch(specs, m, n, 42, allow_put=True)
    for s, r in zip(specs, batch):
        one = ctx.price_american(s, m, n, 42, allow_put=True)
        assert abs(one.price - r.price) <= 1e-12 * max(one.price, 1e-300), (layout, s, one.price, r.price)


@pytest.mark.parametrize("rate,vol", [(0.05, 0.2), (0.15, 0.05), (0.0, 0.3)])
def test_batch_grouped_strikes(ctx, qmcg, rate, vol):
    """The grouped batch walk: many strikes of both kinds sharing (spot, rate, vol, maturity), plus a
    second spot, against single calls. (0.15, 0.05) makes records rarely dominate, so candidate
    lists overflow the per-path buffer and exercise the flush."""
    specs = [spec_of(qmcg, (spot, k, rate, vol, 1.5), kind=kind)
             for spot in (100.0, 97.0) for kind in (0, 1) for k in (70.0, 85.0, 95.0, 100.0, 104.0, 120.0, 150.0)]
    m, n = 128, 4096 + 96
    batch = ctx.price_american_batch(specs, m, n, 7, allow_put=True)
    for s, r in zip(specs, batch):
        one = ctx.price_american(s, m, n, 7, allow_put=True)
        # 1e-12 relative; deep-tail prices (~1e-200, carried by exp(-d^2/2) at |d| ~ 37) differ
        # in the exponent's rounding, so an absolute floor of 1e-15 x spot applies
        assert abs(one.price - r.price) <= 1e-12 * one.price + 1e-15 * s.spot, (s, one.price, r.price)
        assert abs(one.std_error - r.std_error) <= 1e-9 * one.std_error + 1e-15 * s.spot


def test_config4_grid_vs_oracle(ctx, qmcg, oracle_lib):
    """Config 4's contract grid (32 strikes x 32 vols, calls for even i+j) at a reduced size:
    every contract of an 8 x 8 sub-grid against the C restatement."""
    specs, raw = [], []
    for i in range(0, 32, 4):
        for j in range(0, 32, 4):
            sp = (100.0, 80 + 40 * i / 31, 0.05, 0.10 + 0.40 * j / 31, 1.0)
            kind = (i + j) % 2
            specs.append(spec_of(qmcg, sp, kind))
            raw.append((sp, kind))
    batch = ctx.price_american_batch(specs, 16, 3000, 42, allow_put=True)
    for (sp, kind), r in zip(raw, batch):
        p, se = oracle_lib.price_american(*sp, 16, 3000, 42, kind=kind, allow_put=True)
        assert abs(r.price - p) <= PRICE_RTOL * max(p, 1e-12), (sp, kind, r.price, p)


def test_convergence_curve(ctx, qmcg):
    """Acceptance criterion 6 (acceptance.cpp:157-172): non-decreasing in m within 3 se."""
    curve = qmcg.convergence_curve(qmcg.OptionSpec(*REF), [50, 1, 20, 2, 10, 5], 1 << 18, 42)
    assert [c[0] for c in curve] == [1, 2, 5, 10, 20, 50]
    for (m0, p0, s0, _), (m1, p1, s1, _) in zip(curve, curve[1:]):
        assert p1 >= p0 - 3 * (s0 + s1)
    published = [10.4504, 11.3072, 13.3644, 14.9485, 16.2522, 17.4148]  # proj/test_output.txt:32
    assert [float(f"{c[1]:.6g}") for c in curve] == published


def test_config3_2p24_x_256(ctx, qmcg, golden):
    """Config 3 at full size: against the reference's own 2^24 x 256 price when the
    golden holds it (oracle/gen_golden.py --big), and always against the 2^22 golden
    within 3 combined standard errors."""
    s = spec_of(qmcg, REF)
    r = ctx.price_american(s, 256, 1 << 24, 42)
    g22 = [c for c in golden["prices"]["cases"] if c["m"] == 256 and c["n"] == 1 << 22][0]
    assert abs(r.price - fx(g22["price"])) <= 3 * np.hypot(r.std_error, fx(g22["std_error"]))
    g24 = [c for c in golden["prices"]["cases"] if c["m"] == 256 and c["n"] == 1 << 24]
    if g24:
        assert abs(r.price - fx(g24[0]["price"])) <= PRICE_RTOL * fx(g24[0]["price"])
    ctx.clear_cache()


def test_mc_european_vs_reference_goldens(ctx, qmcg, golden):
    """mc_european_price (reference mc_european.cpp:11-46; the §8f-next sibling of the hot path)."""
    for c in golden["european"]["cases"]:
        r = ctx.mc_european_price(spec_of(qmcg, c["spec"], c["kind"]), c["n"], c["seed"])
        p, se = fx(c["price"]), fx(c["std_error"])
        if se == 0.0:  # volatility or maturity 0: the reference's exact host formula
            assert r.price == p and r.std_error == 0.0, c
        else:
            assert abs(r.price - p) <= PRICE_RTOL * p, (c, r.price)
            assert abs(r.std_error - se) <= PRICE_RTOL * se, (c, r.std_error)
        assert r.method == qmcg.Method.EuropeanMC
    # proj/test_output.txt:29,33 -- 10.4505 at 2^20 paths, 10.4503 at 1e6
    assert f"{ctx.mc_european_price(qmcg.OptionSpec(*REF), 1 << 20, 42).price:.6g}" == "10.4505"
    assert f"{ctx.mc_european_price(qmcg.OptionSpec(*REF), 1_000_000, 42).price:.6g}" == "10.4503"
    with pytest.raises(ValueError) as e:
        ctx.mc_european_price(qmcg.OptionSpec(*REF), 1, 42)
    assert str(e.value) == "mc_european_price: n_paths must be >= 2"


@pytest.mark.parametrize("s,kind,m,n", [(REF, 0, 16, 1 << 14), (REF, 0, 256, 1 << 18),
                                        ((110.0, 100.0, 0.05, 0.3, 2.0), 0, 100, 1 << 16),
                                        (REF, 1, 50, 1 << 16), ((90.0, 100.0, 0.03, 0.3, 0.5), 1, 365, 1 << 15),
                                        ((100.0, 110.0, -0.02, 0.3, 1.0), 0, 33, 1 << 14)])
def test_fp32_variant_within_qmc_error(ctx, qmcg, s, kind, m, n):
    """FP32 variant (north star: 'within the QMC standard error for an FP32 variant'):
    uniforms stay bit-exact FP64; normals and the walk run in FP32, exercise values in FP64.
    Bar: |price32 - price64| <= 0.05 se, and every path value within 5e-5 * spot (FP32 log-price
    walk: ~sqrt(m) ulp(V) * b of error in X, i.e. ~1e-7 relative in S per path)."""
    sp = spec_of(qmcg, s, kind)
    put = kind == 1
    r64 = ctx.price_american(sp, m, n, 42, allow_put=put)
    r32 = ctx.price_american(sp, m, n, 42, allow_put=put, fp32=True)
    assert abs(r32.price - r64.price) <= 0.05 * r64.std_error, (r32.price, r64.price, r64.std_error)
    assert abs(r32.std_error - r64.std_error) <= 1e-3 * r64.std_error
    v64 = ctx.path_values(sp, m, n, 42, allow_put=put)
    v32 = ctx.path_values(sp, m, n, 42, allow_put=put, fp32=True)
    err = np.abs(v32 - v64).max()
    assert err <= 5e-5 * s[0], err


@pytest.mark.parametrize("n", [(1 << 23) + 5, (1 << 24) - 1, (1 << 24) + 1])
def test_permutations_key_width_boundary(ctx, oracle_lib, n):
    """K1 sorts 16-bit keys up to n = 2^24 (8 low bits of j ride in the value) and 32-bit keys
    above (2^24 + 1: 25 index bits, 7 carried bits, 18 sorted): both sides of the switch."""
    s = 0x243F6A8885A308D3 ^ n
    assert np.array_equal(ctx.permutation(n, s)[:n], oracle_lib.permutation_indices(n, s)[:n])


@pytest.mark.parametrize("n", [(1 << 25) + 3, 1 << 26])
def test_permutations_binned_scatter_bit_exact(ctx, oracle_lib, n):
    """K1 from 2^25 entries scatters through 256 i-bins (QMCG_K1_BIN_MIN); same table as the
    serial Fisher-Yates of the C restatement."""
    s = 0x9E3779B97F4A7C15 ^ n
    assert np.array_equal(ctx.permutation(n, s)[:n], oracle_lib.permutation_indices(n, s)[:n])


def test_price_nodes_one_pass(ctx, qmcg):
    """qmcg_price_american_nodes (one kernel over a rank's contiguous nodes) == per-node calls,
    and the folded table == the single call, bit for bit; also for the FP32 variant."""
    sp = spec_of(qmcg, REF)
    n, m, depth = 50003, 30, 3
    for fp32 in (False, True):
        single = ctx.price_american(sp, m, n, 42, fp32=fp32)
        per = np.array([ctx.price_american_node(sp, m, n, 42, depth, k, fp32=fp32) for k in range(8)])
        lo = ctx.price_american_nodes(sp, m, n, 42, depth, 0, 3, fp32=fp32)
        hi = ctx.price_american_nodes(sp, m, n, 42, depth, 3, 5, fp32=fp32)
        table = np.concatenate([lo, hi])
        assert np.array_equal(table, per)
        assert qmcg.combine_nodes(n, depth, table) == (single.price, single.std_error)


def test_tables_build_import(ctx, qmcg):
    """qmcg_build_tables + qmcg_import_tables (the cold multi-GPU path, here with one rank): the
    imported tables price bit-identically to tables the context built itself."""
    import torch
    from paper_1205_0106_b200 import distributed
    n, m = 40000, 24
    s = spec_of(qmcg, REF)
    ctx.clear_cache()
    ref = ctx.price_american(s, m, n, 5)
    ctx.clear_cache()
    distributed.warm_tables_sharded(ctx, n, 5, m)
    got = ctx.price_american(s, m, n, 5)
    assert (got.price, got.std_error) == (ref.price, ref.std_error)
    buf = torch.empty((2, n), dtype=torch.int32, device="cuda")
    ctx.build_tables(n, 5, 3, 4, 2, buf.data_ptr(), n)  # dims 3 and 7
    for j, d in enumerate((3, 7)):
        perm = ctx.permutation(n, int(_dim_seed(5, d)))[:n]
        assert np.array_equal(buf[j].cpu().numpy().view(np.uint32), perm + 1)
    ctx.clear_cache()


def _dim_seed(seed, d):
    def sm(x):
        x = (x + 0x9E3779B97F4A7C15) & (2**64 - 1)
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
        return x ^ (x >> 31)
    return sm(sm(seed) ^ ((d + 0x632BE59BD9B4E019) & (2**64 - 1)))


def test_batch_rejects_fp32(ctx, qmcg):
    mod = qmcg.qmcg
    arr = (mod._CSpec * 1)(mod._cspec(spec_of(qmcg, REF)))
    res = (mod._CResult * 1)()
    st = ctx._lib.qmcg_price_american_batch(ctx._h, arr, 1, 8, 1024, 42, mod.FLAG_FP32, res)
    assert st == mod.UNSUPPORTED
    assert b"FP32" in ctx._lib.qmcg_last_error()


def test_batch_arrays_api(ctx, qmcg):
    """Column-array batch entry == the list-of-specs entry, bit for bit."""
    K = np.array([90.0, 100.0, 110.0, 95.0])
    vol = np.array([0.2, 0.2, 0.3, 0.25])
    kind = np.array([0, 1, 0, 1])
    arr = ctx.price_american_batch_arrays(100.0, K, 0.05, vol, 1.0, kind, 16, 5000, 42, allow_put=True)
    lst = ctx.price_american_batch([spec_of(qmcg, (100.0, k, 0.05, v, 1.0), int(t)) for k, v, t in zip(K, vol, kind)],
                                   16, 5000, 42, allow_put=True)
    assert np.array_equal(arr, np.array([(r.price, r.std_error) for r in lst]))


def test_random_specs_vs_oracle(ctx, qmcg, oracle_lib):
    """Seeded random contracts (spot, strike, rate incl. r <= 0, vol, maturity, m, n not a multiple
    of the block) through every K2 instantiation the drop-in reaches: calls (pinned to the
    reference algorithm) and opt-in puts (the oracle's mirrored rule), per-path values and price."""
    rng = np.random.default_rng(20261018)
    for t in range(24):
        s = (float(rng.uniform(50, 150)), float(rng.uniform(60, 140)), float(rng.uniform(-0.03, 0.12)),
             float(rng.uniform(0.05, 0.6)), float(rng.uniform(0.1, 3.0)))
        m = int(rng.integers(1, 70))
        n = int(rng.integers(2, 5000))
        seed = int(rng.integers(0, 2**63))
        kind = t % 2
        kw = dict(kind=O.PUT, allow_put=True) if kind else {}
        p, se, vals = oracle_lib.price_american(*s, m, n, seed, want_values=True, **kw)
        v = ctx.path_values(spec_of(qmcg, s, kind), m, n, seed, **({"allow_put": True} if kind else {}))
        assert np.max(np.abs(v - vals) / np.maximum(np.abs(vals), 1e-300)) < 1e-9, (t, s, m, n)
        r = ctx.price_american(spec_of(qmcg, s, kind), m, n, seed, allow_put=bool(kind))
        assert abs(r.price - p) <= PRICE_RTOL * max(p, 1e-12), (t, s, m, n, r.price, p)
        assert abs(r.std_error - se) <= 1e-8 * max(se, 1e-12), (t, s, m, n, r.std_error, se)
