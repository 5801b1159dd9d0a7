"""Streamed permutation tables (date windows) == resident tables, bit for bit.

When the tables exceed the memory budget (config 5: 2^28 paths x 365 dates =
392 GB), K1 builds one window of dates at a time and K2 carries each path's
walk state (V, last record, dominance accumulator, pending record, best) in HBM
between windows. The windows change nothing arithmetically, so the per-path
values must equal the resident-table values exactly."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REF = (100.0, 100.0, 0.05, 0.2, 1.0)


def row_bytes(cols):
    return (cols + 63) // 64 * 64 * 8  # the uniform table: f64 entries


CASES = [  # (spec, kind, m, n, fp32)
    (REF, 0, 37, 5000, False),
    (REF, 1, 50, 4096, False),
    ((100.0, 110.0, -0.02, 0.3, 1.0), 0, 33, 3000, False),   # r < 0 path
    ((90.0, 100.0, 0.03, 0.3, 0.5), 1, 41, 2048, True),      # FP32 walk
    ((100.0, 100.0, 0.05, 3.0, 40.0), 0, 29, 2000, False),   # per-date range checks (SLOW kernel)
    ((100.0, 100.0, 0.05, 0.0, 1.0), 0, 20, 1000, False),    # deterministic
]


@pytest.mark.parametrize("s,kind,m,n,fp32", CASES)
@pytest.mark.parametrize("window", [8, 16])
def test_streamed_equals_resident(ctx, qmcg, s, kind, m, n, fp32, window):
    sp = qmcg.OptionSpec(*s, kind=qmcg.OptionKind(kind))
    put = kind == 1
    ctx.set_table_budget(0)
    ctx.clear_cache()
    v_res = ctx.path_values(sp, m, n, 7, allow_put=put, fp32=fp32)
    r_res = ctx.price_american(sp, m, n, 7, allow_put=put, fp32=fp32)
    assert ctx.last_window_count() == 1
    ctx.clear_cache()
    ctx.set_table_budget(window * row_bytes(n))
    try:
        v_str = ctx.path_values(sp, m, n, 7, allow_put=put, fp32=fp32)
        r_str = ctx.price_american(sp, m, n, 7, allow_put=put, fp32=fp32)
        if s[3] > 0:
            assert ctx.last_window_count() == -(-m // window)
    finally:
        ctx.set_table_budget(0)
        ctx.clear_cache()
    assert np.array_equal(v_res, v_str)
    assert r_res.price == r_str.price and r_res.std_error == r_str.std_error


def test_streamed_node_ranges(ctx, qmcg):
    """Node (path-slice) pricing with streamed tables: the multi-GPU decomposition still combines
    to the single-call result bit for bit."""
    sp = qmcg.OptionSpec(*REF)
    n, m, depth = 6000, 40, 2
    full = ctx.price_american(sp, m, n, 11)
    ctx.set_table_budget(8 * row_bytes(n // 4 + 64))
    try:
        sums = np.concatenate([ctx.price_american_node(sp, m, n, 11, depth, k) for k in range(4)])
        assert ctx.last_window_count() == 5
    finally:
        ctx.set_table_budget(0)
        ctx.clear_cache()
    price, se = qmcg.combine_nodes(n, depth, sums)
    assert price == full.price and se == full.std_error
