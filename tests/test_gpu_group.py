"""Device groups (qmcg_create_multi): one process pricing over several listed devices.

The group shards the paths as whole pairwise-tree nodes (the reference's pairwise_sum,
proj/src/path_engine.cpp:39-59) and folds the node sums on the host, so its results must be
bit-identical to a single device for any member count -- the GPU analogue of the reference's
lanes-invariance tests (proj/tests/test_american.cpp:140-147, acceptance.cpp:175-207). The
box has one GPU, so the device is listed several times: every member is a full context with
its own stream, tables and scratch, and the sharded table build copies slices between members
with cudaMemcpyPeerAsync exactly as between distinct GPUs (no kernel waits on another).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REF = (100.0, 100.0, 0.05, 0.2, 1.0)


@pytest.fixture(scope="module")
def groups(qmcg):
    gs = {k: qmcg.Context(devices=[0] * k) for k in (2, 3)}
    yield gs
    for g in gs.values():
        g.close()


def _same(a, b):
    return a.price == b.price and a.std_error == b.std_error


@pytest.mark.parametrize("k", [2, 3])
def test_group_price_bit_identical(ctx, qmcg, groups, k):
    g = groups[k]
    assert g.device_count() == k
    for spec, m, n, kw in ((qmcg.OptionSpec(*REF), 64, 1 << 20, {}),
                           (qmcg.OptionSpec(*REF), 33, 100003, {}),
                           (qmcg.OptionSpec(90.0, 100.0, 0.03, 0.3, 0.5, qmcg.OptionKind.Put), 40, 77777,
                            {"allow_put": True}),
                           (qmcg.OptionSpec(*REF), 48, 65536, {"fp32": True}),
                           (qmcg.OptionSpec(100.0, 95.0, -0.02, 0.3, 1.0), 20, 5000, {}),
                           (qmcg.OptionSpec(100.0, 100.0, 0.05, 0.0, 1.0), 10, 3000, {}),
                           (qmcg.OptionSpec(*REF), 5, 130, {}),
                           (qmcg.OptionSpec(*REF), 3, 2, {})):
        one = ctx.price_american(spec, m, n, 42, **kw)
        warm_cold = [g.price_american(spec, m, n, 42, no_cache=True, **kw), g.price_american(spec, m, n, 42, **kw)]
        for r in warm_cold:
            assert _same(r, one), (k, m, n, kw, r, one)


@pytest.mark.parametrize("k", [2, 3])
def test_group_streamed_windows_bit_identical(ctx, qmcg, groups, k):
    """Tables above the members' budget: date windows, each window's dims built sharded."""
    g = groups[k]
    spec = qmcg.OptionSpec(*REF)
    for m, n, fp32 in ((100, 1 << 18, False), (365, 1 << 16, True)):
        one = ctx.price_american(spec, m, n, 42, fp32=fp32)
        ld = -(-n // k // 64) * 64 + 64
        g.set_table_budget(ld * 8 * 24)  # ~3 windows of 8 dates (f64 uniform-table rows)
        try:
            r = g.price_american(spec, m, n, 42, fp32=fp32)
            assert g.last_window_count() > 1
        finally:
            g.set_table_budget(0)
        assert _same(r, one), (k, m, n, fp32)
        g.clear_cache()


def test_group_batch_and_values(ctx, qmcg, groups):
    g = groups[3]
    specs = [qmcg.OptionSpec(100.0, 80 + 40 * i / 7, 0.05, 0.1 + 0.4 * j / 7, 1.0, qmcg.OptionKind((i + j) % 2))
             for i in range(8) for j in range(8)]
    one = ctx.price_american_batch(specs, 32, 1 << 14, 42, allow_put=True)
    grp = g.price_american_batch(specs, 32, 1 << 14, 42, allow_put=True)
    assert all(_same(a, b) for a, b in zip(one, grp))
    v1 = ctx.path_values(qmcg.OptionSpec(*REF), 40, 50001, 42)
    vg = g.path_values(qmcg.OptionSpec(*REF), 40, 50001, 42)
    assert np.array_equal(v1.view(np.uint64), vg.view(np.uint64))


def test_group_timing_hooks(ctx, qmcg, groups):
    g = groups[2]
    spec = qmcg.OptionSpec(*REF)
    k_ms, s_ms, p, se = g.time_device(spec, 32, 1 << 18, 42, 3)
    one = ctx.price_american(spec, 32, 1 << 18, 42)
    assert k_ms > 0 and s_ms >= k_ms and (p, se) == (one.price, one.std_error)
    assert g.time_perm_build(1 << 18, 42, 32) > 0


def test_group_rejects_per_device_calls(qmcg, groups):
    g = groups[2]
    with pytest.raises(RuntimeError):
        g.price_american_nodes(qmcg.OptionSpec(*REF), 8, 4096, 42, 1, 0, 2)
    with pytest.raises(ValueError):  # the reference's own validation still comes first
        g.price_american(qmcg.OptionSpec(*REF, kind=qmcg.OptionKind.Put), 8, 4096, 42)
