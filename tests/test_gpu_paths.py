"""Path-matrix export and batch sweeps on the GPU: the reference's
simulate_batch (proj/src/path_engine.cpp:124-152) and backward_sweep / exercise_point
(proj/src/american.cpp:19-101), with the reference's own test cases
(test_path_engine.cpp:62-91, acceptance criterion 4)."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REF = (100.0, 100.0, 0.05, 0.2, 1.0)


def test_simulate_batch_vs_reference(ctx, qmcg, reference_lib):
    spec = (100.0, 95.0, 0.03, 0.25, 2.0)
    m, n = 5, 20000
    g = ctx.simulate_batch(qmcg.OptionSpec(*spec), m, n, 42)
    r = reference_lib.simulate_batch(*spec, m, n, 42)
    assert g.shape == (n, m + 1) and g.min() > 0.0
    # same normals bit for bit; CUDA exp vs glibc exp differ in the last ulp per step
    assert np.max(np.abs(g - r) / r) < 1e-14
    pm = ctx.simulate_batch(qmcg.OptionSpec(*spec), m, n, 42, point_major=True)
    assert np.array_equal(pm.T, g)


def test_simulate_batch_zero_vol_forward(ctx, qmcg):
    b = ctx.simulate_batch(qmcg.OptionSpec(100.0, 100.0, 0.05, 0.0, 1.0), 1, 1, 7)
    assert b.shape == (1, 2)
    assert b[0, 0] == pytest.approx(100.0 * math.exp(0.05 * 0.5), rel=1e-12)
    assert b[0, 1] == pytest.approx(100.0 * math.exp(0.05), rel=1e-12)


def test_martingale_acceptance_4(ctx, qmcg, oracle_lib):
    """Acceptance criterion 4 (proj/tests/acceptance.cpp:102-115): disc * mean S_T = S0 within 3 se."""
    b = ctx.simulate_batch(qmcg.OptionSpec(*REF), 3, 1 << 20, 42, point_major=True)
    disc = math.exp(-0.05 * 1.0)
    discounted = disc * b[-1]
    mean, se = oracle_lib.reduce_stats(discounted)
    assert abs(mean - 100.0) < 3.0 * se, (mean, se)


def test_simulate_batch_errors(ctx, qmcg):
    with pytest.raises(OverflowError, match="1001"):
        ctx.simulate_batch(qmcg.OptionSpec(*REF), 1000, 1 << 40, 1)
    with pytest.raises(ValueError, match="n_paths must be >= 1"):
        ctx.simulate_batch(qmcg.OptionSpec(*REF), 3, 0, 1)
    with pytest.raises(ValueError, match="s_prev must be > 0"):  # the walk underflows to 0
        ctx.simulate_batch(qmcg.OptionSpec(1e-300, 100.0, 0.05, 30.0, 40.0), 60, 64, 1)


@pytest.mark.parametrize("spec,m,n", [(REF, 20, 4096), ((110.0, 100.0, 0.08, 0.15, 2.0), 64, 8192),
                                      ((100.0, 100.0, 0.0, 0.3, 1.0), 13, 3000)])
def test_sweep_batch(ctx, qmcg, spec, m, n):
    """GPU sweep over the GPU path matrix == host backward_sweep of the same rows (values to the
    cnd FMA ulps, exercise points exactly except at near-ties) == the pricing kernel's values."""
    sp = qmcg.OptionSpec(*spec)
    vals, ex = ctx.sweep_batch(sp, m, n, 42)
    paths = ctx.simulate_batch(sp, m, n, 42)
    host = [qmcg.backward_sweep(paths[p], sp, m) for p in range(n)]
    hv = np.array([h[0][0] for h in host])
    hex_ = np.array([-1 if h[1] is None else h[1] for h in host])
    assert np.max(np.abs(vals - hv) / np.maximum(hv, 1e-300)) < 1e-12
    mismatch = np.nonzero(ex != hex_)[0]  # only where intrinsic and continuation tie to rounding
    assert len(mismatch) <= max(1, n // 1000), mismatch[:10]
    kernel = ctx.path_values(sp, m, n, 42)
    assert np.max(np.abs(vals - kernel) / np.maximum(kernel, 1e-300)) < 1e-9
    assert ((ex >= -1) & (ex <= m)).all()
