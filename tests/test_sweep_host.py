"""Per-path sweep diagnostics on the host (no GPU): qmcg_backward_sweep restates the reference's
backward_sweep / sweep_value (proj/src/american.cpp:19-101). The cases are the reference's own
unit tests (proj/tests/test_american.cpp:28-116), plus random paths against the compiled
reference (oracle/_ref) bit for bit, and simulate_batch's validation (test_path_engine.cpp:93-104)."""
import math

import numpy as np
import pytest

import paper_1205_0106_b200 as q

REF = q.OptionSpec(100.0, 100.0, 0.05, 0.2, 1.0)


def dt_of(m, T=1.0):
    return T / (m + 1)


def test_deep_otm_keeps_continuation(reference_lib):
    spec = q.OptionSpec(100.0, 1000.0, 0.05, 0.2, 1.0)
    values, ex = q.backward_sweep([20.0, 25.0], spec, 1)
    assert values.size == 3
    bs_t1 = reference_lib.bs_price(20.0, 1000.0, 0.05, 0.2, dt_of(1))
    assert values[1] == bs_t1
    assert values[0] == bs_t1 * math.exp(-0.05 * dt_of(1))
    assert ex is None and values[2] == 0.0


def test_near_zero_strike():
    spec = q.OptionSpec(100.0, 1e-9, 0.0, 0.2, 1.0)
    values, _ = q.backward_sweep([90.0, 120.0, 80.0, 110.0], spec, 3)
    assert values[3] == pytest.approx(80.0, rel=1e-9)
    assert values[2] == pytest.approx(120.0, rel=1e-9)
    assert values[1] == pytest.approx(120.0, rel=1e-9)
    assert values[0] == pytest.approx(120.0, rel=1e-9)


def test_hand_enumerated_three_points():
    spec = q.OptionSpec(100.0, 95.0, 0.0, 0.3, 1.0)
    path = [108.0, 91.0, 104.0, 97.0]
    value = q.sweep_value(path, spec, 3)
    assert value == pytest.approx(13.0, rel=1e-15)
    values, ex = q.backward_sweep(path, spec, 3)
    assert ex == 1 and values[0] == value


def test_sweep_locality():
    path = np.array([101.0, 96.0, 108.0, 99.0, 103.0])
    bumped = path.copy()
    bumped[1] = 150.0
    base, _ = q.backward_sweep(path, REF, 4)
    moved, _ = q.backward_sweep(bumped, REF, 4)
    assert moved[3] == base[3] and moved[4] == base[4] and moved[5] == base[5]
    assert moved[2] != base[2]


def test_terminal_entry_is_payoff():
    values, _ = q.backward_sweep([104.0, 99.0, 117.5], REF, 2)
    assert values[-1] == 17.5 and (values >= 0).all()


def test_shape_and_put_rejected():
    with pytest.raises(ValueError, match="path length"):
        q.backward_sweep([100.0, 100.0], REF, 2)
    put = q.OptionSpec(100.0, 100.0, 0.05, 0.2, 1.0, kind=q.OptionKind.Put)
    with pytest.raises(ValueError, match="not implemented for puts"):
        q.backward_sweep([100.0, 100.0, 100.0], put, 2)


def test_random_paths_bit_exact_vs_reference(reference_lib):
    rng = np.random.default_rng(3)
    for trial in range(200):
        m = int(rng.integers(1, 40))
        spec = (float(rng.uniform(50, 150)), float(rng.uniform(50, 150)), float(rng.uniform(-0.02, 0.1)),
                float(rng.choice([0.0, rng.uniform(0.05, 0.6)])), float(rng.uniform(0.1, 3.0)))
        path = spec[0] * np.exp(np.cumsum(rng.normal(0, 0.05, m + 1)))
        v_ref, trace_ref, ex_ref = reference_lib.backward_sweep(path, m, *spec)
        values, ex = q.backward_sweep(path, q.OptionSpec(*spec), m)
        assert np.array_equal(values, trace_ref), (trial, values - trace_ref)
        assert values[0] == v_ref and ex == ex_ref


def test_simulate_batch_validation():
    with pytest.raises(OverflowError) as e:
        q.validate_simulation(REF, 1000, 1 << 40)
    assert "bytes" in str(e.value) and "1001" in str(e.value)
    with pytest.raises(ValueError, match="n_paths must be >= 1"):
        q.validate_simulation(REF, 3, 0)
    with pytest.raises(ValueError, match="m must be >= 1"):
        q.validate_simulation(REF, 0, 10)
    q.validate_simulation(REF, 3, 1 << 20)
