"""Benchmark records in the reference's schema: our emitter's table / CSV /
JSON text is byte-identical to the reference's emit_records (proj/src/bench.cpp:203-283,
compiled into oracle/_ref), both parsers read each other's CSV losslessly, and the parse errors
match. GPU rows carry lanes = -1."""
import math

import numpy as np
import pytest

import paper_1205_0106_b200 as q
from paper_1205_0106_b200 import records as R


def rand_records(seed, k=40):
    rng = np.random.default_rng(seed)
    out = []
    specials = [0.0, 1e-9, 1e-300, 5e-324, 1.0, 13.0, 1e20, 1.5e-7, 123456789.125, 2.0 ** 60, math.pi]
    for i in range(k):
        meth = q.Method(int(rng.integers(0, 3)))
        vals = [float(rng.choice(specials)) if rng.random() < 0.3 else float(rng.lognormal(0, 5)) for _ in range(3)]
        out.append(R.BenchmarkRecord(meth, int(rng.integers(1, 1 << 40)), int(rng.integers(0, 1000)),
                                     int(rng.choice([-1, 0, 1, 8, 64])), int(rng.integers(1, 1 << 20)),
                                     int(rng.integers(0, 2**63 - 1)) * 2 + int(rng.integers(0, 2)), *vals))
    return out


def as_tuples(recs):
    return [(int(r.method), r.n_paths, r.m, r.lanes, r.chunk, r.seed, r.price, r.std_error, r.elapsed_s)
            for r in recs]


@pytest.mark.parametrize("fmt", [R.OutputFormat.Table, R.OutputFormat.Csv, R.OutputFormat.Json])
def test_emit_matches_reference(reference_lib, fmt):
    for seed in range(5):
        recs = rand_records(seed)
        assert R.emit_records(recs, fmt) == reference_lib.emit_records(as_tuples(recs), int(fmt))


def test_csv_round_trip_both_ways(reference_lib):
    recs = rand_records(11)
    text = R.emit_records(recs, R.OutputFormat.Csv)
    theirs = reference_lib.parse_csv_records(text)
    assert theirs == as_tuples(recs)  # lossless: every double round-trips exactly
    ref_text = reference_lib.emit_records(as_tuples(recs), 1)
    assert as_tuples(R.parse_csv_records(ref_text)) == as_tuples(recs)


def test_parse_errors(reference_lib):
    import oracle
    for text in ("", "a,b,c\n", R.CSV_HEADER + "\namerican-ub,1,2,3\n"):
        with pytest.raises(RuntimeError) as ours:
            R.parse_csv_records(text)
        with pytest.raises(oracle.OracleError) as theirs:
            reference_lib.parse_csv_records(text)
        assert str(ours.value) == str(theirs.value)
    with pytest.raises(ValueError, match="records must be non-empty"):
        R.emit_records([], R.OutputFormat.Csv)


def test_to_records_and_emit_results(tmp_path):
    from types import SimpleNamespace
    curve = [SimpleNamespace(m=m, price=10.0 + m, std_error=0.01, elapsed_s=0.0) for m in (1, 5, 10)]
    recs = R.to_records(curve, 1 << 18, R.GPU_LANES, 4096, 42)
    assert [r.m for r in recs] == [1, 5, 10] and all(r.elapsed_s == 1e-9 for r in recs)
    recs = rand_records(3, 4)
    path = tmp_path / "out.csv"
    R.emit_results(recs, R.OutputFormat.Csv, str(path))
    assert as_tuples(R.parse_csv_records(path.read_text())) == as_tuples(recs)
    with pytest.raises(RuntimeError, match="cannot open"):
        R.emit_results(recs, R.OutputFormat.Csv, str(tmp_path / "missing" / "x.csv"))
