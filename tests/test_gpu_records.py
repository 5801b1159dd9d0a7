"""run_benchmark's GPU rows (lanes = -1) in the reference's schema, readable by the reference's own
parse_csv_records next to its CPU rows."""
import pytest

pytestmark = pytest.mark.gpu


def test_run_benchmark_gpu_rows(ctx, qmcg, reference_lib):
    from paper_1205_0106_b200 import records as R
    spec = qmcg.OptionSpec(100.0, 100.0, 0.05, 0.2, 1.0)
    rep = R.run_benchmark(spec, qmcg.Method.AmericanUpperBound, 10, [4096, 1 << 14], 42, ctx=ctx)
    assert not rep.errors and [r.n_paths for r in rep.records] == [4096, 1 << 14]
    for r in rep.records:
        one = ctx.price_american(spec, 10, r.n_paths, 42)
        assert (r.price, r.std_error, r.lanes, r.m) == (one.price, one.std_error, R.GPU_LANES, 10)
        assert r.elapsed_s > 0
    cpu = reference_lib.price_american(100.0, 100.0, 0.05, 0.2, 1.0, 10, 4096, 42, lanes=2)
    rows = [(2, 4096, 10, 2, 4096, 42, cpu[0], cpu[1], cpu[2])]
    text = R.emit_records(rep.records, R.OutputFormat.Csv) + \
        reference_lib.emit_records(rows, 1).split("\n", 1)[1]
    parsed = reference_lib.parse_csv_records(text)
    assert len(parsed) == 3 and parsed[0][3] == -1 and parsed[2][3] == 2
    assert abs(parsed[0][6] - parsed[2][6]) <= 1e-9 * parsed[2][6]  # GPU row vs the reference's CPU row
    eu = R.run_benchmark(spec, qmcg.Method.EuropeanMC, 10, [4096], 42, ctx=ctx)
    assert eu.records[0].m == 0 and eu.records[0].method == qmcg.Method.EuropeanMC
    with pytest.raises(ValueError, match="closed-form"):
        R.run_benchmark(spec, qmcg.Method.ClosedForm, 10, [4096], 42, ctx=ctx)
