"""Benchmark records in the reference's schema.

Mirrors proj/include/qmc/bench.hpp:17-71 and proj/src/bench.cpp:111-330:
BenchmarkRecord, the CSV header, emit_records (table / CSV at 17 significant
digits / JSON with the same field names), emit_results, parse_csv_records,
to_record / to_records, and run_benchmark's timing method (one untimed
warm-up, median of 3 wall-clock repetitions around the pricing call). GPU rows
use lanes = -1 (the reference's lanes >= 1 are its thread counts and 0 its
serial runner), so they sit next to the reference's CPU rows in one file and
parse with its own parse_csv_records.
"""
from __future__ import annotations

import dataclasses
import enum
import io
import json
import sys
import time
from typing import Iterable, List, Optional, Sequence

from . import qmcg

CSV_HEADER = "method,n_paths,m,lanes,chunk,seed,price,std_error,elapsed_s"
GPU_LANES = -1

_METHOD_NAMES = {qmcg.Method.ClosedForm: "closed-form", qmcg.Method.EuropeanMC: "european-mc",
                 qmcg.Method.AmericanUpperBound: "american-ub"}
_METHOD_BY_NAME = {v: k for k, v in _METHOD_NAMES.items()}


class OutputFormat(enum.IntEnum):
    Table = 0
    Csv = 1
    Json = 2


@dataclasses.dataclass
class BenchmarkRecord:
    """reference BenchmarkRecord (bench.hpp:17-27)."""
    method: qmcg.Method = qmcg.Method.EuropeanMC
    n_paths: int = 0
    m: int = 0
    lanes: int = 1
    chunk: int = 4096
    seed: int = 0
    price: float = 0.0
    std_error: float = 0.0
    elapsed_s: float = 0.0


def method_name(method) -> str:
    return _METHOD_NAMES[qmcg.Method(method)]


def method_from_name(name: str) -> qmcg.Method:
    if name not in _METHOD_BY_NAME:
        raise ValueError(f"unknown method '{name}'")
    return _METHOD_BY_NAME[name]


def _g(v: float, prec: int) -> str:
    return "%.*g" % (prec, v)


def emit_records(records: Sequence[BenchmarkRecord], fmt: OutputFormat) -> str:
    """emit_records (bench.cpp:203-283), returned as text."""
    if not records:
        raise ValueError("emit_records: records must be non-empty")
    out = io.StringIO()
    if fmt == OutputFormat.Csv:
        out.write(CSV_HEADER + "\n")
        for r in records:
            out.write(f"{method_name(r.method)},{r.n_paths},{r.m},{r.lanes},{r.chunk},{r.seed},"
                      f"{_g(r.price, 17)},{_g(r.std_error, 17)},{_g(r.elapsed_s, 17)}\n")
    elif fmt == OutputFormat.Json:
        # nlohmann::json objects are key-sorted; dump(2) = 2-space indentation
        rows = [{"method": method_name(r.method), "n_paths": r.n_paths, "m": r.m, "lanes": r.lanes,
                 "chunk": r.chunk, "seed": r.seed, "price": r.price, "std_error": r.std_error,
                 "elapsed_s": r.elapsed_s} for r in records]
        out.write(json.dumps(rows, indent=2, sort_keys=True) + "\n")
    else:
        out.write(f"{'method':<13}{'n_paths':>10}{'m':>5}{'lanes':>7}{'chunk':>7}{'seed':>12}"
                  f"{'price':>16}{'std_error':>13}{'elapsed_s':>12}\n")
        for r in records:
            out.write(f"{method_name(r.method):<13}{r.n_paths:>10}{r.m:>5}{r.lanes:>7}{r.chunk:>7}{r.seed:>12}"
                      f"{_g(r.price, 10):>16}{_g(r.std_error, 4):>13}{_g(r.elapsed_s, 4):>12}\n")
    return out.getvalue()


def emit_results(records: Sequence[BenchmarkRecord], fmt: OutputFormat, out_path: str = "") -> None:
    """emit_results (bench.cpp:285-297): stdout when out_path is empty or '-'."""
    text = emit_records(records, fmt)
    if not out_path or out_path == "-":
        sys.stdout.write(text)
        return
    try:
        with open(out_path, "w", newline="") as f:
            f.write(text)
    except OSError:
        raise RuntimeError(f"emit_results: cannot open '{out_path}' for writing") from None


def parse_csv_records(text: str) -> List[BenchmarkRecord]:
    """parse_csv_records (bench.cpp:299-330)."""
    lines = text.split("\n")
    if not text or (len(lines) == 1 and not lines[0]):
        raise RuntimeError("parse_csv_records: empty input")
    header = lines[0].rstrip("\r")
    if header != CSV_HEADER:
        raise RuntimeError(f"parse_csv_records: unrecognized header '{header}'")
    out = []
    for line in lines[1:]:
        line = line.rstrip("\r")
        if not line:
            continue
        f = line.split(",")
        if len(f) != 9:
            raise RuntimeError(f"parse_csv_records: expected 9 fields, got line '{line}'")
        out.append(BenchmarkRecord(method_from_name(f[0]), int(f[1]), int(f[2]), int(f[3]), int(f[4]), int(f[5]),
                                   float(f[6]), float(f[7]), float(f[8])))
    return out


def to_record(result: "qmcg.PricingResult", m: int, lanes: int, chunk: int) -> BenchmarkRecord:
    """to_record (bench.cpp:185-199)."""
    return BenchmarkRecord(result.method, result.n_paths,
                           m if result.method == qmcg.Method.AmericanUpperBound else 0, lanes, chunk, result.seed,
                           result.price, result.std_error, max(result.elapsed_s, 1e-9))


def to_records(curve: Iterable, n_paths: int, lanes: int, chunk: int, seed: int) -> List[BenchmarkRecord]:
    """to_records (bench.cpp:201-219) for a convergence curve."""
    return [BenchmarkRecord(qmcg.Method.AmericanUpperBound, n_paths, p.m, lanes, chunk, seed, p.price, p.std_error,
                            max(p.elapsed_s, 1e-9)) for p in curve]


@dataclasses.dataclass
class BenchmarkReport:
    records: List[BenchmarkRecord]
    errors: List[str]


def run_benchmark(spec: "qmcg.OptionSpec", method: "qmcg.Method", m: int, path_counts: Sequence[int], seed: int,
                  chunk: int = 4096, ctx: Optional["qmcg.Context"] = None) -> BenchmarkReport:
    """run_benchmark (bench.cpp:111-183) on the GPU: one GPU row (lanes = -1) per path count, timed
    like the reference (untimed warm-up, then the median of 3 wall-clock repetitions of the call,
    which includes the host copies of the result). Failures are recorded, not raised."""
    method = qmcg.Method(method)
    if method == qmcg.Method.ClosedForm:
        raise ValueError("run_benchmark: closed-form has no path sweep; use european-mc or american-ub")
    if not path_counts:
        raise ValueError("run_benchmark: path_counts must be non-empty")
    ctx = ctx or qmcg.default_context()
    report = BenchmarkReport([], [])
    for n in path_counts:
        def run():
            if method == qmcg.Method.EuropeanMC:
                return ctx.mc_european_price(spec, n, seed)
            return ctx.price_american(spec, m, n, seed)
        try:
            run()
            times, res = [], None
            for _ in range(3):
                t0 = time.perf_counter()
                res = run()
                times.append(time.perf_counter() - t0)
            rec = to_record(res, m, GPU_LANES, chunk)
            rec.elapsed_s = max(sorted(times)[1], 1e-9)
            report.records.append(rec)
        except Exception as e:  # noqa: BLE001 -- the reference records every failure
            report.errors.append(f"bench configuration n_paths={n} lanes={GPU_LANES} failed: {e}")
    return report
