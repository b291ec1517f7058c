"""Scenario-grid results as CSV, in the reference's file format (suite.py).

The reference's suite (suite.py:23-54 column contract, 137-172 rows and
writer) writes one ``data`` row per (scenario, seed) cell and one
``summary`` row per scenario: ensemble mean in the metric columns, sample
standard deviation (0 for one seed) in the ``*_std`` columns; rows sorted by
scenario id then seed, integers as ``str`` and floats as ``repr`` so equal
runs give byte-identical files.  ``extended=True`` appends the measured-run
columns this package adds (clock, device, decode tokens/s); without it the
file is byte-identical to the reference's for the same cells
(tests/test_results_csv.py against tests/golden/suite.csv).
"""

from __future__ import annotations

import csv
import math
from dataclasses import dataclass, field

from .arrivals import FixedLength
from .metrics import Metrics, compute_metrics
from .scenario import ConstantArrival, Scenario, run_scenario

# (column, Metrics attribute) -- the metric block of the reference's columns
_METRICS = (
    ("makespan_ms", "makespan_ms"),
    ("mean_latency_ms", "mean_latency_ms"),
    ("p50_latency_ms", "p50_latency_ms"),
    ("p99_latency_ms", "p99_latency_ms"),
    ("total_iterations", "total_stream_iterations"),
    ("overlap", "overlap_percent"),
    ("bytes_shuffled", "bytes_shuffled"),
    ("shuffle_count", "shuffle_count"),
)
_IDENTITY = ("scenario_id", "discipline", "n_requests", "arrival", "interval_ms", "lengths", "length_lo",
             "length_hi", "max_output_length", "batch_size", "tp_size", "placement")
COLUMNS = (["row_type", _IDENTITY[0], _IDENTITY[1], "seed"] + list(_IDENTITY[2:]) + [c for c, _ in _METRICS]
           + [f"{c}_std" for c, _ in _METRICS])
EXTENDED_COLUMNS = COLUMNS + ["clock", "device", "decode_tokens_per_s"]


@dataclass(frozen=True)
class CellResult:
    scenario: Scenario
    seed: int
    metrics: Metrics
    # measured runs (extended columns): clock, device name, decode tokens/s
    extra: dict = field(default_factory=dict)


def _text(v) -> str:
    return str(v) if isinstance(v, int) else repr(v)


def _identity(s: Scenario) -> dict:
    constant = isinstance(s.arrival, ConstantArrival)
    fixed = isinstance(s.lengths, FixedLength)
    lo, hi = (s.lengths.tokens, s.lengths.tokens) if fixed else (s.lengths.lo, s.lengths.hi)
    vals = {
        "scenario_id": s.scenario_id,
        "discipline": s.discipline.value,
        "n_requests": s.n_requests,
        "arrival": "constant" if constant else "poisson",
        "interval_ms": repr(float(s.arrival.interval_ms if constant else s.arrival.mean_interval_ms)),
        "lengths": "fixed" if fixed else "uniform",
        "length_lo": lo,
        "length_hi": hi,
        "max_output_length": s.max_output_length,
        "batch_size": s.batch_size,
        "tp_size": s.tp.tp_size,
        "placement": s.tp.placement.value,
    }
    return {k: v if isinstance(v, str) else _text(v) for k, v in vals.items()}


def run_cells(scenarios, *, executor_for=None, clock: str = "cost", device: str = "") -> list[CellResult]:
    """Every (scenario, seed) cell in (scenario id, seed) order.  With
    ``executor_for(scenario, seed)`` each cell runs through a device executor
    on ``clock``; the extended columns then carry the clock, ``device`` and the
    decode tokens/s over the makespan."""
    out = []
    for sc in sorted(scenarios, key=lambda x: x.scenario_id):
        for seed in sc.seeds:
            ex = executor_for(sc, seed) if executor_for else None
            trace = run_scenario(sc, seed, executor=ex, clock=clock if ex is not None else "cost")
            m = compute_metrics(trace, sc.n_requests)
            extra = {}
            if ex is not None:
                toks = sum(len(t) for t in ex.tokens().values()) if hasattr(ex, "tokens") else 0
                extra = {"clock": clock, "device": device,
                         "decode_tokens_per_s": repr(1e3 * toks / m.makespan_ms if m.makespan_ms else 0.0)}
            out.append(CellResult(sc, seed, m, extra))
    return out


def result_rows(results: list[CellResult], extended: bool = False) -> list[dict]:
    cols = EXTENDED_COLUMNS if extended else COLUMNS
    groups: dict[str, list[CellResult]] = {}
    for c in results:
        groups.setdefault(c.scenario.scenario_id, []).append(c)
    rows = []
    for sid in sorted(groups):
        cells = sorted(groups[sid], key=lambda c: c.seed)
        ident = _identity(cells[0].scenario)
        samples = {c: [] for c, _ in _METRICS}
        for cell in cells:
            row = dict.fromkeys(cols, "")
            row.update(ident, row_type="data", seed=str(cell.seed))
            for col, attr in _METRICS:
                v = getattr(cell.metrics, attr)
                row[col] = _text(v)
                samples[col].append(float(v))
            if extended:
                row.update(cell.extra)
            rows.append(row)
        summary = dict.fromkeys(cols, "")
        summary.update(ident, row_type="summary")
        for col, vals in samples.items():
            mean = sum(vals) / len(vals)
            sd = math.sqrt(sum((v - mean) ** 2 for v in vals) / (len(vals) - 1)) if len(vals) > 1 else 0.0
            summary[col] = _text(mean)
            summary[col + "_std"] = _text(sd)
        rows.append(summary)
    return rows


def write_csv(rows: list[dict], path, extended: bool = False) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=EXTENDED_COLUMNS if extended else COLUMNS, lineterminator="\n")
        w.writeheader()
        w.writerows(rows)


def run_suite(scenarios, out_path) -> list[CellResult]:
    """Run every cell on the cost clock and write the reference's CSV."""
    cells = run_cells(scenarios)
    write_csv(result_rows(cells), out_path)
    return cells


def format_trace(trace) -> str:
    """The trace as one TSV text (the reference's suite helper)."""
    return "\n".join(trace.format_lines()) + "\n"
