"""Machine-readable sequence reports in the reference's schema (SURVEY.md
§8(f) row 4; the reference writes them from its CLI, ``cli.py:35-36`` and
``cli.py:181-244``).

The CLI itself (YAML grids, subcommands) is out of scope; these writers let a
caller that drives ``run_sequence`` / ``SequenceRunner`` on the device emit the
same artifacts the reference's tooling reads:

* ``runs.csv`` - one row per solved system, columns ``CSV_HEADER``;
* ``summary.json`` - per run: averages of iterations / n_c / times and the
  convergence flag, keyed ``"<strategy>|<preconditioner>|<tol>|seed<seed>"``;
* ``<curve>_<tag>.dat`` - "k value" lines for iterations, n_c and time per
  system (plot-ready).

Host-side formatting only; the numbers come from ``SequenceReport`` records.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass
from pathlib import Path

from .recycle import SequenceReport

CSV_HEADER = ("strategy,preconditioner,tol,k,iterations,n_c_before,"
              "n_c_selected,solve_seconds,augmentation_seconds,final_residual")

__all__ = ["CSV_HEADER", "RunResult", "csv_rows", "summarize", "write_report"]


@dataclass
class RunResult:
    """One (strategy, preconditioner, tolerance, seed) run of a sequence."""

    name: str
    preconditioner: str
    tol: float
    seed: int
    report: SequenceReport


def csv_rows(run: RunResult):
    """The run's ``runs.csv`` rows (no header)."""
    out = []
    for rec in run.report.records:
        fields = [run.name, run.preconditioner, format(run.tol, "g"), str(rec.k), str(rec.iterations),
                  str(rec.n_c_before), str(rec.n_c_selected), format(rec.solve_seconds, ".6f"),
                  format(rec.augmentation_seconds, ".6f"), format(rec.final_residual, ".17g")]
        out.append(",".join(fields))
    return out


def _mean(values):
    return float(sum(values) / len(values)) if values else math.nan


def summarize(runs):
    """``summary.json`` content for a list of RunResult."""
    table = {}
    for run in runs:
        recs = run.report.records
        ncs = [r.n_c_before for r in recs]
        table[f"{run.name}|{run.preconditioner}|{run.tol:g}|seed{run.seed}"] = {
            "strategy": run.name,
            "preconditioner": run.preconditioner,
            "tol": run.tol,
            "seed": run.seed,
            "systems": len(recs),
            "avg_iterations": _mean([r.iterations for r in recs]),
            "avg_n_c": _mean(ncs),
            "max_n_c": int(max(ncs)) if ncs else 0,
            "avg_solve_seconds": _mean([r.solve_seconds for r in recs]),
            "avg_augmentation_seconds": _mean([r.augmentation_seconds for r in recs]),
            "all_converged": all(r.converged for r in recs) and not run.report.aborted,
        }
    return table


def _dat(points):
    lines = []
    for k, v in points:
        lines.append(f"{k} {v:.17g}" if isinstance(v, float) else f"{k} {v}")
    return "\n".join(lines) + "\n"


def write_report(out_dir, runs):
    """Write runs.csv, summary.json and the per-run curves; returns the summary."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    rows = [CSV_HEADER]
    for run in runs:
        rows += csv_rows(run)
    (out / "runs.csv").write_text("\n".join(rows) + "\n")
    table = summarize(runs)
    (out / "summary.json").write_text(json.dumps(table, indent=2, sort_keys=True) + "\n")
    for run in runs:
        tag = f"{run.name}_{run.preconditioner}_{run.tol:g}_seed{run.seed}".replace("-", "m")
        recs = run.report.records
        (out / f"iterations_vs_system_{tag}.dat").write_text(_dat([(r.k, r.iterations) for r in recs]))
        (out / f"nc_vs_system_{tag}.dat").write_text(_dat([(r.k, r.n_c_before) for r in recs]))
        (out / f"time_vs_system_{tag}.dat").write_text(
            _dat([(r.k, r.solve_seconds + r.augmentation_seconds) for r in recs]))
    return table
