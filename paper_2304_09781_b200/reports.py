"""Eval-log and report writers.

* ``write_evals_csv``      per-step anneal log, header ``iter,temp,ged_from_center,f,h,p95_ms,
                           sla_met,accepted,new_best``, one block per chain
* ``write_timeline_csv``   TimelineReport rows
* ``write_summary_json``   TimelineReport summary, fixed key order
* ``write_comparison_csv`` one row per scheme: carbon saved %, accuracy delta %, p95
                           normalised to BASE
* ``compare``              run_trace for several schemes on one trace -> comparison rows

Floats are written with ``repr`` so identical reports serialise byte-identically
(SPEC:622 timeline determinism).
"""

from __future__ import annotations

import csv
import json
from typing import Iterable, Optional, Sequence

import numpy as np

EVAL_FIELDS = ("iter", "temp", "ged_from_center", "f", "h", "p95_ms", "sla_met", "accepted", "new_best")
TIMELINE_FIELDS = ("t", "ci", "scheme", "p95_ms", "sla_met", "accuracy", "gco2_per_request", "cumulative_gco2",
                   "optimizing", "des_p95_ms", "des_sla_met")
COMPARISON_FIELDS = ("scheme", "carbon_saved_pct", "accuracy_delta_pct", "p95_norm_to_base", "total_gco2",
                     "mean_accuracy", "mean_p95_ms", "replans", "candidates_scored", "sla_violation_ticks")


def _cell(v):
    if isinstance(v, (bool, np.bool_)):
        return "1" if v else "0"
    if isinstance(v, (float, np.floating)):
        return repr(float(v))
    if isinstance(v, (int, np.integer)):
        return str(int(v))
    return "" if v is None else str(v)


def write_evals_csv(path: str, log, chains: Optional[Iterable[int]] = None, steps=None) -> int:
    """Write the per-step log of ``clv_anneal`` (LOG_DTYPE [chains, max_steps]).

    ``steps[c]`` (chain results' step counts) bounds the rows of chain c; a ``chain``
    column precedes the SPEC fields when more than one chain is written.  Returns the
    number of rows."""
    log = np.asarray(log)
    if log.ndim == 1:
        log = log[None, :]
    sel = list(range(log.shape[0])) if chains is None else list(chains)
    multi = len(sel) > 1
    rows = 0
    with open(path, "w", newline="\n", encoding="utf-8") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow((("chain",) if multi else ()) + EVAL_FIELDS)
        for c in sel:
            n = log.shape[1] if steps is None else int(steps[c])
            for k in range(n):
                r = log[c, k]
                vals = [r["iter"], r["temp"], r["ged_from_center"], r["f"], r["h"], r["p95_ms"],
                        bool(r["sla_met"]), bool(r["accepted"]), bool(r["new_best"])]
                w.writerow(([c] if multi else []) + [_cell(v) for v in vals])
                rows += 1
    return rows


def write_timeline_csv(path: str, report) -> None:
    with open(path, "w", newline="\n", encoding="utf-8") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(TIMELINE_FIELDS)
        for r in report.rows:
            w.writerow([_cell(r.get(k)) for k in TIMELINE_FIELDS])


def write_summary_json(path: str, report) -> None:
    with open(path, "w", newline="\n", encoding="utf-8") as fh:
        json.dump({k: (float(v) if isinstance(v, np.floating) else v) for k, v in report.summary.items()}, fh,
                  indent=1)
        fh.write("\n")


def comparison_rows(reports: Sequence) -> list[dict]:
    """Paper-style comparison: carbon saved and accuracy delta vs BASE from each
    report's summary, mean p95 normalised to the BASE report's mean p95 (1.0 when no BASE)."""
    base = next((r for r in reports if r.summary.get("scheme") == "base"), None)
    mean_p95 = lambda r: float(np.mean([row["p95_ms"] for row in r.rows])) if r.rows else 0.0
    bp = mean_p95(base) if base is not None else None
    out = []
    for r in reports:
        s = r.summary
        mp = mean_p95(r)
        out.append(dict(scheme=s["scheme"], carbon_saved_pct=s["carbon_saved_vs_base_pct"],
                        accuracy_delta_pct=s["accuracy_delta_vs_base_pct"],
                        p95_norm_to_base=(mp / bp) if bp else 1.0, total_gco2=s["total_gco2"],
                        mean_accuracy=s["mean_accuracy"], mean_p95_ms=mp, replans=s["replans"],
                        candidates_scored=s["candidates_scored"], sla_violation_ticks=s["sla_violation_ticks"]))
    return out


def write_comparison_csv(path: str, rows: Sequence[dict]) -> None:
    with open(path, "w", newline="\n", encoding="utf-8") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(COMPARISON_FIELDS)
        for r in rows:
            w.writerow([_cell(r[k]) for k in COMPARISON_FIELDS])


def write_trace_run(out_dir: str, report, log=None, steps=None) -> None:
    """``trace-run --out DIR`` artefacts: timeline.csv, summary.json, evals.csv."""
    import os
    os.makedirs(out_dir, exist_ok=True)
    write_timeline_csv(os.path.join(out_dir, "timeline.csv"), report)
    write_summary_json(os.path.join(out_dir, "summary.json"), report)
    evals = log if log is not None else getattr(report, "evals_log", None)
    with_steps = steps if steps is not None else getattr(report, "evals_steps", None)
    if evals is not None:
        write_evals_csv(os.path.join(out_dir, "evals.csv"), evals, steps=with_steps)
    else:
        with open(os.path.join(out_dir, "evals.csv"), "w", newline="\n", encoding="utf-8") as fh:
            fh.write(",".join(EVAL_FIELDS) + "\n")


def compare(engine, trace, schemes: Sequence[str], n: int, profile, lam: float = 0.5, seed: int = 0,
            **kw) -> list[dict]:
    """run_trace for each scheme on the same trace and seed -> comparison rows."""
    from .controller import run_trace
    reps = [run_trace(engine, trace, s, n, profile, lam, seed=seed, **kw) for s in schemes]
    return comparison_rows(reps)
