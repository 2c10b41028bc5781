"""RunReport JSON (schema v1) and bench CSV rows, in the reference's exact
formats (proj/include/aco/report.hpp:13-86), so acotsp-style tooling can
consume the B200 engine's output unchanged.

    report_to_json(report)        -> dict  (json.dumps(..., indent=2) ~ dump(2))
    bench_csv_header()            -> str   (report.hpp:72-75)
    bench_csv_row(instance, n, selection, deposit, theta, rep, record) -> str
"""
from __future__ import annotations

import json
import math

from .aco import Deposit, IterationRecord, RunReport, Selection, deposit_name, selection_name

SCHEMA_VERSION = 1  # report.hpp:13


def format_double(v: float) -> str:
    """std::to_chars(double) (report.hpp:16-21): the shortest round-trip
    digits, printed in fixed or scientific notation — whichever is shorter,
    fixed on ties; integral values print without a decimal point."""
    if math.isnan(v):
        return "nan" if math.copysign(1.0, v) > 0 else "-nan"
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    r = repr(float(v))
    sign = "-" if r.startswith("-") else ""
    r = r.lstrip("-")
    if "e" in r:
        mant, exp = r.split("e")
        exp = int(exp)
    else:
        mant, exp = r, 0
    if "." in mant:
        ip, fp = mant.split(".")
    else:
        ip, fp = mant, ""
    digits = (ip + fp).lstrip("0")
    # decimal exponent of the first significant digit
    if ip.strip("0"):
        point = len(ip.lstrip("0")) + exp
    else:
        lead = len(fp) - len(fp.lstrip("0"))
        point = -lead + exp
    digits = digits.rstrip("0") or "0"
    if digits == "0":
        return sign + "0"
    nd = len(digits)
    # fixed form
    if point >= nd:  # integral: fixed notation prints the exact integer digits
        fixed = str(int(abs(float(v))))
    elif point > 0:
        fixed = digits[:point] + "." + digits[point:]
    else:
        fixed = "0." + "0" * (-point) + digits
    # scientific form d.ddde[+-]XX (at least two exponent digits)
    e = point - 1
    sci = digits[0] + ("." + digits[1:] if nd > 1 else "") + "e" + ("-" if e < 0 else "+") + \
        f"{abs(e):02d}"
    return sign + (fixed if len(fixed) <= len(sci) else sci)


def ledger_to_json(ledger) -> dict:  # report.hpp:23-30
    return {"global_loads": ledger.global_loads, "global_stores": ledger.global_stores,
            "shared_loads": ledger.shared_loads, "atomic_ops": ledger.atomic_ops}


def report_to_json(report: RunReport) -> dict:  # report.hpp:32-67
    cfg = report.config
    return {
        "schema_version": SCHEMA_VERSION,
        "instance": report.instance_name,
        "n": report.n,
        "m": report.m,
        "seed": report.seed,
        "config": {
            "alpha": cfg.params.alpha, "beta": cfg.params.beta, "rho": cfg.params.rho,
            "nn": cfg.params.nn, "iters": cfg.params.iterations, "theta": cfg.params.tile_size,
            "workers": cfg.workers, "selection": selection_name(cfg.selection.variant),
            "deposit": deposit_name(cfg.deposit.variant), "random_start": bool(cfg.random_start),
        },
        "best_length": int(report.best_length),
        "best_tour": [int(c) for c in report.best_tour],
        "per_iteration": [
            {"iteration": r.iteration, "best_len": int(r.best_length), "mean_len": r.mean_length,
             "construct_ms": r.construct_ms, "update_ms": r.update_ms,
             "ledger": ledger_to_json(r.deposit_ledger)}
            for r in report.per_iteration],
    }


def dumps(report: RunReport) -> str:
    return json.dumps(report_to_json(report), indent=2)


def bench_csv_header() -> str:  # report.hpp:72-75
    return ("instance,n,selection,deposit,theta,rep,iter,construct_ms,update_ms,"
            "best_len,global_loads,atomic_ops,schema_version")


def bench_csv_row(instance: str, n: int, selection: Selection, deposit: Deposit, theta: int,
                  rep: int, rec: IterationRecord) -> str:  # report.hpp:77-86
    return ",".join([instance, str(n), selection_name(selection), deposit_name(deposit),
                     str(theta), str(rep), str(rec.iteration), format_double(rec.construct_ms),
                     format_double(rec.update_ms), str(int(rec.best_length)),
                     format_double(rec.deposit_ledger.global_loads),
                     format_double(rec.deposit_ledger.atomic_ops), str(SCHEMA_VERSION)])
