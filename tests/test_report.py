"""RunReport JSON / bench CSV in the reference's formats (report.hpp), pinned
against the reference's own report.hpp compiled into oracle/_ref."""
import json
import math

import numpy as np
import pytest


@pytest.fixture(scope="module")
def report():
    from paper_1101_2678_b200 import report as _r

    return _r


def test_format_double_matches_to_chars(reference, report):
    if not hasattr(reference.lib, "ref_format_double"):
        pytest.skip("reference harness built without report.hpp")
    rng = np.random.default_rng(5)
    vals = [0.0, 1.0, -2.0, 100.0, 1e16, 1e15, 123456789012345680.0, 0.1, 0.5, 1.5e-5, 3.25,
            1e-300, 2.5e300, 20000.0, 312.5, 389034.21717171714, 0.0015039764225110329,
            1e21, 1e22, 12345678.9, 1234567890123.0]
    vals += list(rng.random(200) * 10.0 ** rng.integers(-12, 20, 200))
    vals += [float(x) for x in rng.integers(0, 10**12, 50)]
    for v in vals:
        assert report.format_double(v) == reference.format_double(v), v


def test_csv_header(report):
    assert report.bench_csv_header().split(",")[-1] == "schema_version"


@pytest.mark.gpu
@pytest.mark.parametrize("deposit", [1, 3])
def test_report_json_and_csv_match_reference(report, deposit):
    """tests/golden/report_synth198_dep*.{json,csv} were written by the
    reference's own report.hpp (oracle/ref_report_main.cpp)."""
    import os

    from paper_1101_2678_b200 import aco
    from pyoracle import synth_coords

    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    ref = json.load(open(os.path.join(here, f"report_synth198_dep{deposit}.json")))
    ref_csv = open(os.path.join(here, f"report_synth198_dep{deposit}.csv")).read()
    n, iters = 198, 6
    xs, ys = synth_coords(n)
    spec = aco.InstanceSpec("synth198", n, aco.EdgeWeightType.euc_2d, xs, ys)
    cfg = aco.RunConfig(params=aco.Parameters(iterations=iters, seed=1), workers=1,
                        selection=aco.SelectionStrategy(aco.Selection.roulette_full),
                        deposit=aco.DepositStrategy(aco.Deposit(deposit)))
    with aco.Engine(aco.build_problem(spec), cfg) as eng:
        rep = eng.run()
    rep.instance_name = "synth198"
    mine = report.report_to_json(rep)
    for r in mine["per_iteration"] + ref["per_iteration"]:
        r.pop("construct_ms"), r.pop("update_ms")  # wall-clock fields
    assert mine == ref
    rows_m = [report.bench_csv_row("synth198", n, aco.Selection.roulette_full,
                                   aco.Deposit(deposit), 64, 0, r).split(",")
              for r in rep.per_iteration]
    rows_r = [l.split(",") for l in ref_csv.strip().splitlines()[1:]]
    assert len(rows_m) == len(rows_r)
    for a, b in zip(rows_m, rows_r):
        assert a[:7] + a[9:] == b[:7] + b[9:]  # all but the two timing columns
