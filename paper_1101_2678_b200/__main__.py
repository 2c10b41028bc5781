"""acotsp-compatible CLI on the B200 engine (tools/acotsp.cpp:238-278):

    python -m paper_1101_2678_b200 solve  INSTANCE [--out report.json] [flags]
    python -m paper_1101_2678_b200 bench  INSTANCE... [--deposits a,b] [--reps R] [flags]
    python -m paper_1101_2678_b200 verify INSTANCE [flags]

Flags and defaults follow acotsp.cpp:57-87 (selection nn, deposit
accumulate, theta 64, alpha 1, beta 2, rho 0.5, ants = n, nn 30, iters 100,
seed 1).  Exit codes (acotsp.cpp:44-55): 0 ok, 1 config/other, 2 I/O-class
errors, 3 verify failure.
"""
import argparse
import json
import sys

from . import aco, report

EXIT_OK, EXIT_CONFIG, EXIT_IO, EXIT_VERIFY = 0, 1, 2, 3
SEL = {"roulette": aco.Selection.roulette_full, "nn": aco.Selection.roulette_nn,
       "data-parallel": aco.Selection.data_parallel_tiled}
DEP = {"accumulate": aco.Deposit.accumulate, "scatter-gather": aco.Deposit.scatter_gather,
       "scatter-gather-tiled": aco.Deposit.scatter_gather_tiled,
       "symmetric-reduction": aco.Deposit.symmetric_reduction}


def _common(p):
    p.add_argument("--selection", default="nn")
    p.add_argument("--theta", type=int, default=64)
    p.add_argument("--alpha", type=float, default=1.0)
    p.add_argument("--beta", type=float, default=2.0)
    p.add_argument("--rho", type=float, default=0.5)
    p.add_argument("--ants", type=int, default=0)
    p.add_argument("--nn", type=int, default=30)
    p.add_argument("--iters", type=int, default=100)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--workers", type=int, default=0)
    p.add_argument("--random-start", action="store_true")
    p.add_argument("--device", type=int, default=0)


def _config(a, instance, deposit):
    if a.selection not in SEL:
        raise aco.Error(aco.Errc.config_error, f"unknown selection '{a.selection}' "
                        "(expected roulette, nn, or data-parallel)")
    if deposit not in DEP:
        raise aco.Error(aco.Errc.config_error, f"unknown deposit '{deposit}'")
    return aco.RunConfig(
        params=aco.Parameters(alpha=a.alpha, beta=a.beta, rho=a.rho, m=a.ants, nn=a.nn,
                              iterations=a.iters, seed=a.seed, tile_size=a.theta),
        selection=aco.SelectionStrategy(SEL[a.selection], a.theta),
        deposit=aco.DepositStrategy(DEP[deposit], a.theta), workers=a.workers,
        random_start=a.random_start, instance_path=instance, device=a.device)


def main(argv=None):
    ap = argparse.ArgumentParser(prog="acotsp-b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("solve")
    s.add_argument("instance")
    s.add_argument("--deposit", default="accumulate")
    s.add_argument("--out", default="")
    _common(s)
    b = sub.add_parser("bench")
    b.add_argument("instances", nargs="+")
    b.add_argument("--deposits", default="accumulate")
    b.add_argument("--reps", type=int, default=1)
    b.add_argument("--csv", default="")
    _common(b)
    v = sub.add_parser("verify")
    v.add_argument("instance")
    v.add_argument("--tolerance", type=float, default=1e-9)
    _common(v)
    a = ap.parse_args(argv)
    try:
        if a.cmd == "solve":
            rep = aco.run(_config(a, a.instance, a.deposit))
            if a.out:
                try:
                    with open(a.out, "w") as f:
                        f.write(report.dumps(rep) + "\n")
                except OSError:
                    raise aco.Error(aco.Errc.io_error, "cannot write report: " + a.out) from None
            print(f"instance {rep.instance_name} n={rep.n} m={rep.m} best={rep.best_length}")
            return EXIT_OK
        if a.cmd == "bench":
            out = open(a.csv, "w") if a.csv else sys.stdout
            print(report.bench_csv_header(), file=out)
            for inst in a.instances:
                for dep in a.deposits.split(","):
                    for rep_i in range(a.reps):
                        cfg = _config(a, inst, dep)
                        cfg.params.seed = a.seed + rep_i  # acotsp.cpp:171-173
                        r = aco.run(cfg)
                        for rec in r.per_iteration:
                            print(report.bench_csv_row(r.instance_name, r.n, cfg.selection.variant,
                                                       cfg.deposit.variant, a.theta, rep_i, rec),
                                  file=out)
            return EXIT_OK
        spec = aco.load_instance(a.instance)
        vr = aco.verify_deposit_equivalence(aco.build_problem(spec),
                                            _config(a, a.instance, "accumulate"), a.tolerance)
        for va, vb, d, ok in vr.pairs:
            print(f"{aco.deposit_name(va)} vs {aco.deposit_name(vb)}: max |diff| "
                  f"{d.max_abs_diff:.3e} at ({d.i},{d.j}) {'ok' if ok else 'FAIL'}")
        return EXIT_OK if vr.all_pass else EXIT_VERIFY
    except aco.Error as e:
        print(f"error: {e}", file=sys.stderr)
        io = {aco.Errc.io_error, aco.Errc.missing_field, aco.Errc.unsupported_edge_weight_type,
              aco.Errc.malformed_coord, aco.Errc.dimension_mismatch}
        return EXIT_IO if e.code in io else EXIT_CONFIG


if __name__ == "__main__":
    sys.exit(main())
