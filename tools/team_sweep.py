"""Construction kernel time vs warps per ant (ACO_TEAM) and colony size."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_1101_2678_b200 import aco

    cases = [(198, 198), (1002, 1002), (2392, 299), (2392, 598), (2392, 1196), (2392, 2392)]
    if len(sys.argv) > 1:
        cases = [tuple(map(int, c.split("x"))) for c in sys.argv[1].split(",")]
    for n, m in cases:
        prob = aco.build_problem(aco.synthetic_instance(n))
        for K in ("1", "2", "4", "8"):
            os.environ["ACO_TEAM"] = K
            cfg = aco.RunConfig(params=aco.Parameters(m=m, seed=1),
                                selection=aco.SelectionStrategy(aco.Selection.roulette_full),
                                deposit=aco.DepositStrategy(aco.Deposit.accumulate))
            try:
                eng = aco.Engine(prob, cfg)
            except Exception as e:  # noqa: BLE001
                print(json.dumps({"n": n, "m": m, "K": K, "error": str(e)}))
                continue
            ks = []
            for i in range(6):
                r = eng.run_iteration()
                if i >= 2:
                    ks.append(r.construct_kernel_ms)
            print(json.dumps({"n": n, "m": m, "K": K, "kernel_ms": round(statistics.median(ks), 4),
                              "fb": r.fallbacks, "desc": eng.describe()}), flush=True)
            eng.close()


if __name__ == "__main__":
    main()
