"""GPU parity of the roulette relay (k_construct_roulette_relay): when m is a
little above a multiple of the SM count, the leftover ants are built in
segments by several warps that hand the tabu set and current city over
through global memory.  Tours must stay bit-exact with the oracle
(construction.hpp:42-68, :181-201), including the tour stream into mapped
host memory and random start cities."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def aco():
    from paper_1101_2678_b200 import aco as _aco

    return _aco


def sms():
    import torch

    return torch.cuda.get_device_properties(0).multi_processor_count


def engine(aco, n, m, deposit=3, random_start=False, seed=1):
    prob = aco.build_problem(aco.synthetic_instance(n))
    cfg = aco.RunConfig(params=aco.Parameters(m=m, seed=seed),
                        selection=aco.SelectionStrategy(aco.Selection.roulette_full),
                        deposit=aco.DepositStrategy(aco.Deposit(deposit)),
                        random_start=random_start)
    return prob, aco.Engine(prob, cfg)


# the relay runs at q a multiple of 4, q >= 8 (aco_gpu.cu: where the leftover
# warp would create a new busiest SM sub-partition)
@pytest.mark.parametrize("n,q,extra,random_start", [(600, 8, 5, False), (1200, 8, 3, True), (700, 8, 1, False),
                                                     (200, 8, 3, False), (300, 12, 5, True)])
def test_relay_multi_iteration_bit_exact(aco, oracle, n, q, extra, random_start):
    """q = 12 warps per SM also forms the tour lengths, 1/C_k and the gather's
    succ/pred in the relay kernel's fused tail (checked through tau)."""
    m = q * sms() + extra
    prob, eng = engine(aco, n, m, random_start=random_start)
    with eng:
        tau = np.full((n, n), eng.tau0)
        for it in range(2):
            ch = oracle.choice(prob.dist, tau)
            eng.run_iteration()
            assert "relay:" in eng.describe()
            t_ref, l_ref, _ = oracle.construct(prob.dist, ch, 1, it, 0, m, random_start=random_start)
            t, l = eng.ants()
            assert np.array_equal(t, t_ref), f"iteration {it}"
            assert np.array_equal(l, l_ref)
            tau = oracle.update(tau, t_ref, l_ref, 0.5, 1)
            assert np.array_equal(eng.pheromone(), tau)


def test_relay_streams_tours_to_pinned_host_buffer(aco):
    import torch

    n = 900
    m = 8 * sms() + 7
    prob, eng = engine(aco, n, m, deposit=0)
    with eng:
        tb = torch.empty((m, n + 1), dtype=torch.int32, pin_memory=True).numpy()
        lb = torch.empty(m, dtype=torch.int64, pin_memory=True).numpy()
        for _ in range(2):
            tb[:] = -7
            eng.run_iteration(tours_out=tb, lengths_out=lb)
            d = eng.describe()
            assert "streams_tours_to_host" in d and "relay:" in d
            t, l = eng.ants()
            assert np.array_equal(tb, t)
            assert np.array_equal(lb, l)


def test_relay_matches_plain_launch(aco, tmp_path):
    """The relay and the plain one-warp-per-ant launch (ACO_RELAY=0, read at
    library load, so in a subprocess) build identical colonies."""
    import subprocess
    import sys

    code = (
        "import sys, numpy as np\n"
        "sys.path.insert(0, %r)\n"
        "from paper_1101_2678_b200 import aco\n"
        "prob = aco.build_problem(aco.synthetic_instance(2392))\n"
        "cfg = aco.RunConfig(params=aco.Parameters(m=0, seed=3),"
        " selection=aco.SelectionStrategy(aco.Selection.roulette_full),"
        " deposit=aco.DepositStrategy(aco.Deposit.scatter_gather))\n"
        "with aco.Engine(prob, cfg) as e:\n"
        "    for _ in range(2): e.run_iteration()\n"
        "    t, l = e.ants()\n"
        "    np.save(sys.argv[1], t); print(e.describe())\n"
    )
    import os

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for relay in ("0", "4"):
        env = dict(os.environ, ACO_RELAY=relay)
        f = str(tmp_path / f"t{relay}.npy")
        r = subprocess.run([sys.executable, "-c", code % root, f], env=env, capture_output=True,
                           text=True, check=True)
        outs.append((np.load(f), r.stdout))
    if sms() == 148:
        assert "relay:" in outs[1][1] and "relay:" not in outs[0][1]
    assert np.array_equal(outs[0][0], outs[1][0])
