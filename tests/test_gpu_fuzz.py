"""Deterministic fuzz of the iteration against the oracle: instance sizes on
and around every streamed-layout boundary (lanes x vectors per lane), small
and odd colony sizes, every selection rule, both deposits and both weight
streams.  Tours and lengths must be bit-exact; the gather tau too."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# 32 lanes x 4 floats x NV in {2,4,8,12,16,19,20} -> 256 .. 2560 cities; the
# fp64 stream's 2 doubles per vector halves them; beyond 2560: 8-round layout
BOUNDARY_N = [31, 32, 33, 255, 256, 257, 511, 512, 513, 1023, 1024, 1025, 1279, 1280, 1281,
              1535, 1536, 1537, 2047, 2048, 2049, 2431, 2432, 2433, 2559, 2560, 2561, 3001]


def _cases():
    rng = np.random.default_rng(20261017)
    out = []
    for n in BOUNDARY_N:
        m = int(rng.choice([1, 3, 17, 33, 64]))
        sel = int(rng.integers(0, 3)) if n <= 600 else 0
        dep = int(rng.integers(0, 2))
        stream = int(rng.choice([1, 2]))
        out.append((n, m, sel, dep, stream, int(rng.integers(1, 1000))))
    return out


@pytest.fixture(scope="module")
def aco():
    from paper_1101_2678_b200 import aco as _aco

    return _aco


@pytest.mark.parametrize("n,m,sel,dep,stream,seed", _cases())
def test_fuzz_iteration_bit_exact(aco, oracle, n, m, sel, dep, stream, seed):
    nn = min(30, n - 1)
    prob = aco.build_problem(aco.synthetic_instance(n, seed_state=seed))
    cfg = aco.RunConfig(params=aco.Parameters(m=m, seed=seed, nn=nn),
                        selection=aco.SelectionStrategy(aco.Selection(sel)),
                        deposit=aco.DepositStrategy(aco.Deposit(dep)),
                        stream=aco.WeightStream(stream))
    nnl = oracle.nn_lists(prob.dist, nn) if sel == 1 else None
    with aco.Engine(prob, cfg) as eng:
        tau = np.full((n, n), eng.tau0)
        for it in range(2):
            if dep == 0:
                eng.set_pheromone(tau)
            ch = oracle.choice(prob.dist, tau)
            eng.run_iteration()
            t_ref, l_ref, _ = oracle.construct(prob.dist, ch, seed, it, 0, m, selection=sel,
                                               nn_lists=nnl)
            t, l = eng.ants()
            assert np.array_equal(t, t_ref), f"tours differ at iteration {it}"
            assert np.array_equal(l, l_ref)
            tau_ref = oracle.update(tau, t_ref, l_ref, 0.5, dep if dep else 0)
            got = eng.pheromone()
            if dep:
                assert np.array_equal(got, tau_ref)
            else:
                assert (np.abs(got - tau_ref) / np.abs(tau_ref)).max() <= 1e-5
            tau = tau_ref
