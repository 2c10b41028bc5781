"""SPEC.md properties (SURVEY §4 checklist) re-asserted on the GPU engine's
own outputs, independent of the oracle: forced moves, the roulette's
selection law (chi-square), tau symmetry and deposit conservation,
determinism, and the att48 quality band."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def aco():
    from paper_1101_2678_b200 import aco as _aco

    return _aco


def _engine(aco, spec, m=0, selection=0, deposit=1, seed=1, nn=30, iterations=100):
    prob = aco.build_problem(spec)
    cfg = aco.RunConfig(params=aco.Parameters(m=m, seed=seed, nn=nn, iterations=iterations),
                        selection=aco.SelectionStrategy(aco.Selection(selection)),
                        deposit=aco.DepositStrategy(aco.Deposit(deposit)))
    return prob, aco.Engine(prob, cfg)


def _att48(aco, golden):
    g = golden["att48"]
    return aco.InstanceSpec("att48", 48, aco.EdgeWeightType.att, np.array(g["xs"]),
                            np.array(g["ys"]))


@pytest.mark.parametrize("selection", [0, 1, 2])
def test_forced_moves(aco, selection):
    """tau zero everywhere except a Hamiltonian cycle i -> i+1: every
    selection rule must follow the only positive-weight edge."""
    n = 64
    # cities on a circle, in order: i+1 is among i's nearest neighbours, so
    # the nn rule sees the positive edge in its list too
    ang = 2 * np.pi * np.arange(n) / n
    spec = aco.InstanceSpec("circle64", n, aco.EdgeWeightType.euc_2d,
                            np.round(5000 + 4000 * np.cos(ang)), np.round(5000 + 4000 * np.sin(ang)))
    prob, eng = _engine(aco, spec, selection=selection, nn=8)
    with eng:
        tau = np.zeros((n, n))
        for i in range(n):
            tau[i, (i + 1) % n] = 1.0
        eng.set_pheromone(tau)
        eng.construct()
        tours, _ = eng.ants()
        for k, t in enumerate(tours):
            assert t[0] == k % n and t[-1] == t[0]
            # while the successor is unvisited it is the only positive weight
            assert all(t[s + 1] == (t[s] + 1) % n for s in range(n - 1)), f"ant {k}"


def test_roulette_first_move_law_chi_square(aco):
    """First moves from a fixed start follow p_j = w_j / sum w (Eq. 1 of the
    paper): chi-square over 4000 ants per start city."""
    from scipy.stats import chisquare

    n, per = 6, 4000
    prob, eng = _engine(aco, aco.synthetic_instance(n), m=n * per)
    with eng:
        eng.construct()
        tours, _ = eng.ants()
        w = eng.choice()
        for s in range(n):
            first = tours[s::n, 1]
            obs = np.bincount(first, minlength=n).astype(float)
            p = w[s].copy()
            p[s] = 0.0
            p /= p.sum()
            keep = p > 0
            stat, pval = chisquare(obs[keep], per * p[keep])
            assert pval > 1e-4, f"start {s}: p = {pval}"


def test_tau_symmetry_and_deposit_conservation(aco):
    """Scatter-to-gather path: tau stays exactly symmetric, and every update
    adds exactly the deposited mass sum_k 2 n / C_k."""
    n = 300
    prob, eng = _engine(aco, aco.synthetic_instance(n))
    with eng:
        for it in range(4):
            before = eng.pheromone()
            eng.run_iteration()
            after = eng.pheromone()
            assert np.array_equal(after, after.T), f"asymmetric at iteration {it}"
            _, lens = eng.ants()
            mass = (after - before * 0.5).sum()
            expect = (2.0 * n / lens.astype(np.float64)).sum()
            assert abs(mass - expect) <= 1e-9 * expect


@pytest.mark.parametrize("selection", [0, 2])
def test_accumulate_one_gpu_symmetric_and_conserving(aco, selection):
    """One-GPU accumulate (k_deposit_sym + k_rows<DELTA_SYM>): both cells of an
    edge receive the same fl(fl(tau*keep) + delta), so tau stays EXACTLY
    symmetric; the deposited mass matches sum_k 2n/C_k to rounding."""
    n = 300
    prob, eng = _engine(aco, aco.synthetic_instance(n), deposit=0, selection=selection)
    with eng:
        for it in range(4):
            before = eng.pheromone()
            eng.run_iteration()
            after = eng.pheromone()
            assert np.array_equal(after, after.T), f"asymmetric at iteration {it}"
            _, lens = eng.ants()
            mass = (after - before * 0.5).sum()
            expect = (2.0 * n / lens.astype(np.float64)).sum()
            assert abs(mass - expect) <= 1e-9 * expect


@pytest.mark.parametrize("deposit", [1, 0])
def test_determinism(aco, deposit):
    """Same configuration and seed, two engines: identical tours, lengths and
    best tour; gather tau bitwise, atomic tau within 1e-12."""
    spec = aco.synthetic_instance(400)
    _, a = _engine(aco, spec, deposit=deposit, seed=9)
    _, b = _engine(aco, spec, deposit=deposit, seed=9)
    with a, b:
        for _ in range(3):
            ra, rb = a.run_iteration(), b.run_iteration()
            assert ra.best_length == rb.best_length and ra.mean_length == rb.mean_length
            assert np.array_equal(a.ants()[0], b.ants()[0])
        assert np.array_equal(a.best_tour(), b.best_tour())
        pa, pb = a.pheromone(), b.pheromone()
        if deposit:
            assert np.array_equal(pa, pb)
        else:
            assert (np.abs(pa - pb) / pa).max() <= 1e-12


def test_att48_quality_band(aco, golden):
    """att48, m = 48, roulette over nn-30 lists, 100 iterations, 10 seeds:
    median best within 10% of the optimum 10628."""
    spec = _att48(aco, golden)
    best = []
    for seed in range(1, 11):
        _, eng = _engine(aco, spec, m=48, selection=1, deposit=0, seed=seed)
        with eng:
            rep = eng.run()
            best.append(rep.best_length)
            assert aco.tour_length(aco.build_problem(spec), rep.best_tour) == rep.best_length
    assert np.median(best) <= 1.10 * 10628, best
