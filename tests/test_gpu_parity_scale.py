"""GPU parity at the BASELINE configurations' own sizes (VERDICT r1, next-round
item 1): the whole pr2392 m = n colony over several gather iterations, the
synthetic 10k nn-30 configuration on an oracle-evolved tau with the top-K
argmax cache live, and the late-run regime whose scaled fp32 weights go
subnormal (the certification's absolute-error terms then carry the proof and
the fp64 tiers must fire).  The oracle (oracle/aco_oracle.c, pinned to the
reference in tests/test_oracle.py) runs chunked over all host cores —
ctypes releases the GIL — so a full pr2392 colony is a few seconds.

Matches /root/reference/proj/include/aco/construction.hpp:42-68 (roulette),
:73-121 (nn + argmax fallback) and pheromone.hpp:213-228 (scatter-gather)."""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def aco():
    from paper_1101_2678_b200 import aco as _aco

    return _aco


def par_construct(oracle, dist, choice, seed, it, k0, k1, **kw):
    """oracle.construct over [k0, k1) split across host threads (identical
    output: every ant's tour is a pure function of (choice, seed, it, k))."""
    threads = max(1, min(os.cpu_count() or 1, 32))
    cnt = k1 - k0
    step = max(1, -(-cnt // (threads * 2)))
    ranges = [(a, min(k1, a + step)) for a in range(k0, k1, step)]
    with ThreadPoolExecutor(threads) as ex:
        parts = list(ex.map(lambda r: oracle.construct(dist, choice, seed, it, r[0], r[1], **kw),
                            ranges))
    return (np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts]))


def make(aco, prob, selection=0, deposit=1, stream=0, m=0, nn=30, ant_range=None):
    cfg = aco.RunConfig(params=aco.Parameters(m=m, nn=nn, seed=1),
                        selection=aco.SelectionStrategy(aco.Selection(selection)),
                        deposit=aco.DepositStrategy(aco.Deposit(deposit)),
                        stream=aco.WeightStream(stream))
    if ant_range:
        cfg.ant_begin, cfg.ant_end = ant_range
    return aco.Engine(prob, cfg)


def test_pr2392_full_colony_gather_bit_exact(aco, oracle):
    """BASELINE config 3 in full: all 2392 ants, three scatter-to-gather
    iterations on the default (fp32-filter) stream — every tour, length,
    tau and choice cell bit-exact, statistics equal."""
    n = 2392
    prob = aco.build_problem(aco.synthetic_instance(n))
    with make(aco, prob, deposit=1) as eng:
        tau = np.full((n, n), eng.tau0)
        best = None
        for it in range(3):
            ch = oracle.choice(prob.dist, tau)
            assert np.array_equal(eng.choice(), ch), f"choice at iteration {it}"
            rec = eng.run_iteration()
            t_ref, l_ref = par_construct(oracle, prob.dist, ch, 1, it, 0, n)
            t, l = eng.ants()
            assert np.array_equal(t, t_ref), f"tours differ at iteration {it}"
            assert np.array_equal(l, l_ref)
            assert rec.best_length == int(l_ref.min())
            assert rec.mean_length == float(l_ref.sum()) / n
            best = int(l_ref.min()) if best is None else min(best, int(l_ref.min()))
            assert rec.best_so_far == best == eng.best_length()
            tau = oracle.update(tau, t_ref, l_ref, 0.5, 1)
            assert np.array_equal(eng.pheromone(), tau), f"tau at iteration {it}"


def _converged_tau(n, rng):
    """A late-run pheromone (symmetric): cities [0, n/2) still mix (tau
    2^-U(0, 20) among themselves), cities [n/2, n) have converged onto
    4-cliques (tau 1 inside a clique), and every other edge was unused for
    250-300 evaporations at rho = 0.5 (tau 2^-U(250, 300)).  Scaled to its
    row maximum, such an edge lands below the fp32 subnormal range, so a step
    whose unvisited cities are all of that kind can only be decided by the
    exact replay, while the mixing half keeps the ordinary fp32/fp64 tiers
    busy."""
    h = n // 2
    tau = np.exp2(-rng.uniform(250.0, 300.0, size=(n, n)))
    tau[:h, :h] = np.exp2(-rng.uniform(0.0, 20.0, size=(h, h)))
    perm = h + rng.permutation(n - h)
    for g in range(0, len(perm) - 3, 4):
        q = perm[g:g + 4]
        tau[np.ix_(q, q)] = 1.0
    return np.minimum(tau, tau.T)


def test_late_run_subnormal_regime_tiers_fire_bit_exact(aco, oracle):
    """pr2392 on the fp32 stream with a converged, wide-range tau (2^-300 ..
    1): the row-scaled fp32 weights of the decayed edges underflow, so the
    fp32 certification (tier 1) must defer; the fp64 re-sum over the staged
    row (tier 2) certifies the rounding-bound cases and the exact replay
    (tier 3) the underflowed ones.  Both tiers must actually fire, and every
    tour, length and tau cell stays bit-exact."""
    n, ants = 2392, 384
    prob = aco.build_problem(aco.synthetic_instance(n))
    rng = np.random.default_rng(7)
    tau = _converged_tau(n, rng)
    tier2 = exact = 0
    with make(aco, prob, deposit=1, stream=2, ant_range=(0, ants)) as eng:
        for it in range(2):
            eng.set_pheromone(tau)
            ch = oracle.choice(prob.dist, tau)
            assert np.array_equal(eng.choice(), ch)
            rec = eng.construct()
            # 384 ants: the plain launch, rows in the natural layout (odd NV)
            assert ",nat>" in eng.describe()
            tier2 += rec.certified_fp64
            exact += rec.fallbacks
            t_ref, l_ref = par_construct(oracle, prob.dist, ch, 1, it, 0, ants)
            t, l = eng.ants()
            assert np.array_equal(t, t_ref), f"tours differ at iteration {it}"
            assert np.array_equal(l, l_ref)
            eng.update()
            tau = oracle.update(tau, t_ref, l_ref, 0.5, 1)
            assert np.array_equal(eng.pheromone(), tau)
    assert tier2 > 0, "the fp64 re-sum tier never fired"
    assert exact > 0, "the exact replay tier never fired"


def test_synth10k_nn30_evolved_tau_topk_live(aco, oracle):
    """BASELINE config 5 at its own size: synthetic 10k cities, nn = 30, on
    a tau evolved by one full oracle iteration of all 10000 ants (gather
    deposit), then two engine iterations over 160 ants spread across the
    colony: tours, lengths and the gather tau bit-exact, with the per-row
    top-128 argmax cache rebuilt after every update and taking the fallbacks."""
    n, nn = 10000, 30
    prob = aco.build_problem(aco.synthetic_instance(n))
    nnl = oracle.nn_lists(prob.dist, nn)
    tau0 = oracle.tau0(prob.dist, n)
    tau = np.full((n, n), tau0)
    ch = oracle.choice(prob.dist, tau)
    t0, l0 = par_construct(oracle, prob.dist, ch, 1, 0, 0, n, selection=1, nn_lists=nnl)
    tau = oracle.update(tau, t0, l0, 0.5, 1)  # evolved: one full-colony iteration
    del ch, t0, l0
    for lo in (0, 6000):
        with make(aco, prob, selection=1, deposit=1, nn=nn, ant_range=(lo, lo + 80)) as eng:
            assert eng.tau0 == tau0
            eng.set_pheromone(tau)
            tau_e = tau
            for it in (1, 2):
                ch = oracle.choice(prob.dist, tau_e)
                # the engine's iteration counter starts at 0: key the oracle's draws the same
                eng.construct()
                desc = dict(kv.split("=") for kv in eng.describe().split() if "=" in kv)
                t_ref, l_ref = par_construct(oracle, prob.dist, ch, 1, it - 1, lo, lo + 80,
                                             selection=1, nn_lists=nnl)
                del ch
                t, l = eng.ants()
                assert np.array_equal(t, t_ref), f"ants {lo}.. iteration {it}"
                assert np.array_equal(l, l_ref)
                assert int(desc["topk"]) >= 128  # the cache is live
                assert int(desc["argmax_fallbacks"]) > 0
                assert int(desc["full_row_scans"]) < int(desc["argmax_fallbacks"])
                eng.update()
                tau_e = oracle.update(tau_e, t_ref, l_ref, 0.5, 1)
                assert np.array_equal(eng.pheromone(), tau_e), f"tau, ants {lo}.., it {it}"
