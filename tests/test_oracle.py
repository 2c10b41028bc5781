"""The CPU oracle (oracle/aco_oracle.c) pinned against the reference: golden
vectors generated from the reference's own headers (tests/golden/golden.json,
tests/golden/make_golden.py), the Random123 Philox known-answer vectors, the
SURVEY App. B trace, att48.opt.tour = 10628, and — where oracle/_ref is
built — direct comparison with the reference on identical inputs."""
import numpy as np
import pytest

from pyoracle import fnv1a64, synth_coords


def test_philox_known_answers(oracle, golden):
    # Random123 KATs (SURVEY [E4]) as produced by rng.hpp
    expect = {0: [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8],
              1: [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD],
              2: [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]}
    for i, kat in enumerate(golden["philox_kat"]):
        assert kat["out"] == expect[i]
        assert oracle.philox(kat["ctr"], kat["key"]).tolist() == expect[i]


def test_uniform_at_golden(oracle, golden):
    for seed, it, ant, st, dr, val in golden["uniform_at"]:
        assert oracle.uniform_at(seed, it, ant, st, dr) == float(val)
    assert oracle.uniform_at(1, 0, 0, 1, 0) == 0.134225263379676  # SURVEY [E4]


def test_synth_generator_app_b(oracle, golden):
    xs, ys = synth_coords(198)
    assert [xs[0], ys[0], xs[-1], ys[-1]] == [7124.0, 992.0, 7976.0, 5725.0]
    d = oracle.build_dist(xs, ys)
    assert fnv1a64(d) == golden["synth198"]["dist_fnv"]
    assert int(d.max()) == golden["synth198"]["max_d"] == 13061


@pytest.mark.parametrize("n", [1002, 2392])
def test_dist_tau0_choice_nn_golden(oracle, golden, n):
    g = golden[f"synth{n}"]
    xs, ys = synth_coords(n)
    d = oracle.build_dist(xs, ys)
    assert fnv1a64(d) == g["dist_fnv"]
    tau0 = oracle.tau0(d, n)
    assert repr(tau0) == g["tau0"]
    assert fnv1a64(oracle.choice(d, np.full((n, n), tau0))) == g["choice0_fnv"]
    assert fnv1a64(oracle.nn_lists(d, 30)) == g["nn30_fnv"]


def test_construct_golden_pr1002_subset(oracle, golden):
    g = golden["synth1002"]
    n = 1002
    xs, ys = synth_coords(n)
    d = oracle.build_dist(xs, ys)
    ch = oracle.choice(d, np.full((n, n), oracle.tau0(d, n)))
    t, l, _ = oracle.construct(d, ch, 1, 0, 0, g["ants"])
    assert fnv1a64(t) == g["roulette_tours_fnv"]
    assert l.tolist() == g["roulette_lengths"]
    t, l, _ = oracle.construct(d, ch, 1, 0, 0, g["ants"], selection=1,
                               nn_lists=oracle.nn_lists(d, 30))
    assert fnv1a64(t) == g["nn_tours_fnv"]
    assert l.tolist() == g["nn_lengths"]


def _oracle_trace(oracle, d, n, m, selection, deposit, iters, nn_lists=None, random_start=False):
    tau = np.full((n, n), oracle.tau0(d, m))
    out = []
    best_so_far, best_tour = None, None
    for it in range(iters):
        ch = oracle.choice(d, tau)
        t, l, _ = oracle.construct(d, ch, 1, it, 0, m, selection=selection, nn_lists=nn_lists,
                                   random_start=random_start)
        k = int(np.argmin(l))  # first minimum = lowest ant index (engine.hpp:126)
        if best_so_far is None or l[k] < best_so_far:
            best_so_far, best_tour = int(l[k]), t[k].tolist()
        out.append((int(l[k]), repr(float(l.sum() / m)), fnv1a64(t)))
        tau = oracle.update(tau, t, l, 0.5, deposit)
    return out, tau, oracle.choice(d, tau), best_so_far, best_tour


@pytest.mark.parametrize("idx", range(7))
def test_oracle_reproduces_reference_traces_synth198(oracle, golden, idx):
    tr = golden["synth198"]["traces"][idx]
    n = 198
    xs, ys = synth_coords(n)
    d = oracle.build_dist(xs, ys)
    nnl = oracle.nn_lists(d, tr["nn"]) if tr["selection"] == 1 else None
    dep = 0 if tr["deposit"] == 0 else 1
    out, tau, ch, bsf, btour = _oracle_trace(oracle, d, n, tr["m"], tr["selection"], dep,
                                             tr["iters"], nnl, tr["random_start"])
    assert [o[0] for o in out] == tr["best"]
    assert [o[1] for o in out] == tr["mean"]
    assert [o[2] for o in out] == tr["tours_fnv"]
    assert fnv1a64(tau) == tr["tau_fnv"]
    assert fnv1a64(ch) == tr["choice_fnv"]
    assert bsf == tr["best_so_far"] and btour == tr["best_tour"]


def test_survey_app_b_best_lengths(golden):
    assert golden["synth198"]["traces"][0]["best"] == [
        337609, 295944, 292432, 273201, 240896, 210992, 183553, 161663, 147270, 139482]
    assert golden["synth198"]["traces"][1]["best"] == golden["synth198"]["traces"][0]["best"]
    assert golden["synth198"]["traces"][0]["mean"][0] == "389034.21717171714"
    assert golden["synth198"]["tau0"] == "0.0015039764225110329"


def test_att48(oracle, golden):
    g = golden["att48"]
    xs, ys = np.array(g["xs"]), np.array(g["ys"])
    d = oracle.build_dist(xs, ys, g["ewt"])
    assert fnv1a64(d) == g["dist_fnv"]
    tour = np.array(g["opt_tour"] + [g["opt_tour"][0]], np.int32)
    assert oracle.tour_length(d, tour) == g["opt_len"] == 10628
    assert repr(oracle.tau0(d, 48)) == g["tau0"] == "0.0037322136692325637"
    tr = g["trace_roulette_accumulate"]
    out, *_ = _oracle_trace(oracle, d, 48, 48, 0, 0, 10)
    assert [o[0] for o in out] == tr["best"] == [19597, 18652, 15920, 15477, 14151, 13836,
                                                 13567, 13062, 11937, 12421]


def test_gather_restatement_equals_reference_gather_family(oracle, reference):
    """SURVEY [E7]: the O(m n) restated gather equals scatter-gather, tiled and
    symmetric-reduction bitwise, from an evolved tau."""
    n, m = 60, 90
    xs, ys = synth_coords(n)
    d = oracle.build_dist(xs, ys)
    tau = np.full((n, n), oracle.tau0(d, m))
    for it in range(3):
        ch = oracle.choice(d, tau)
        t, l, _ = oracle.construct(d, ch, 1, it, 0, m)
        tau = oracle.update(tau, t, l, 0.5, 1)
    ch = oracle.choice(d, tau)
    t, l, _ = oracle.construct(d, ch, 1, 3, 0, m)
    mine = oracle.update(tau, t, l, 0.5, 1)
    for variant in (1, 2, 3):
        ref, led = reference.update(d, tau, t, l, 0.5, variant, theta=7)
        assert np.array_equal(mine, ref), f"variant {variant}"
        assert np.array_equal(led, reference.predicted_access_cost(variant, n, m, 7))
    acc_o = oracle.update(tau, t, l, 0.5, 0)
    acc_r, _ = reference.update(d, tau, t, l, 0.5, 0)
    assert np.array_equal(acc_o, acc_r)


@pytest.mark.parametrize("sel", [0, 1, 2])
def test_oracle_construct_equals_reference(oracle, reference, sel):
    n = 150
    xs, ys = synth_coords(n, state=9)
    d = oracle.build_dist(xs, ys)
    assert np.array_equal(d, reference.build_problem(xs, ys))
    rng = np.random.default_rng(1)
    tau = rng.random((n, n)) * 1e-3
    tau = (tau + tau.T) / 2
    ch = oracle.choice(d, tau)
    assert np.array_equal(ch, reference.choice(d, tau))
    nnl = oracle.nn_lists(d, 10) if sel == 1 else None
    if sel == 1:
        assert np.array_equal(nnl, reference.nn_lists(d, 10))
    t1, l1, _ = oracle.construct(d, ch, 5, 3, 0, 40, selection=sel, nn_lists=nnl, theta=7)
    t2, l2 = reference.construct(d, ch, 5, 3, 0, 40, selection=sel, nn_lists=nnl, theta=7)
    assert np.array_equal(t1, t2) and np.array_equal(l1, l2)


def test_oracle_degenerate_branches(oracle, reference):
    """Zero weights (zero-total branch) and coincident cities (d == 0 -> eta 1)."""
    n = 40
    xs, ys = synth_coords(n, state=3)
    xs[5], ys[5] = xs[6], ys[6]  # coincident pair
    d = oracle.build_dist(xs, ys)
    assert d[5, 6] == 0
    tau = np.full((n, n), 1e-3)
    tau[:, :20] = 0.0  # half the columns carry no pheromone
    ch = oracle.choice(d, tau)
    assert np.array_equal(ch, reference.choice(d, tau))
    t1, l1, st = oracle.construct(d, ch, 2, 0, 0, n)
    t2, l2 = reference.construct(d, ch, 2, 0, 0, n)
    assert np.array_equal(t1, t2)
    assert st[2] > 0  # the zero-total branch fired


def test_philox_uniform_ks(oracle):
    """Draw 0 of consecutive steps is uniform on [0, 1) (KS)."""
    from scipy.stats import kstest

    u = np.array([oracle.uniform_at(1, 0, 0, s, 0) for s in range(20000)])
    assert u.min() >= 0.0 and u.max() < 1.0
    assert kstest(u, "uniform").pvalue > 1e-4
    v = np.array([oracle.uniform_at(1, 0, 1, s, 0) for s in range(20000)])
    assert np.corrcoef(u, v)[0, 1] < 0.05  # ant streams are separate


def test_data_parallel_theta_invariance(oracle, reference):
    """The reference's tiled data-parallel selection does not depend on the
    tile size theta, and equals the oracle's (untiled)."""
    n = 150
    xs, ys = synth_coords(n)
    d = oracle.build_dist(xs, ys)
    ch = oracle.choice(d, np.full((n, n), oracle.tau0(d, n)))
    base, _, _ = oracle.construct(d, ch, 3, 0, 0, 40, selection=2)
    for theta in (1, 7, 32, 64, 150, 1000):
        t, _ = reference.construct(d, ch, 3, 0, 0, 40, selection=2, theta=theta)
        assert np.array_equal(t, base), theta
