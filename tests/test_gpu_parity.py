"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Integer outputs (tours, lengths) and the deterministic
pheromone path must be bit-exact; the atomic path is checked per iteration
from a shared state within 1e-5 relative (north_star)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ATOMIC_RTOL = 1e-5


@pytest.fixture(scope="module")
def aco():
    from paper_1101_2678_b200 import aco as _aco

    return _aco


def make(aco, n, selection=0, deposit=0, stream=0, m=0, ant_range=None, nn=30, seed=1,
         random_start=False, alpha=1.0, beta=2.0, rho=0.5, spec=None):
    spec = spec or aco.synthetic_instance(n)
    prob = aco.build_problem(spec)
    cfg = aco.RunConfig(params=aco.Parameters(m=m, nn=nn, seed=seed, alpha=alpha, beta=beta,
                                              rho=rho),
                        selection=aco.SelectionStrategy(aco.Selection(selection)),
                        deposit=aco.DepositStrategy(aco.Deposit(deposit)),
                        stream=aco.WeightStream(stream), random_start=random_start)
    if ant_range:
        cfg.ant_begin, cfg.ant_end = ant_range
    return prob, aco.Engine(prob, cfg)


def test_device_philox_matches_oracle(aco, oracle, golden):
    rows = golden["uniform_at"]
    for seed, it, ant, st, dr, val in rows[:8]:
        got = aco.philox_uniform_device(seed, it, ant, [st], [dr])[0]
        assert got == float(val) == oracle.uniform_at(seed, it, ant, st, dr)
    rng = np.random.default_rng(3)
    steps = rng.integers(0, 5000, 4096).astype(np.uint32)
    draws = rng.integers(0, 5000, 4096).astype(np.uint32)
    got = aco.philox_uniform_device(1, 7, 123, steps, draws)
    ref = np.array([oracle.uniform_at(1, 7, 123, int(s), int(d)) for s, d in zip(steps, draws)])
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("n", [198, 1002])
def test_initial_choice_bit_exact(aco, oracle, n):
    prob, eng = make(aco, n)
    with eng:
        tau = np.full((n, n), eng.tau0)
        assert eng.tau0 == oracle.tau0(prob.dist, n)
        assert np.array_equal(eng.choice(), oracle.choice(prob.dist, tau))
        assert np.array_equal(eng.pheromone(), tau)


@pytest.mark.parametrize("stream", [1, 2])
def test_roulette_iteration0_d198_all_ants(aco, oracle, stream):
    n = 198
    prob, eng = make(aco, n, stream=stream)
    with eng:
        rec = eng.run_iteration()
        tau = np.full((n, n), eng.tau0)
        t_ref, l_ref, _ = oracle.construct(prob.dist, oracle.choice(prob.dist, tau), 1, 0, 0, n)
        t, l = eng.ants()
        assert np.array_equal(t, t_ref)
        assert np.array_equal(l, l_ref)
        assert rec.best_length == l_ref.min()
        assert rec.mean_length == l_ref.sum() / n


def test_golden_trace_synth198_gather(aco, oracle, golden):
    """SURVEY App. B trace, reproduced bit-for-bit on the deterministic path."""
    from pyoracle import fnv1a64

    tr = golden["synth198"]["traces"][1]  # roulette + scatter-gather, 10 iterations
    assert tr["deposit"] == 1 and tr["selection"] == 0
    n = 198
    prob, eng = make(aco, n, deposit=1)
    with eng:
        for it in range(10):
            rec = eng.run_iteration()
            assert rec.best_length == tr["best"][it]
            assert repr(rec.mean_length) == tr["mean"][it]
            t, _ = eng.ants()
            assert fnv1a64(t) == tr["tours_fnv"][it]
        assert fnv1a64(eng.pheromone()) == tr["tau_fnv"]
        assert fnv1a64(eng.choice()) == tr["choice_fnv"]
        assert eng.best_length() == tr["best_so_far"]
        assert eng.best_tour().tolist() == tr["best_tour"]


def test_golden_trace_synth198_atomic_best_lengths(aco, golden):
    """Atomic deposit: order-nondeterministic tau (<=1e-15), yet the survey's
    best-length trace is reproduced (SURVEY [E9])."""
    tr = golden["synth198"]["traces"][0]
    prob, eng = make(aco, 198, deposit=0)
    with eng:
        best = [eng.run_iteration().best_length for _ in range(10)]
    assert best == tr["best"]


@pytest.mark.parametrize("n,stream", [(1002, 2), (1002, 1)])
def test_roulette_multi_iteration_gather_bit_exact(aco, oracle, n, stream):
    prob, eng = make(aco, n, deposit=3, stream=stream)
    with eng:
        tau = np.full((n, n), eng.tau0)
        for it in range(3):
            ch = oracle.choice(prob.dist, tau)
            assert np.array_equal(eng.choice(), ch)
            eng.run_iteration()
            t_ref, l_ref, _ = oracle.construct(prob.dist, ch, 1, it, 0, n)
            t, l = eng.ants()
            assert np.array_equal(t, t_ref), f"iteration {it}"
            assert np.array_equal(l, l_ref)
            tau = oracle.update(tau, t_ref, l_ref, 0.5, 1)
            assert np.array_equal(eng.pheromone(), tau)


def test_atomic_update_within_tolerance_from_shared_state(aco, oracle):
    n = 1002
    prob, eng = make(aco, n, deposit=0)
    with eng:
        tau = np.full((n, n), eng.tau0)
        for it in range(3):
            eng.set_pheromone(tau)
            ch = oracle.choice(prob.dist, tau)
            assert np.array_equal(eng.choice(), ch)
            eng.run_iteration()
            t_ref, l_ref, _ = oracle.construct(prob.dist, ch, 1, it, 0, n)
            t, l = eng.ants()
            assert np.array_equal(t, t_ref)
            tau_ref = oracle.update(tau, t_ref, l_ref, 0.5, 0)
            got = eng.pheromone()
            rel = np.abs(got - tau_ref) / np.abs(tau_ref)
            assert rel.max() <= ATOMIC_RTOL
            tau = tau_ref


def test_pr2392_ant_subset_iteration0(aco, oracle, golden):
    """pr2392 scale: ants 0..15 of iteration 0 against the reference's own
    golden hash, plus ants 1000..1031 against the oracle."""
    from pyoracle import fnv1a64

    g = golden["synth2392"]
    n = 2392
    for stream in (2, 1):
        prob, eng = make(aco, n, stream=stream, ant_range=(0, g["ants"]))
        with eng:
            eng.construct()
            t, l = eng.ants()
            assert fnv1a64(t) == g["roulette_tours_fnv"]
            assert l.tolist() == g["roulette_lengths"]
    prob, eng = make(aco, n, ant_range=(1000, 1032))
    with eng:
        eng.construct()
        t, l = eng.ants()
        tau = np.full((n, n), eng.tau0)
        t_ref, l_ref, _ = oracle.construct(prob.dist, oracle.choice(prob.dist, tau), 1, 0, 1000,
                                           1032)
        assert np.array_equal(t, t_ref)


@pytest.mark.parametrize("n", [198, 1002])
def test_nn_selection_bit_exact(aco, oracle, n):
    prob, eng = make(aco, n, selection=1, deposit=1)
    with eng:
        nnl = oracle.nn_lists(prob.dist, 30)
        tau = np.full((n, n), eng.tau0)
        for it in range(3):
            ch = oracle.choice(prob.dist, tau)
            eng.run_iteration()
            t_ref, l_ref, st = oracle.construct(prob.dist, ch, 1, it, 0, n, selection=1,
                                                nn_lists=nnl)
            t, l = eng.ants()
            assert np.array_equal(t, t_ref), f"iteration {it}"
            tau = oracle.update(tau, t_ref, l_ref, 0.5, 1)
            assert np.array_equal(eng.pheromone(), tau)


def test_data_parallel_selection_bit_exact(aco, oracle):
    n = 198
    prob, eng = make(aco, n, selection=2, deposit=1)
    with eng:
        tau = np.full((n, n), eng.tau0)
        for it in range(2):
            ch = oracle.choice(prob.dist, tau)
            eng.run_iteration()
            t_ref, l_ref, _ = oracle.construct(prob.dist, ch, 1, it, 0, n, selection=2)
            t, _ = eng.ants()
            assert np.array_equal(t, t_ref)
            tau = oracle.update(tau, t_ref, l_ref, 0.5, 1)


def test_random_start_bit_exact(aco, oracle):
    n = 198
    prob, eng = make(aco, n, random_start=True, deposit=1)
    with eng:
        tau = np.full((n, n), eng.tau0)
        eng.run_iteration()
        t_ref, _, _ = oracle.construct(prob.dist, oracle.choice(prob.dist, tau), 1, 0, 0, n,
                                       random_start=True)
        t, _ = eng.ants()
        assert np.array_equal(t, t_ref)


def test_att48_trace(aco, golden):
    g = golden["att48"]
    spec = aco.InstanceSpec("att48", 48, aco.EdgeWeightType.att, np.array(g["xs"]),
                            np.array(g["ys"]))
    prob, eng = make(aco, 48, spec=spec, deposit=0)
    with eng:
        best = [eng.run_iteration().best_length for _ in range(10)]
    assert best == g["trace_roulette_accumulate"]["best"]


@pytest.mark.parametrize("topk", ["1", "0"])
def test_nn_argmax_cache_bit_exact(aco, oracle, monkeypatch, topk):
    """The nn selection's argmax fallback through the per-row top-K cache
    (k_row_topk) and through the full-row scan (ACO_NN_TOPK=0) both give the
    reference's tours; n=3000 with nn=8 makes the fallback frequent, and the
    cache must take most of them."""
    monkeypatch.setenv("ACO_NN_TOPK", topk)
    n, nn = 3000, 8
    prob, eng = make(aco, n, selection=1, deposit=1, nn=nn, ant_range=(0, 96))
    with eng:
        nnl = oracle.nn_lists(prob.dist, nn)
        tau = np.full((n, n), eng.tau0)
        ch = oracle.choice(prob.dist, tau)
        eng.construct()
        desc = eng.describe()
        t_ref, l_ref, _ = oracle.construct(prob.dist, ch, 1, 0, 0, 96, selection=1, nn_lists=nnl)
        t, l = eng.ants()
        assert np.array_equal(t, t_ref)
        assert np.array_equal(l, l_ref)
        fields = dict(kv.split("=") for kv in desc.split() if "=" in kv)
        argmax, full = int(fields["argmax_fallbacks"]), int(fields["full_row_scans"])
        assert argmax > 1000
        if topk == "1":
            assert int(fields["topk"]) >= 128 and full < argmax // 2
        else:
            assert fields["topk"] == "off" and full == argmax


_TAIL_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1101_2678_b200 import aco
prob = aco.build_problem(aco.synthetic_instance(700))
for dep in (0, 1):
    cfg = aco.RunConfig(params=aco.Parameters(m=64, nn=12, seed=4),
                        selection=aco.SelectionStrategy(aco.Selection.roulette_nn),
                        deposit=aco.DepositStrategy(aco.Deposit(dep)))
    with aco.Engine(prob, cfg) as eng:
        for _ in range(3 if dep else 1):  # atomic tau is order-nondeterministic
            eng.run_iteration()
        t, l = eng.ants()
        np.save(sys.argv[2] + f"_{dep}_tours.npy", t)
        np.save(sys.argv[2] + f"_{dep}_lens.npy", l)
        np.save(sys.argv[2] + f"_{dep}_tau.npy", eng.pheromone())
        print(eng.describe())
"""


def test_nn_tour_tail_matches_k_tour_length(tmp_path):
    """The nn kernel's fused tour tail (C_k, 1/C_k, succ/pred) and the
    separate k_tour_length launch (ACO_FUSED_TAIL=0, read once per process,
    hence the subprocesses) give identical tours, lengths and — for the
    gather deposit, which reads succ/pred and 1/C_k — bit-identical tau
    over three iterations (the atomic deposit: one iteration, tau within
    1e-5)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for v in ("1", "0"):
        env = dict(os.environ, ACO_FUSED_TAIL=v)
        r = subprocess.run([sys.executable, "-c", _TAIL_SCRIPT, root, str(tmp_path / v)],
                           env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        out[v] = {dep: [np.load(tmp_path / f"{v}_{dep}_{k}.npy") for k in ("tours", "lens", "tau")]
                  for dep in (0, 1)}
    for dep in (0, 1):
        a, b = out["1"][dep], out["0"][dep]
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        if dep == 1:
            assert np.array_equal(a[2], b[2])
        else:
            assert np.max(np.abs(a[2] - b[2]) / b[2]) <= 1e-5


def _expected_topk(choice, k):
    n = choice.shape[0]
    out = np.full((n, k), -1, np.int32)
    idx = np.arange(n)
    for i in range(n):
        order = np.lexsort((idx, -choice[i]))[:k]  # (w desc, index asc)
        out[i, :len(order)] = order
    return out


@pytest.mark.parametrize("n,pattern", [(1500, "uniform"), (1500, "loguniform"),
                                       (2392, "ties"), (100, "uniform"), (300, "loguniform")])
def test_nn_topk_lists_exact(aco, n, pattern):
    """k_row_topk's lists equal the exact top-K under (choice desc, index
    asc) of the device choice rows: uniform tau (eta ties from integer
    distances), log-uniform tau over 2^-100..1 (exponents spread across the
    threshold search), tau from 3 values (heavy ties), and n < K (the list
    ends with -1).  A row may only be marked -2 (full scan) when more of
    its cities than the kernel's candidate scratch holds (6 K) tie at or
    above its K-th value's 2^-20 band."""
    prob, eng = make(aco, n, selection=1, deposit=0, nn=8, ant_range=(0, 1))
    rng = np.random.default_rng(n)
    with eng:
        if pattern == "uniform":
            tau = np.full((n, n), eng.tau0)
        elif pattern == "loguniform":
            tau = np.exp2(-100.0 * rng.random((n, n)))
        else:
            tau = rng.choice([1.0, 0.5, 0.25], size=(n, n))
        tau = np.minimum(tau, tau.T)  # symmetric like the colony's
        eng.set_pheromone(tau)
        eng.compute_choice_info()
        ch = eng.choice()
        got = eng.topk()
    K = got.shape[1]
    assert K in (128, 256, 512)
    cap = 6 * K if K <= 256 else 4 * K
    exp = _expected_topk(ch, K)
    bad = got[:, 0] == -2
    for i in np.nonzero(bad)[0]:
        kth = np.sort(ch[i])[::-1][K - 1]
        assert np.count_nonzero(ch[i] >= kth * (1 - 2.0 ** -20)) > cap, f"row {i} flagged without overflow"
    assert np.array_equal(got[~bad], exp[~bad])
    if pattern != "ties":
        assert not bad.any()


def test_gather_cta_row_kernel_bit_exact(aco, oracle):
    """n = 4500: a row of doubles no longer fits one warp's shared slice, so
    the gather update runs the CTA-per-row k_rows<GATHER> (paired, batched
    epilogue) — bit-exact tau and choice over two iterations."""
    n, m = 4500, 64
    prob, eng = make(aco, n, deposit=1, m=m)
    with eng:
        tau = np.full((n, n), eng.tau0)
        for it in range(2):
            ch = oracle.choice(prob.dist, tau)
            assert np.array_equal(eng.choice(), ch)
            eng.run_iteration()
            t_ref, l_ref, _ = oracle.construct(prob.dist, ch, 1, it, 0, m)
            t, l = eng.ants()
            assert np.array_equal(t, t_ref), f"iteration {it}"
            tau = oracle.update(tau, t_ref, l_ref, 0.5, 1)
            assert np.array_equal(eng.pheromone(), tau)
        assert np.array_equal(eng.choice(), oracle.choice(prob.dist, tau))


def test_gather_fold_converged_colony_bit_exact(aco, oracle):
    """The warp-per-row gather fold reproduces the reference's
    scatter-to-gather tau over iterations in which the colony concentrates on
    few edges (rho = 0.9: many equal columns inside each 16-ant chunk)."""
    n = 1002
    prob, eng = make(aco, n, deposit=1, rho=0.9)
    with eng:
        tau = np.full((n, n), eng.tau0)
        for it in range(3):
            ch = oracle.choice(prob.dist, tau)
            eng.run_iteration()
            t_ref, l_ref, _ = oracle.construct(prob.dist, ch, 1, it, 0, n)
            t, l = eng.ants()
            assert np.array_equal(t, t_ref), f"iteration {it}"
            tau = oracle.update(tau, t_ref, l_ref, 0.9, 1)
            assert np.array_equal(eng.pheromone(), tau)


def _spec_dup(aco, n, seed=5):
    """EUC_2D instance with duplicated and collinear cities (zero distances:
    eta = 1 by model.hpp:142, many equal weights)."""
    rng = np.random.default_rng(seed)
    xs = rng.integers(0, 50, n).astype(np.float64)
    ys = rng.integers(0, 50, n).astype(np.float64)
    xs[n // 2:] = xs[: n - n // 2]  # every city of the second half duplicates one of the first
    ys[n // 2:] = ys[: n - n // 2]
    ys[: n // 4] = 7.0               # a collinear run
    return aco.InstanceSpec(name=f"dup{n}", dimension=n, xs=xs, ys=ys)


@pytest.mark.parametrize("n", [2, 3, 5, 33, 97])
@pytest.mark.parametrize("selection", [0, 1, 2])
@pytest.mark.parametrize("dup", [False, True])
def test_small_and_degenerate_instances_bit_exact(aco, oracle, n, selection, dup):
    """Edge cases: tiny n (one-lane chunks, a single unvisited city, n < warp
    width), duplicate cities (zero distances) and ties, for every selection
    rule; gather-path tau bit-exact over three iterations."""
    if dup and n < 5:
        pytest.skip("duplicates need n >= 5")
    nn = min(30, n - 1)
    spec = _spec_dup(aco, n) if dup else aco.synthetic_instance(n)
    prob, eng = make(aco, n, selection=selection, deposit=1, nn=nn, spec=spec)
    with eng:
        nnl = oracle.nn_lists(prob.dist, nn) if selection == 1 else None
        tau = np.full((n, n), eng.tau0)
        for it in range(3):
            ch = oracle.choice(prob.dist, tau)
            assert np.array_equal(eng.choice(), ch)
            eng.run_iteration()
            t_ref, l_ref, _ = oracle.construct(prob.dist, ch, 1, it, 0, n, selection=selection,
                                               nn_lists=nnl)
            t, l = eng.ants()
            assert np.array_equal(t, t_ref), f"iteration {it}"
            assert np.array_equal(l, l_ref)
            tau = oracle.update(tau, t_ref, l_ref, 0.5, 1)
            assert np.array_equal(eng.pheromone(), tau)


def test_roulette_exact_kernel_forced_bit_exact(aco, oracle, monkeypatch):
    """k_construct_roulette_exact (every step the exact replay) forced at
    n = 1002: tours and the gather tau bit-exact over two iterations."""
    monkeypatch.setenv("ACO_ROULETTE_EXACT", "1")
    n = 1002
    prob, eng = make(aco, n, deposit=1)
    with eng:
        tau = np.full((n, n), eng.tau0)
        for it in range(2):
            ch = oracle.choice(prob.dist, tau)
            eng.run_iteration()
            assert "k_construct_roulette_exact" in eng.describe()
            t_ref, l_ref, _ = oracle.construct(prob.dist, ch, 1, it, 0, n)
            t, l = eng.ants()
            assert np.array_equal(t, t_ref), f"iteration {it}"
            tau = oracle.update(tau, t_ref, l_ref, 0.5, 1)
            assert np.array_equal(eng.pheromone(), tau)


def test_roulette_beyond_streamed_layout_limit(aco, oracle):
    """n beyond the streamed layouts (fp64 stream: 8 rounds x 32 lanes x 40
    cities = 10240) falls back to the exact-replay kernel instead of failing:
    n = 10300, four ants, tours bit-exact against the oracle."""
    n, m = 10300, 4
    prob, eng = make(aco, n, stream=1, m=m)
    with eng:
        eng.construct()
        assert "k_construct_roulette_exact" in eng.describe()
        t, l = eng.ants()
        tau = np.full((n, n), eng.tau0)
        t_ref, l_ref, _ = oracle.construct(prob.dist, oracle.choice(prob.dist, tau), 1, 0, 0, m)
        assert np.array_equal(t, t_ref)
        assert np.array_equal(l, l_ref)


@pytest.mark.parametrize("pinned", [True, False])
def test_iterate_host_tour_buffers(aco, pinned):
    """aco_gpu_iterate with caller buffers: pinned (device-mapped: the
    construction kernel streams the tours into it) and pageable (copied after
    the construction) both return exactly the engine's tours and lengths."""
    import torch

    n = 1002
    prob, eng = make(aco, n, deposit=0)
    with eng:
        if pinned:
            tb = torch.empty((n, n + 1), dtype=torch.int32, pin_memory=True).numpy()
            lb = torch.empty(n, dtype=torch.int64, pin_memory=True).numpy()
        else:
            tb = np.empty((n, n + 1), np.int32)
            lb = np.empty(n, np.int64)
        for _ in range(2):
            tb[:] = -7
            eng.run_iteration(tours_out=tb, lengths_out=lb)
            assert ("streams_tours_to_host" in eng.describe()) == pinned
            t, l = eng.ants()
            assert np.array_equal(tb, t)
            assert np.array_equal(lb, l)


@pytest.mark.parametrize("alpha,beta,rho", [(0.0, 2.0, 0.5), (1.0, 1.0, 0.1), (1.0, 3.0, 0.9),
                                            (1.0, 2.5, 0.25)])
def test_parameter_variants_bit_exact(aco, oracle, alpha, beta, rho):
    """alpha in {0, 1} (pow exact) with other beta (the host-libm eta^beta
    table) and rho: tours and the gather tau stay bit-exact."""
    n = 300
    prob, eng = make(aco, n, deposit=1, alpha=alpha, beta=beta, rho=rho)
    with eng:
        tau = np.full((n, n), eng.tau0)
        for it in range(3):
            ch = oracle.choice(prob.dist, tau, alpha=alpha, beta=beta)
            assert np.array_equal(eng.choice(), ch)
            eng.run_iteration()
            t_ref, l_ref, _ = oracle.construct(prob.dist, ch, 1, it, 0, n)
            assert np.array_equal(eng.ants()[0], t_ref), f"iteration {it}"
            tau = oracle.update(tau, t_ref, l_ref, rho, 1)
            assert np.array_equal(eng.pheromone(), tau)


@pytest.mark.parametrize("ewt", ["ceil_2d", "att"])
def test_edge_weight_types_bit_exact(aco, oracle, ewt):
    """CEIL_2D and ATT distances (tsplib.hpp:190-210) through the whole
    iteration: tours and the gather tau bit-exact."""
    n = 200
    base = aco.synthetic_instance(n)
    spec = aco.InstanceSpec(f"{ewt}{n}", n, getattr(aco.EdgeWeightType, ewt), base.xs, base.ys)
    prob, eng = make(aco, n, deposit=1, spec=spec)
    with eng:
        tau = np.full((n, n), eng.tau0)
        for it in range(2):
            ch = oracle.choice(prob.dist, tau)
            eng.run_iteration()
            t_ref, l_ref, _ = oracle.construct(prob.dist, ch, 1, it, 0, n)
            assert np.array_equal(eng.ants()[0], t_ref)
            tau = oracle.update(tau, t_ref, l_ref, 0.5, 1)
            assert np.array_equal(eng.pheromone(), tau)


@pytest.mark.parametrize("nn", [33, 48, 64])
def test_nn_long_lists_bit_exact(aco, oracle, nn):
    """nn lists longer than a warp (two passes of the exact fold, no fp32
    fast path): tours and the gather tau bit-exact."""
    n = 300
    prob, eng = make(aco, n, selection=1, deposit=1, nn=nn)
    with eng:
        nnl = oracle.nn_lists(prob.dist, nn)
        tau = np.full((n, n), eng.tau0)
        for it in range(2):
            ch = oracle.choice(prob.dist, tau)
            eng.run_iteration()
            t_ref, l_ref, _ = oracle.construct(prob.dist, ch, 1, it, 0, n, selection=1,
                                               nn_lists=nnl)
            assert np.array_equal(eng.ants()[0], t_ref), f"iteration {it}"
            tau = oracle.update(tau, t_ref, l_ref, 0.5, 1)
            assert np.array_equal(eng.pheromone(), tau)


@pytest.mark.parametrize("n,nn,ants", [(1002, 30, None), (3000, 8, (0, 400))])
@pytest.mark.parametrize("compact", ["1", "0"])
def test_nn_accumulate_compact_deposit_within_tolerance(aco, oracle, monkeypatch, n, nn, ants,
                                                        compact):
    """nn selection + accumulate: list edges fold into the compact n x nn
    slots (k_deposit_nn + k_apply_nn), the rest scatter into tau — tau within
    1e-5 relative of deposit_accumulate (pheromone.hpp:195-208) from a shared
    state each iteration, tours bit-exact; ACO_NN_COMPACT=0 is the plain
    scatter.  n=3000/nn=8 makes argmax fallbacks (non-list edges) frequent."""
    monkeypatch.setenv("ACO_NN_COMPACT", compact)
    prob, eng = make(aco, n, selection=1, deposit=0, nn=nn, ant_range=ants)
    k0, k1 = ants or (0, n)
    with eng:
        nnl = oracle.nn_lists(prob.dist, nn)
        tau = np.full((n, n), eng.tau0)
        for it in range(3):
            eng.set_pheromone(tau)
            ch = oracle.choice(prob.dist, tau)
            eng.run_iteration()
            t_ref, l_ref, _ = oracle.construct(prob.dist, ch, 1, it, k0, k1, selection=1,
                                               nn_lists=nnl)
            t, l = eng.ants()
            assert np.array_equal(t, t_ref), f"iteration {it}"
            tau_ref = oracle.update(tau, t_ref, l_ref, 0.5, 0)
            got = eng.pheromone()
            assert (np.abs(got - tau_ref) / np.abs(tau_ref)).max() <= ATOMIC_RTOL
            tau = tau_ref
