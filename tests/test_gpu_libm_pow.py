"""pow(tau, alpha) for alpha outside {0, 1}: the device
replay of the host glibc pow (csrc/libm_pow.cuh) is bit-identical to the
host's own pow — the function compute_choice_info calls
(/root/reference/proj/include/aco/model.hpp:167) — over the whole pheromone
domain, and an engine with alpha = 1.5 / 2 / 0.7 reproduces the reference's
choice matrix and tours bit for bit."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _device_pow(x, y):
    import ctypes as C

    from paper_1101_2678_b200 import _lib

    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(np.broadcast_to(y, x.shape), np.float64)
    out = np.zeros_like(x)
    st = _lib.lib.aco_gpu_libm_pow(0, len(x), _lib.ptr(x), _lib.ptr(y), _lib.ptr(out))
    assert st == 0, _lib.lib.aco_last_error()
    return out


def _domain(rng, k):
    """Pheromone-like x: log-uniform over every binade incl. the subnormals,
    values around 1, exact powers of two, +0."""
    e = rng.uniform(-1074.0, 40.0, k)
    x = np.exp2(e) * rng.uniform(1.0, 2.0, k)
    extra = [0.0, 1.0, np.nextafter(1.0, 2), np.nextafter(1.0, 0), 5e-324, 2.2250738585072014e-308,
             np.nextafter(2.2250738585072014e-308, 0)]
    near1 = 1.0 + rng.uniform(-1e-3, 1e-3, 4096)
    pow2 = np.exp2(np.arange(-1074, 60, dtype=np.float64))
    return np.concatenate([x, extra, near1, pow2])


@pytest.mark.parametrize("alpha", [0.5, 1.5, 2.0, 2.5, 3.0, 0.25, 0.7, 4.0, 7.3, 1e-20, 1e-300,
                                   5e18, 1e19])
def test_device_pow_bit_identical_to_host_libm(oracle, alpha):
    rng = np.random.default_rng(int(alpha * 1000) % 2**32)
    x = _domain(rng, 300_000)
    got = _device_pow(x, alpha)
    ref = oracle.pow(x, alpha)
    bad = np.flatnonzero(got.view(np.uint64) != ref.view(np.uint64))
    assert bad.size == 0, [(x[i].hex(), got[i].hex(), ref[i].hex()) for i in bad[:5]]


def test_device_pow_random_exponents(oracle):
    rng = np.random.default_rng(99)
    x = _domain(rng, 400_000)
    y = np.exp2(rng.uniform(-10.0, 4.0, x.size))
    got = _device_pow(x, y)
    ref = oracle.pow(x, y)
    bad = np.flatnonzero(got.view(np.uint64) != ref.view(np.uint64))
    assert bad.size == 0, [(x[i].hex(), y[i].hex(), got[i].hex(), ref[i].hex()) for i in bad[:5]]


@pytest.mark.parametrize("alpha,deposit", [(1.5, 1), (2.0, 1), (0.7, 0)])
def test_engine_alpha_choice_and_tours_bit_exact(oracle, alpha, deposit):
    from paper_1101_2678_b200 import aco

    n = 700
    prob = aco.build_problem(aco.synthetic_instance(n))
    cfg = aco.RunConfig(params=aco.Parameters(m=0, seed=1, alpha=alpha),
                        selection=aco.SelectionStrategy(aco.Selection.roulette_full),
                        deposit=aco.DepositStrategy(aco.Deposit(deposit)))
    with aco.Engine(prob, cfg) as eng:
        tau = np.full((n, n), eng.tau0)
        for it in range(3):
            if deposit == 0:
                eng.set_pheromone(tau)
            ch = oracle.choice(prob.dist, tau, alpha, 2.0)
            assert np.array_equal(eng.choice(), ch), f"choice at iteration {it}"
            eng.run_iteration()
            t_ref, l_ref, _ = oracle.construct(prob.dist, ch, 1, it, 0, n)
            t, _ = eng.ants()
            assert np.array_equal(t, t_ref)
            tau = oracle.update(tau, t_ref, l_ref, 0.5, deposit)
            if deposit != 0:
                assert np.array_equal(eng.pheromone(), tau)


def test_engine_alpha_wide_tau_matches_reference(reference, oracle):
    """compute_choice_info of the reference itself (oracle/_ref) on a tau
    spanning 2^-1074 .. 2^8 with alpha = 2.5."""
    from paper_1101_2678_b200 import aco

    n = 400
    prob = aco.build_problem(aco.synthetic_instance(n))
    rng = np.random.default_rng(3)
    tau = np.exp2(rng.uniform(-1074.0, 8.0, (n, n)))
    cfg = aco.RunConfig(params=aco.Parameters(m=0, seed=1, alpha=2.5),
                        selection=aco.SelectionStrategy(aco.Selection.roulette_full),
                        deposit=aco.DepositStrategy(aco.Deposit.scatter_gather))
    with aco.Engine(prob, cfg) as eng:
        eng.set_pheromone(tau)
        assert np.array_equal(eng.choice(), reference.choice(prob.dist, tau, 2.5, 2.0))
