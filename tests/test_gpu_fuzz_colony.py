"""Colony-size fuzz against the oracle: the launch variants that only large
colonies reach — the roulette relay (m a little above a multiple of the SM
count), its fused tour tail (>= 12 warps per SM), the tour stream into pinned
host memory, the nn kernel's latency-bound (early list request) and
full-occupancy variants, the in-place and fma warp scans — over random
instance sizes, colony sizes, seeds, start rules and deposits.  Tours and
lengths bit-exact; the gather tau too (construction.hpp:42-121,
pheromone.hpp:213-228).  ACO_FUZZ_CASES sets the number of cases (default 8)."""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _sms():
    import torch

    return torch.cuda.get_device_properties(0).multi_processor_count


def _cases(count):
    rng = np.random.default_rng(171020261)
    out = []
    for _ in range(count):
        sel = int(rng.choice([0, 0, 1]))
        n = int(rng.integers(150, 1300))
        q = int(rng.choice([2, 4, 8, 12, 16]))
        extra = int(rng.choice([0, 1, 3, 7, 20]))
        out.append((n, q, extra, sel, int(rng.integers(0, 2)), bool(rng.integers(0, 2)),
                    bool(rng.integers(0, 2)), int(rng.integers(1, 10_000))))
    return out


def _par_construct(oracle, dist, ch, seed, it, m, **kw):
    threads = max(1, min(os.cpu_count() or 1, 32))
    step = max(1, -(-m // (threads * 2)))
    ranges = [(a, min(m, a + step)) for a in range(0, m, step)]
    with ThreadPoolExecutor(threads) as ex:
        parts = list(ex.map(lambda r: oracle.construct(dist, ch, seed, it, r[0], r[1], **kw), ranges))
    return np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts])


@pytest.mark.parametrize("n,q,extra,sel,dep,random_start,pinned,seed",
                         _cases(int(os.environ.get("ACO_FUZZ_CASES", "8"))))
def test_fuzz_colony_bit_exact(oracle, n, q, extra, sel, dep, random_start, pinned, seed):
    import torch

    from paper_1101_2678_b200 import aco

    m = q * _sms() + extra
    nn = 30
    prob = aco.build_problem(aco.synthetic_instance(n, seed_state=seed))
    cfg = aco.RunConfig(params=aco.Parameters(m=m, seed=seed, nn=nn),
                        selection=aco.SelectionStrategy(aco.Selection(sel)),
                        deposit=aco.DepositStrategy(aco.Deposit(dep)), random_start=random_start)
    nnl = oracle.nn_lists(prob.dist, nn) if sel == 1 else None
    tb = torch.empty((m, n + 1), dtype=torch.int32, pin_memory=True).numpy() if pinned else None
    lb = torch.empty(m, dtype=torch.int64, pin_memory=True).numpy() if pinned else None
    with aco.Engine(prob, cfg) as eng:
        tau = np.full((n, n), eng.tau0)
        for it in range(2):
            if dep == 0:
                eng.set_pheromone(tau)
            ch = oracle.choice(prob.dist, tau)
            eng.run_iteration(tours_out=tb, lengths_out=lb)
            t_ref, l_ref = _par_construct(oracle, prob.dist, ch, seed, it, m, selection=sel, nn_lists=nnl,
                                          random_start=random_start)
            t, l = eng.ants()
            assert np.array_equal(t, t_ref), f"tours differ at iteration {it} ({eng.describe()})"
            assert np.array_equal(l, l_ref)
            if pinned:
                assert np.array_equal(tb, t_ref) and np.array_equal(lb, l_ref)
            tau_ref = oracle.update(tau, t_ref, l_ref, 0.5, dep)
            if dep:
                assert np.array_equal(eng.pheromone(), tau_ref)
            tau = tau_ref
