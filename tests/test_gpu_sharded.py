"""The ant-sharded device path on ONE GPU: G contexts in external-exchange
mode (world = G, zero NCCL id) each construct their ant shard; the test
performs the all-gather / all-reduce the engine would run over NCCL, then
every context updates.  Tours must equal the single-context colony
bit-for-bit, the gather-path tau must be bit-identical on every shard, and
the atomic-path tau must agree within 1e-5 (the order of the Δτ reduction
differs)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


class DevArray:
    """__cuda_array_interface__ view of a raw device pointer (for torch.as_tensor)."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3}


def _engines(aco, n, m, deposit, G):
    spec = aco.synthetic_instance(n)
    prob = aco.build_problem(spec)

    def cfg(world=1, rank=0):
        return aco.RunConfig(params=aco.Parameters(m=m, seed=3),
                             selection=aco.SelectionStrategy(aco.Selection.roulette_full),
                             deposit=aco.DepositStrategy(aco.Deposit(deposit)),
                             world=world, rank=rank)

    single = aco.Engine(prob, cfg())
    shards = [aco.Engine(prob, cfg(G, r)) for r in range(G)]
    return prob, single, shards


@pytest.mark.parametrize("deposit", [1, 0])
@pytest.mark.parametrize("G,m", [(2, 300), (3, 301)])
def test_virtual_shards_match_single_context(deposit, G, m):
    import torch

    from paper_1101_2678_b200 import aco

    n = 300
    prob, single, shards = _engines(aco, n, m, deposit, G)
    bufs = [e.exchange_buffers() for e in shards]
    S = bufs[0]["S"]
    P64 = bufs[0]["P64"]
    for it in range(3):
        single.run_iteration()
        t_ref, l_ref = single.ants()
        for e in shards:
            e.construct()
        torch.cuda.synchronize()
        got = np.concatenate([e.ants()[0] for e in shards])
        assert np.array_equal(got, t_ref), f"tours differ at iteration {it}"
        if deposit != 0:  # all-gather the shard blocks (succ, pred, 1/C_k)
            blk = n * S
            for name, typ, width in (("succ", "<i4", blk), ("pred", "<i4", blk), ("inv", "<f8", S)):
                views = [torch.as_tensor(DevArray(b[name], (G * width,), typ), device="cuda")
                         for b in bufs]
                for r in range(G):
                    src = views[r][r * width:(r + 1) * width]
                    for q in range(G):
                        if q != r:
                            views[q][r * width:(r + 1) * width].copy_(src)
        else:  # all-reduce the local deltas
            views = [torch.as_tensor(DevArray(b["delta"], (n * P64,), "<f8"), device="cuda")
                     for b in bufs]
            total = torch.zeros_like(views[0])
            for v in views:
                total += v
            for v in views:
                v.copy_(total)
        torch.cuda.synchronize()
        for e in shards:
            e.update()
        tau_ref = single.pheromone()
        for e in shards:
            tau = e.pheromone()
            if deposit != 0:
                assert np.array_equal(tau, tau_ref), "gather tau must be bit-identical"
            else:
                assert np.max(np.abs(tau - tau_ref) / np.abs(tau_ref)) <= 1e-5
            if deposit != 0:
                assert np.array_equal(e.choice(), single.choice())
        if deposit == 0:  # keep the colonies on the same trajectory
            for e in shards:
                e.set_pheromone(tau_ref)
    for e in shards + [single]:
        e.close()


@pytest.mark.parametrize("G,n,m", [(2, 300, 300), (3, 301, 301), (8, 300, 2400)])
def test_row_sharded_gather_fold_bit_exact(G, n, m):
    """The row-sharded gather deposit: shard r folds only
    rows [r*B, r*B+B) of the ordered deposit into delta rows (aco_gpu_fold),
    the delta row blocks are all-gathered (here by the test), and every shard
    applies them (aco_gpu_update) — tau and choice bit-identical with the
    single-context colony on every shard (pheromone.hpp:213-228)."""
    import torch

    from paper_1101_2678_b200 import aco

    prob, single, shards = _engines(aco, n, m, 1, G)
    bufs = [e.exchange_buffers() for e in shards]
    S, P64 = bufs[0]["S"], bufs[0]["P64"]
    B = -(-n // G)
    for it in range(3):
        single.run_iteration()
        for e in shards:
            e.construct()
        torch.cuda.synchronize()
        # every shard's succ/pred rows of shard q's block go to shard q
        for name in ("succ", "pred"):
            views = [torch.as_tensor(DevArray(b[name], (G, n, S), "<i4"), device="cuda") for b in bufs]
            for g in range(G):
                for q in range(G):
                    if q != g:
                        views[q][g, q * B:min(n, (q + 1) * B)].copy_(views[g][g, q * B:min(n, (q + 1) * B)])
        views = [torch.as_tensor(DevArray(b["inv"], (G * S,), "<f8"), device="cuda") for b in bufs]
        for g in range(G):
            for q in range(G):
                if q != g:
                    views[q][g * S:(g + 1) * S].copy_(views[g][g * S:(g + 1) * S])
        torch.cuda.synchronize()
        assert all(e.fold() == B for e in shards)
        deltas = [torch.as_tensor(DevArray(b["delta"], (G * B, P64), "<f8"), device="cuda") for b in bufs]
        for g in range(G):
            for q in range(G):
                if q != g:
                    deltas[q][g * B:(g + 1) * B].copy_(deltas[g][g * B:(g + 1) * B])
        torch.cuda.synchronize()
        for e in shards:
            e.update()
        tau_ref, ch_ref = single.pheromone(), single.choice()
        for e in shards:
            assert np.array_equal(e.pheromone(), tau_ref), f"tau differs at iteration {it}"
            assert np.array_equal(e.choice(), ch_ref)
        got = np.concatenate([e.ants()[0] for e in shards])
        assert np.array_equal(got, single.ants()[0])
    for e in shards + [single]:
        e.close()


@pytest.mark.parametrize("deposit,wire", [(1, 0), (0, 0), (0, 1)])
def test_nccl_exchange_path_one_rank(deposit, wire):
    """The NCCL exchange path (all-gather of succ/pred/1/C_k, or all-reduce of
    the local delta + k_rows<DELTA/DELTA32>; NCCL reduction of the statistics
    and broadcast of the best tour) on a one-rank communicator: tours, best
    tour and statistics equal the unsharded engine's; tau bit-exact on the
    gather path.  Accumulate over the default fp64 wire: a free-running
    multi-iteration trajectory (no pheromone reset) stays on the unsharded
    colony's tours with tau within 1e-12 relative (the two differ only in the
    order of the fp64 adds).  The opt-in fp32 wire rounds every delta once
    (<= 1e-5 relative per iteration), so its trajectory is resynchronised."""
    from paper_1101_2678_b200 import aco

    n = 300
    prob = aco.build_problem(aco.synthetic_instance(n))

    def cfg(nccl_id=None):
        return aco.RunConfig(params=aco.Parameters(m=0, seed=2),
                             selection=aco.SelectionStrategy(aco.Selection.roulette_full),
                             deposit=aco.DepositStrategy(aco.Deposit(deposit)), nccl_id=nccl_id,
                             wire=aco.Wire(wire))

    plain = aco.Engine(prob, cfg())
    nccl = aco.Engine(prob, cfg(aco.nccl_unique_id()))
    for it in range(6):
        ra = plain.run_iteration()
        rb = nccl.run_iteration()
        ta, la = plain.ants()
        tb, lb = nccl.ants()
        assert np.array_equal(ta, tb), f"tours differ at iteration {it}"
        assert ra.best_length == rb.best_length and ra.mean_length == rb.mean_length
        assert plain.best_length() == nccl.best_length()
        assert np.array_equal(plain.best_tour(), nccl.best_tour())
        pa, pb = plain.pheromone(), nccl.pheromone()
        if deposit != 0:
            assert np.array_equal(pa, pb)
        elif wire == 0:
            assert (np.abs(pa - pb) / pa).max() <= 1e-12
        else:
            assert (np.abs(pa - pb) / pa).max() <= 1e-5
            nccl.set_pheromone(pa)  # fp32 wire: keep the construction inputs identical
    plain.close()
    nccl.close()


@pytest.mark.parametrize("wire,selection", [(2, 0), (3, 0), (2, 1), (3, 1)])
def test_fixed_point_exchange_bit_identical_for_any_world(wire, selection):
    """ACO_WIRE_FIXED64 / MULTIMEM: every deposit is an exact int64
    fixed-point sum, so tau does not depend on the order of the reds or on
    the exchange.  The sharded protocol on a one-rank NCCL communicator
    (ncclUint64 all-reduce; MULTIMEM at world 1 runs the same FIXED64 path —
    its multicast object needs >= 2 GPUs) reproduces the single-context
    fixed-point colony BIT FOR BIT over a free-running trajectory, and two
    single-context runs agree bit for bit (the fp64 atomic path does not).
    nn selection (nn = 8: frequent argmax fallbacks) runs the compact-slot +
    record exchange (count all-gather, record all-gather, slot all-reduce)."""
    from paper_1101_2678_b200 import aco

    n = 500
    prob = aco.build_problem(aco.synthetic_instance(n))

    def cfg(nccl_id=None, w=wire):
        return aco.RunConfig(params=aco.Parameters(m=0, seed=5, nn=8),
                             selection=aco.SelectionStrategy(aco.Selection(selection)),
                             deposit=aco.DepositStrategy(aco.Deposit.accumulate), nccl_id=nccl_id,
                             wire=aco.Wire(w))

    a = aco.Engine(prob, cfg())
    b = aco.Engine(prob, cfg())
    c = aco.Engine(prob, cfg(aco.nccl_unique_id()))
    for it in range(6):
        ra, rb, rc = a.run_iteration(), b.run_iteration(), c.run_iteration()
        ta, _ = a.ants()
        assert np.array_equal(ta, b.ants()[0]) and np.array_equal(ta, c.ants()[0]), it
        assert ra.best_length == rb.best_length == rc.best_length
        assert ra.mean_length == rc.mean_length
        pa = a.pheromone()
        assert np.array_equal(pa, b.pheromone()), f"run-to-run tau differs at {it}"
        assert np.array_equal(pa, c.pheromone()), f"sharded tau differs at {it}"
        assert np.array_equal(a.choice(), c.choice())
    for e in (a, b, c):
        e.close()


@pytest.mark.parametrize("selection", [0, 1])
def test_fixed_point_deposit_within_tolerance_of_reference(oracle, selection):
    """The fixed-point accumulate against deposit_accumulate
    (pheromone.hpp:195-208) from a shared state: within 1e-5 relative
    (measured ~1e-15), tours bit-exact; nn selection through the compact
    slots + records."""
    from paper_1101_2678_b200 import aco

    n = 1002
    prob = aco.build_problem(aco.synthetic_instance(n))
    nnl = oracle.nn_lists(prob.dist, 10)
    cfg = aco.RunConfig(params=aco.Parameters(m=0, seed=1, nn=10),
                        selection=aco.SelectionStrategy(aco.Selection(selection)),
                        deposit=aco.DepositStrategy(aco.Deposit.accumulate), wire=aco.Wire.fixed64)
    with aco.Engine(prob, cfg) as eng:
        tau = np.full((n, n), eng.tau0)
        worst = 0.0
        for it in range(3):
            eng.set_pheromone(tau)
            ch = oracle.choice(prob.dist, tau)
            eng.run_iteration()
            t_ref, l_ref, _ = oracle.construct(prob.dist, ch, 1, it, 0, n, selection=selection,
                                               nn_lists=nnl if selection else None)
            assert np.array_equal(eng.ants()[0], t_ref)
            tau_ref = oracle.update(tau, t_ref, l_ref, 0.5, 0)
            rel = float((np.abs(eng.pheromone() - tau_ref) / np.abs(tau_ref)).max())
            worst = max(worst, rel)
            tau = tau_ref
        assert worst <= 1e-12


def test_multimem_setup_agrees_and_falls_back(monkeypatch):
    """MULTIMEM (f2) where the NVLS multicast object cannot be created — here a
    one-rank communicator, which cuMulticastCreate refuses — every rank agrees
    (MIN all-reduce per setup step), nothing is left allocated, and the
    engine runs the FIXED64 all-reduce of the same exact int64 sums: tau is
    bit-identical with the fixed64 wire and describe() says which exchange
    ran (pheromone.hpp:195-208)."""
    from paper_1101_2678_b200 import aco

    monkeypatch.setenv("ACO_MC_ONE_RANK", "1")
    n = 300
    prob = aco.build_problem(aco.synthetic_instance(n))

    def eng(wire):
        return aco.Engine(prob, aco.RunConfig(
            params=aco.Parameters(m=0, seed=7),
            selection=aco.SelectionStrategy(aco.Selection.roulette_full),
            deposit=aco.DepositStrategy(aco.Deposit.accumulate),
            nccl_id=aco.nccl_unique_id(), wire=aco.Wire(wire)))

    a, b = eng(3), eng(2)
    assert "multicast unavailable" in a.describe()
    for _ in range(3):
        a.run_iteration()
        b.run_iteration()
        assert np.array_equal(a.ants()[0], b.ants()[0])
        assert np.array_equal(a.pheromone(), b.pheromone())
    a.close()
    b.close()
