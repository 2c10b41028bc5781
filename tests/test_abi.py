"""The C-ABI library (libaco_gpu.so): loads, exports every symbol
include/aco_gpu.h declares, and its host-side model (TSPLIB parsing, edge
weights, nn lists, greedy tau0, tour_length, ledger) matches the reference's
values AND error codes.  No device work here (the CPU suite runs without a
GPU); on a CPU-only machine engine creation must fail loudly."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from pyoracle import synth_coords

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def aco():
    from paper_1101_2678_b200 import aco as _aco

    return _aco


def header_functions():
    text = open(os.path.join(ROOT, "include", "aco_gpu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(aco_\w+)\s*\(", text)))


def test_exports_every_declared_symbol():
    from paper_1101_2678_b200 import _lib

    declared = header_functions()
    assert len(declared) >= 25
    assert sorted(_lib.EXPORTS) == declared
    for name in declared:
        assert hasattr(_lib.lib, name), name
    out = os.popen(f"nm -D --defined-only {_lib.LIB_PATH}").read()
    for name in declared:
        assert re.search(rf"\bT {name}$", out, re.M), name


def test_library_is_sm100a_only():
    from paper_1101_2678_b200 import _lib

    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_parse_instance_matches_reference(aco, reference, golden):
    text = "NAME: t\nTYPE: TSP\nDIMENSION: 4\nEDGE_WEIGHT_TYPE: ATT\nNODE_COORD_SECTION\n" \
           "1 0 0\n2 3 4\n 3 10.5 -2\r\n4 1e3 7\nEOF\n"
    spec = aco.parse_instance(text)
    xs, ys, ewt = reference.parse_instance(text)
    assert spec.name == "t" and spec.dimension == 4 and int(spec.edge_weight_type) == ewt == 2
    assert np.array_equal(spec.xs, xs) and np.array_equal(spec.ys, ys)


BAD = [
    ("NAME: x\nDIMENSION: 3\nEDGE_WEIGHT_TYPE: EUC_2D\n", "missing_field"),
    ("NAME: x\nEDGE_WEIGHT_TYPE: EUC_2D\nNODE_COORD_SECTION\n1 0 0\n", "missing_field"),
    ("NAME: x\nDIMENSION: 2\nEDGE_WEIGHT_TYPE: GEO\nNODE_COORD_SECTION\n1 0 0\n2 1 1\n",
     "unsupported_edge_weight_type"),
    ("NAME: x\nDIMENSION: 2\nEDGE_WEIGHT_TYPE: EUC_2D\nNODE_COORD_SECTION\n1 0 0\n2 1\n",
     "malformed_coord"),
    ("NAME: x\nDIMENSION: 2\nEDGE_WEIGHT_TYPE: EUC_2D\nNODE_COORD_SECTION\n1 0 0\n1 1 1\n",
     "malformed_coord"),
    ("NAME: x\nDIMENSION: 2\nEDGE_WEIGHT_TYPE: EUC_2D\nNODE_COORD_SECTION\n1 0 0\n3 1 1\n",
     "malformed_coord"),
    ("NAME: x\nDIMENSION: 3\nEDGE_WEIGHT_TYPE: EUC_2D\nNODE_COORD_SECTION\n1 0 0\n2 1 1\nEOF\n",
     "dimension_mismatch"),
    ("NAME: x\nDIMENSION: 2\nEDGE_WEIGHT_TYPE: EUC_2D\nNODE_COORD_SECTION\n1 0 0\n2 1 1\n3 2 2\n",
     "dimension_mismatch"),
    ("NAME: x\nDIMENSION: 1\nEDGE_WEIGHT_TYPE: EUC_2D\n", "dimension_mismatch"),
    ("NAME: x\nDIMENSION: two\n", "missing_field"),
    ("NAME: x\nDIMENSION: 2\nEDGE_WEIGHT_SECTION\n", "unsupported_edge_weight_type"),
]


@pytest.mark.parametrize("text,code", BAD)
def test_parse_errors_match_reference(aco, reference, text, code):
    with pytest.raises(aco.Error) as ei:
        aco.parse_instance(text)
    assert ei.value.code == aco.Errc[code]
    with pytest.raises(RuntimeError) as er:
        reference.parse_instance(text)
    assert f"rc={1 + int(aco.Errc[code])}" in str(er.value)


def test_load_instance_io_error(aco):
    with pytest.raises(aco.Error) as ei:
        aco.load_instance("/nonexistent/file.tsp")
    assert ei.value.code == aco.Errc.io_error


def test_att48_via_abi(aco, oracle, golden):
    g = golden["att48"]
    spec = aco.InstanceSpec("att48", 48, aco.EdgeWeightType.att, np.array(g["xs"]),
                            np.array(g["ys"]))
    prob = aco.build_problem(spec)
    assert np.array_equal(prob.dist, oracle.build_dist(spec.xs, spec.ys, 2))
    tour = g["opt_tour"] + [g["opt_tour"][0]]
    assert aco.tour_length(prob, tour) == 10628
    assert repr(aco.initial_pheromone(prob, 48)) == g["tau0"]
    text = "NAME : att48.opt.tour\nTYPE : TOUR\nDIMENSION : 48\nTOUR_SECTION\n" + \
        "\n".join(str(c + 1) for c in g["opt_tour"]) + "\n-1\nEOF\n"
    assert aco.parse_tour(text).tolist() == g["opt_tour"]


@pytest.mark.parametrize("ewt", [0, 1, 2])
def test_build_problem_nn_greedy_match_oracle(aco, oracle, reference, ewt):
    n = 300
    xs, ys = synth_coords(n, state=11)
    xs = xs * 0.37  # non-integer coordinates exercise sqrt/ceil/nint rounding
    spec = aco.InstanceSpec("s", n, aco.EdgeWeightType(ewt), xs, ys)
    prob = aco.build_problem(spec)
    assert np.array_equal(prob.dist, oracle.build_dist(xs, ys, ewt))
    assert np.array_equal(prob.dist, reference.build_problem(xs, ys, ewt))
    assert np.array_equal(aco.build_nn_lists(prob, 30), reference.nn_lists(prob.dist, 30))
    assert aco.greedy_nn_tour_length(prob) == oracle.greedy(prob.dist)
    assert aco.initial_pheromone(prob, n) == reference.tau0(prob.dist, n)


def test_tour_length_errors(aco):
    xs, ys = synth_coords(10)
    prob = aco.build_problem(aco.InstanceSpec("s", 10, aco.EdgeWeightType.euc_2d, xs, ys))
    good = list(range(10)) + [0]
    assert aco.tour_length(prob, good) > 0
    for bad, code in [(good[:-1], "not_closed"), (list(range(10)) + [1], "not_closed"),
                      ([0, 1, 1, 3, 4, 5, 6, 7, 8, 9, 0], "not_a_permutation"),
                      ([0, 1, 2, 3, 4, 5, 6, 7, 8, 12, 0], "not_a_permutation")]:
        with pytest.raises(aco.Error) as ei:
            aco.tour_length(prob, bad)
        assert ei.value.code == aco.Errc[code]
    with pytest.raises(aco.Error) as ei:
        aco.build_nn_lists(prob, 10)
    assert ei.value.code == aco.Errc.invalid_length


@pytest.mark.parametrize("dep", [0, 1, 2, 3])
def test_predicted_access_cost_matches_reference(aco, reference, dep):
    for n, m, th in [(10, 10, 64), (198, 198, 64), (2392, 2392, 64), (2392, 19136, 32)]:
        got = aco.predicted_access_cost(aco.DepositStrategy(aco.Deposit(dep)), n, m, th)
        ref = reference.predicted_access_cost(dep, n, m, th)
        assert [got.global_loads, got.global_stores, got.shared_loads, got.atomic_ops] == \
            ref.tolist()
    # SPEC.md closed forms, n = m = 10, theta = 64 (atomic 200 ops, sg 20000 loads)
    if dep == 0:
        assert aco.predicted_access_cost(aco.DepositStrategy(aco.Deposit(0)), 10, 10, 64).atomic_ops == 200
    if dep == 1:
        assert aco.predicted_access_cost(aco.DepositStrategy(aco.Deposit(1)), 10, 10,
                                         64).global_loads == 20000


def test_engine_config_errors_before_device(aco):
    """Parameter validation (model.hpp:39-53) is reported as config_error."""
    xs, ys = synth_coords(20)
    prob = aco.build_problem(aco.InstanceSpec("s", 20, aco.EdgeWeightType.euc_2d, xs, ys))
    for params, sel in [(aco.Parameters(rho=0.0), 0), (aco.Parameters(rho=1.5), 0),
                        (aco.Parameters(alpha=-1.0), 0), (aco.Parameters(m=-1), 0),
                        (aco.Parameters(tile_size=0), 0), (aco.Parameters(nn=20), 1),
                        (aco.Parameters(iterations=0), 0)]:
        cfg = aco.RunConfig(params=params, selection=aco.SelectionStrategy(aco.Selection(sel)))
        with pytest.raises(aco.Error) as ei:
            aco.Engine(prob, cfg)
        assert ei.value.code == aco.Errc.config_error


def test_no_cpu_fallback_without_gpu(aco):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    xs, ys = synth_coords(64)
    prob = aco.build_problem(aco.InstanceSpec("s", 64, aco.EdgeWeightType.euc_2d, xs, ys))
    with pytest.raises(aco.Error) as ei:
        aco.Engine(prob, aco.RunConfig())
    assert ei.value.code == 100  # ACO_E_CUDA: fails loudly, never computes on the host


def test_host_uniform_at_matches_oracle(oracle, golden):
    from paper_1101_2678_b200 import _lib

    for seed, it, ant, st, dr, val in golden["uniform_at"][:8]:
        assert _lib.lib.aco_uniform_at(seed, it, ant, st, dr) == float(val)
    rng = np.random.default_rng(11)
    for _ in range(500):
        seed = int(rng.integers(0, 2**63))
        args = [int(x) for x in rng.integers(0, 2**32, 4)]
        assert _lib.lib.aco_uniform_at(seed, *args) == oracle.uniform_at(seed, *args)


@pytest.mark.parametrize("kw,msg", [
    (dict(rho=0.0), "rho must be in (0,1]"), (dict(rho=1.5), "rho must be in (0,1]"),
    (dict(alpha=-1.0), "alpha and beta must be >= 0"), (dict(m=-1), "ant count must be >= 1"),
    (dict(iterations=0), "iterations must be >= 1"), (dict(tile_size=0), "tile size must be >= 1"),
    (dict(nn=10, nn_selected=1), "nn must satisfy 1 <= nn < n (n=10)"),
])
def test_validate_parameters_reference_messages(kw, msg):
    """Parameters::validate (model.hpp:39-53): same checks, order and text."""
    from paper_1101_2678_b200 import _lib

    a = dict(alpha=1.0, beta=2.0, rho=0.5, m=0, nn=30, iterations=10, tile_size=64, n=10,
             nn_selected=0)
    a.update(kw)
    st = _lib.lib.aco_validate_parameters(a["alpha"], a["beta"], a["rho"], a["m"], a["nn"],
                                          a["iterations"], a["tile_size"], a["n"],
                                          a["nn_selected"])
    assert st == 13  # 1 + Errc::config_error
    assert _lib.lib.aco_last_error().decode() == msg
    a.update(rho=0.5, alpha=1.0, m=0, iterations=10, tile_size=64, nn=5)
    assert _lib.lib.aco_validate_parameters(a["alpha"], a["beta"], a["rho"], a["m"], a["nn"],
                                            a["iterations"], a["tile_size"], a["n"],
                                            a["nn_selected"]) == 0
