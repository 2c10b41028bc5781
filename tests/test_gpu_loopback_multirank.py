"""The engine's multi-rank protocol (world = 2, 3, 4, 8) executed for real on
ONE GPU: G engine contexts in G threads of one process, the collectives served
by the in-process loopback NCCL (tests/loopnccl/loopnccl.cu, loaded through
ACO_NCCL_LIB; real NCCL refuses two ranks on one device).  This runs the
code that otherwise only an 8-GPU node would: ncclCommInitRank with
world > 1, the statistics key MIN / SUM all-reduces and the winning tour's MAX
replication, the delta all-reduce on the fp64 / fp32 / fixed64 wires, the
row-sharded gather (succ/pred row blocks by send/recv, the delta rows
all-gathered), the nn fixed-point slot all-reduce + record all-gather, and the
MULTIMEM setup's cross-rank agreement and its FIXED64 fallback.  Every rank
must agree with the single-context colony: tours, lengths, statistics and
best tour identical; tau bit-identical on the gather and fixed-point paths,
within 1e-12 (fp64 wire: only the add order differs) or 1e-5 (fp32 wire).

Matches /root/reference/proj/include/aco/engine.hpp:98-129 (the ant fork the
sharding splits), :151-154 (best-so-far), pheromone.hpp:195-228 (deposits)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "loopnccl", "loopnccl.cu")
LIB = os.path.join(ROOT, "tests", "loopnccl", "_build", "libloopnccl.so")


@pytest.fixture(scope="module")
def loopnccl():
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        os.makedirs(os.path.dirname(LIB), exist_ok=True)
        subprocess.run(["nvcc", "-O2", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
                        "-shared", "-Xcompiler", "-fPIC", SRC, "-o", LIB], check=True)
    return LIB


def run(lib, tmp_path, G, deposit, wire, n=400, iters=4, sel=0):
    out = str(tmp_path / f"g{G}_d{deposit}_w{wire}_s{sel}.json")
    env = dict(os.environ, ACO_NCCL_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "_loopback_worker.py"), out, str(G),
                        str(deposit), str(wire), str(n), str(iters), str(sel)],
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    with open(out) as f:
        return json.load(f)


def check(rep, deposit, wire):
    for it, r in enumerate(rep["iterations"]):
        assert r["tau_identical_across_ranks"], f"ranks disagree on tau at iteration {it}"
        assert r["choice_identical_across_ranks"], f"ranks disagree on choice at iteration {it}"
        if wire == 1 and it > 0:
            # fp32 wire: one 2^-24 rounding per delta and iteration — the
            # trajectory may leave the single-GPU colony's after iteration 0
            assert r["tau_max_rel"] <= 1e-5 or not r["tours_equal"]
            continue
        assert r["tours_equal"] and r["lengths_equal"], f"tours differ at iteration {it}"
        assert r["best_equal"] and r["mean_equal"] and r["best_so_far_equal"], it
        assert r["best_tour_equal"], it
        if deposit != 0 or wire in (2, 3):
            assert r["tau_bit_equal_single"], f"tau differs from one GPU at iteration {it}"
        else:
            assert r["tau_max_rel"] <= (1e-12 if wire == 0 else 1e-5), (it, r["tau_max_rel"])


@pytest.mark.parametrize("G", [2, 3, 8])
@pytest.mark.parametrize("deposit,wire", [(1, 0), (0, 0), (0, 1), (0, 2)])
def test_loopback_sharded_engine_matches_single_gpu(loopnccl, tmp_path, G, deposit, wire):
    rep = run(loopnccl, tmp_path, G, deposit, wire)
    assert rep["world"] == G
    check(rep, deposit, wire)


def test_loopback_row_sharded_gather_uneven_blocks(loopnccl, tmp_path):
    """n = 401 over 4 ranks: row blocks of 101, 101, 101, 98 (the last padded)."""
    rep = run(loopnccl, tmp_path, 4, 1, 0, n=401)
    check(rep, 1, 0)


def test_loopback_multimem_agrees_and_falls_back(loopnccl, tmp_path):
    """MULTIMEM on one device: the multicast object cannot be built, every
    rank agrees (MIN all-reduces), and the FIXED64 all-reduce of the same
    integers runs — tau bit-identical with the single-context colony."""
    rep = run(loopnccl, tmp_path, 2, 0, 3)
    assert "multicast unavailable" in rep["describe"] or "multimem" in rep["describe"]
    check(rep, 0, 3)


@pytest.mark.parametrize("wire", [0, 2])
def test_loopback_nn_selection_sharded(loopnccl, tmp_path, wire):
    """nn selection (nn = 8: frequent argmax fallbacks): fp64 delta
    all-reduce, or on the fixed64 wire the compact slots + record exchange."""
    rep = run(loopnccl, tmp_path, 4, 0, wire, sel=1)
    check(rep, 0, wire)
