"""Source compatibility of the C++ drop-in:
the reference's own CLI bodies — make_config, cmd_solve, cmd_bench,
cmd_verify from /root/reference/proj/tools/acotsp.cpp:24-236, extracted
unchanged minus the CLI11 wiring (tests/cpp/build_dropin.py) — compile
against include/aco/*.hpp (-> include/aco_gpu.hpp) and, on the GPU,
reproduce the reference's own RunReport JSON / bench CSV golden outputs
(tests/golden/report_synth198_dep*.{json,csv}, written by the reference's
report.hpp) and its verify verdict."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_1101_2678_b200", "acotsp_dropin")
GOLDEN = os.path.join(ROOT, "tests", "golden")


def _binary():
    if os.path.exists("/root/reference/proj/tools/acotsp.cpp"):
        sys.path.insert(0, os.path.join(ROOT, "tests", "cpp"))
        import build_dropin

        return build_dropin.build()
    if not os.path.exists(BIN):
        pytest.skip("reference sources absent and acotsp_dropin not prebuilt")
    return BIN


def _synth198(tmp_path):
    from paper_1101_2678_b200 import aco

    spec = aco.synthetic_instance(198)
    text = "NAME : synth198\nTYPE : TSP\nDIMENSION : 198\nEDGE_WEIGHT_TYPE : EUC_2D\n" \
           "NODE_COORD_SECTION\n" + "".join(f"{i + 1} {int(x)} {int(y)}\n" for i, (x, y) in
                                            enumerate(zip(spec.xs, spec.ys))) + "EOF\n"
    p = tmp_path / "synth198.tsp"
    p.write_text(text)
    return str(p)


def test_reference_cli_bodies_compile_and_map_errors(tmp_path):
    cli = _binary()
    r = subprocess.run([cli, "solve", str(tmp_path / "missing.tsp"), "", "roulette",
                        "accumulate", "3"], capture_output=True, text=True)
    assert r.returncode == 2 and "cannot open file" in r.stderr  # io_error -> exit 2
    bad = tmp_path / "bad.tsp"
    bad.write_text("NAME: x\nDIMENSION: 3\n")
    r = subprocess.run([cli, "solve", str(bad), "", "roulette", "accumulate", "3"],
                       capture_output=True, text=True)
    assert r.returncode == 2  # missing_field -> exit 2
    r = subprocess.run([cli, "solve", _synth198(tmp_path), "", "bogus", "accumulate", "3"],
                       capture_output=True, text=True)
    assert r.returncode == 1 and "unknown selection" in r.stderr  # config_error -> exit 1


def test_dropin_fails_loudly_without_gpu(tmp_path):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    cli = _binary()
    r = subprocess.run([cli, "solve", _synth198(tmp_path), "", "roulette", "accumulate", "2"],
                       capture_output=True, text=True)
    assert r.returncode == 1 and "cuda" in r.stderr.lower()


def _strip_times(rep):
    for it in rep["per_iteration"]:
        it.pop("construct_ms"), it.pop("update_ms")
    return rep


@pytest.mark.gpu
@pytest.mark.parametrize("deposit,name", [(1, "scatter-gather"), (3, "symmetric-reduction")])
def test_reference_cmd_solve_reproduces_golden_report(tmp_path, deposit, name):
    cli = _binary()
    out = tmp_path / "r.json"
    r = subprocess.run([cli, "solve", _synth198(tmp_path), str(out), "roulette", name, "6", "1"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "best length 210992" in r.stdout
    mine = _strip_times(json.loads(out.read_text()))
    ref = _strip_times(json.load(open(os.path.join(GOLDEN, f"report_synth198_dep{deposit}.json"))))
    assert mine == ref


@pytest.mark.gpu
def test_reference_cmd_bench_rows_match_golden_csv(tmp_path):
    cli = _binary()
    out = tmp_path / "b.csv"
    r = subprocess.run([cli, "bench", _synth198(tmp_path), str(out), "roulette",
                        "scatter-gather", "6", "1"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    mine = out.read_text().strip().splitlines()
    ref = open(os.path.join(GOLDEN, "report_synth198_dep1.csv")).read().strip().splitlines()
    assert mine[0] == ref[0] and len(mine) == len(ref)
    for a, b in zip(mine[1:], ref[1:]):
        a, b = a.split(","), b.split(",")
        assert a[:7] + a[9:] == b[:7] + b[9:]  # all but construct_ms / update_ms


@pytest.mark.gpu
@pytest.mark.parametrize("selection", ["roulette", "nn"])
def test_reference_cmd_verify_passes(tmp_path, selection):
    cli = _binary()
    r = subprocess.run([cli, "verify", _synth198(tmp_path), selection], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all strategy pairs agree within 1e-9" in r.stdout
    assert r.stdout.count("PASS") == 4 + 6
