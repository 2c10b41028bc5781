"""The C++ drop-in (include/aco_gpu.hpp via tools/acotsp_gpu.cpp): compiles
here against the header, and on the GPU reproduces the reference's own
golden traces through the C++ API."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1101_2678_b200", "acotsp_gpu")


def build_cli():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_1101_2678_b200", "csrc"),
                    "../acotsp_gpu"], check=True)
    return CLI


def test_cpp_wrapper_compiles_and_fails_loudly_without_gpu():
    import torch

    cli = build_cli()
    assert os.path.exists(cli)
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    r = subprocess.run([cli, "synth:50", "2"], capture_output=True, text=True)
    assert r.returncode == 1 and "cuda" in r.stderr.lower()


def test_cpp_wrapper_io_error_exit_code():
    cli = build_cli()
    r = subprocess.run([cli, "/nonexistent.tsp"], capture_output=True, text=True)
    assert r.returncode == 2  # acotsp.cpp:44-55: io_error -> exit 2


@pytest.mark.gpu
@pytest.mark.parametrize("deposit,idx", [("scatter-gather", 1), ("symmetric-reduction", 1),
                                         ("accumulate", 0)])
def test_cpp_wrapper_golden_trace(golden, deposit, idx):
    cli = build_cli()
    r = subprocess.run([cli, "synth:198", "10", "roulette", deposit], capture_output=True,
                       text=True, check=True)
    best = [int(l.split()[3]) for l in r.stdout.splitlines() if l.startswith("iter")]
    assert best == golden["synth198"]["traces"][idx]["best"]
