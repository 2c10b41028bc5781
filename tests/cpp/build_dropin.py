"""Compile the reference's own CLI bodies (acotsp.cpp: parse_selection,
parse_deposit, exit_code_for, CommonFlags, make_config, cmd_solve, cmd_bench,
cmd_verify — everything but the CLI11 option wiring and main) UNCHANGED
against the B200 drop-in headers (include/aco/*.hpp -> include/aco_gpu.hpp)
and libaco_gpu.so.  The extracted source goes to a git-ignored build
directory, never into the repo; the binary lands next to libaco_gpu.so
(paper_1101_2678_b200/acotsp_dropin, rpath $ORIGIN) so it travels to the GPU
box with the other built artefacts.

    python tests/cpp/build_dropin.py        # needs /root/reference
"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF = "/root/reference/proj/tools/acotsp.cpp"
PKG = os.path.join(ROOT, "paper_1101_2678_b200")
BUILD = os.path.join(PKG, "_dropin")
BIN = os.path.join(PKG, "acotsp_dropin")


def extract(text: str) -> str:
    """acotsp.cpp minus `#include "CLI11.hpp"`, minus add_common_flags (CLI11
    types) and minus main (CLI11); every other line verbatim."""
    lines = text.splitlines()
    out, skip = [], False
    for ln in lines:
        if ln.startswith('#include "CLI11.hpp"'):
            continue
        if ln.startswith("void add_common_flags("):
            skip = True
        if ln.startswith("int main("):
            break
        if not skip:
            out.append(ln)
        elif ln == "}":
            skip = False
    src = "\n".join(out) + "\n"
    assert "aco::RunConfig make_config(" in src and "int cmd_solve(" in src
    assert "CLI::" not in src, "CLI11 usage left in the extracted bodies"
    return src


def build() -> str:
    with open(REF) as f:
        body = extract(f.read())
    with open(os.path.join(ROOT, "tests", "cpp", "dropin_main.inc")) as f:
        main = f.read()
    os.makedirs(BUILD, exist_ok=True)
    src = os.path.join(BUILD, "acotsp_dropin.cpp")
    with open(src, "w") as f:
        f.write("// GENERATED from " + REF + " by tests/cpp/build_dropin.py — do not commit\n")
        f.write(body + "\n" + main)
    cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-Wall",
           "-I" + os.path.join(ROOT, "include"), src, "-o", BIN, "-L" + PKG, "-laco_gpu",
           "-Wl,-rpath,$ORIGIN"]
    subprocess.run(cmd, check=True)
    return BIN


if __name__ == "__main__":
    if not os.path.exists(REF):
        sys.exit(f"{REF} not found")
    print(build())
