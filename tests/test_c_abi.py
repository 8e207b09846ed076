"""The C ABI from a pure-C program (tests/c_abi/consumer.c, compiled with gcc
against include/bnf.h and linked to libbnf.so): host calls and the no-GPU
refusal on CPU; on a B200, bnf_apply_Ar against the oracle fixture
(tests/golden/c_abi_fcc654.bin, scripts/make_c_fixture.py)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1806_10284_b200")
FIX = os.path.join(ROOT, "tests", "golden", "c_abi_fcc654.bin")


def _build(tmp_path):
    exe = str(tmp_path / "consumer")
    cmd = ["gcc", "-O2", "-std=c99", "-Wall", "-Werror", os.path.join(ROOT, "tests", "c_abi", "consumer.c"),
           "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include", "-L" + PKG, "-lbnf",
           "-L/usr/local/cuda/lib64", "-lcudart", "-lm", "-Wl,-rpath," + PKG, "-Wl,-rpath,/usr/local/cuda/lib64",
           "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_consumer_builds_and_runs_host_calls(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe, FIX], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "lattice m = " in r.stdout


@pytest.mark.gpu
def test_c_consumer_apply_matches_oracle(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = _build(tmp_path)
    r = subprocess.run([exe, FIX], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "pass" in r.stdout, r.stdout + r.stderr
