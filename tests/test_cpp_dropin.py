"""Build the C++ drop-in test (tests/cpp/test_dropin.cpp) against the C ABI library
and the C oracle; compile on CPU, run on the GPU."""
import os
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
LIB = os.path.join(ROOT, "paper_1610_06209_b200", "_lib")
ORC = os.path.join(ROOT, "oracle", "_build")
BIN = os.path.join(ROOT, "tests", "cpp", "test_dropin")


def build_binary():
    cmd = ["g++", "-std=c++20", "-O2", SRC, "-o", BIN, f"-L{LIB}", "-lspinners_b200", f"-L{ORC}", "-loracle",
           f"-Wl,-rpath,{LIB}", f"-Wl,-rpath,{ORC}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_dropin_header_compiles(oracle):
    build_binary()
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_dropin_cases_pass_on_gpu(oracle):
    build_binary()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL PASSED" in r.stdout
