"""The C++ drop-in API (include/rotconv/*.hpp) through its own test binary
(tests/cpp/test_cpp_api.cpp, built by __graft_entry__.build()).  --cpu covers the host
containers, transforms, packers and the reference's validation messages; --gpu runs every
device-served op against the CPU oracle (bit-exact on dyadic inputs)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_cpp_api")


def _binary():
    if not os.path.exists(BIN):
        import sys
        sys.path.insert(0, ROOT)
        sys.path.insert(0, os.path.join(ROOT, "tests", "cpp"))
        from paper_2512_08888_b200 import build as B
        import build_cpp_tests
        B.build()
        build_cpp_tests.build_cpp_tests()
    return BIN


def _run(flag):
    r = subprocess.run([_binary(), flag], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


def test_cpp_api_host_side():
    _run("--cpu")


@pytest.mark.gpu
def test_cpp_api_device_ops_vs_oracle(dev):
    _run("--gpu")
