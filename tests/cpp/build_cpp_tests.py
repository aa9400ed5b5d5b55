"""Build of the C++ drop-in API test binary (TEST INFRASTRUCTURE): tests/cpp/test_cpp_api
links the product library and the CPU oracle (the checker)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
PKG = os.path.join(ROOT, "paper_2512_08888_b200")
LIB = os.path.join(PKG, "librotconv_b200.so")


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else 0.0


def build_cpp_tests(verbose: bool = False) -> str:
    """g++ build of tests/cpp/test_cpp_api: the C++ drop-in headers (include/rotconv/*.hpp)
    linked against librotconv_b200.so (the product) and oracle/librc_oracle.so (the
    checker).  Test infrastructure only; rpaths are $ORIGIN-relative so the binary runs
    from the repo snapshot on the GPU box."""
    src = os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp")
    out = os.path.join(ROOT, "tests", "cpp", "test_cpp_api")
    oracle = os.path.join(ROOT, "oracle")
    deps = [src, LIB, os.path.join(oracle, "librc_oracle.so")] + [
        os.path.join(ROOT, "include", "rotconv", f) for f in os.listdir(os.path.join(ROOT, "include", "rotconv"))]
    if _mtime(out) >= max(_mtime(d) for d in deps):
        return out
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-march=x86-64-v3",
           f"-I{os.path.join(ROOT, 'include')}", f"-I{oracle}", src, "-o", out,
           f"-L{PKG}", "-lrotconv_b200", f"-L{oracle}", "-lrc_oracle",
           "-Wl,-rpath,$ORIGIN/../../paper_2512_08888_b200", "-Wl,-rpath,$ORIGIN/../../oracle", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"C++ API test build failed:\n{r.stderr[-6000:]}")
    if verbose:
        print(f"[build] {out}", file=sys.stderr)
    return out
