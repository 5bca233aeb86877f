"""The reference-named C++ façade (include/detshare/corosim.hpp): compiled
against libdetshare.so and run on the host (no GPU): Rational, make_policy /
policy_names, built-ins through the C ABI, a user Policy through the vtable
trampolines.  The GPU half runs in tests/test_gpu_boundary.py."""
import os
import subprocess

from paper_2603_15042_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2603_15042_b200")


def build_facade_test(out):
    _abi.lib()  # builds libdetshare.so in-tree if needed
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_facade.cpp"), "-o", str(out),
                    "-L" + PKG, "-l:libdetshare.so", "-Wl,-rpath," + PKG], check=True)
    return str(out)


def test_facade_host(tmp_path):
    exe = build_facade_test(tmp_path / "test_facade")
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "host facade tests: ok" in r.stdout
