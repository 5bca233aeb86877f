"""Compile and run the C++ policy unit tests (host logic, no GPU)."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_policy_cpp(tmp_path):
    exe = tmp_path / "test_policy"
    src = [os.path.join(ROOT, "tests", "cpp", "test_policy.cpp"),
           os.path.join(ROOT, "paper_2603_15042_b200", "csrc", "policy.cpp")]
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-o", str(exe)] + src, check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "policy tests ok" in r.stdout
