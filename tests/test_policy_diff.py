"""Policy parity: the B200 runtime's policies
(csrc/policy.cpp: slo-aware, tpot-first, temporal, static + predict_hol_blocking)
against the reference's own policies.cpp, compiled unmodified into
oracle/_ref, on random PolicyView / LaunchContext snapshots.  Every hook's
decision (kind and target), order key and review time must be identical;
the duration predictor must agree with the reference's exact-rational EWMA."""
import os
import subprocess

import pytest

from oracle import loader

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("seed", [1, 2024])
def test_policies_match_reference_on_random_snapshots(ref, tmp_path, seed):
    exe = tmp_path / "policy_diff"
    src = [os.path.join(ROOT, "tests", "cpp", "policy_diff.cpp"),
           os.path.join(ROOT, "paper_2603_15042_b200", "csrc", "policy.cpp"),
           os.path.join(ROOT, "paper_2603_15042_b200", "csrc", "policy_abi.cpp")]
    subprocess.run(["g++", "-std=c++20", "-O2", "-o", str(exe)] + src + ["-ldl"], check=True)
    r = subprocess.run([str(exe), loader.REF_PATH, "100000", str(seed)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "cases 100000 mismatches 0 ref_errors 0" in r.stdout
    # the built-ins through the C ABI (ds_builtin_decide over a ds_view) decide identically
    import re
    m = re.search(r"c_abi checked (\d+) mismatches (\d+)", r.stdout)
    assert m and int(m.group(1)) > 20000 and int(m.group(2)) == 0, r.stdout
    # the EWMA predictor (double, truncated to ns) is within 1 ns of the exact rational EWMA
    assert "ewma sequences 2000 outside_1ns 0 " in r.stdout
    # every decision branch was exercised
    for line in r.stdout.splitlines():
        if line.startswith("policy 0") or line.startswith("policy 1"):
            assert " preempt 0 " not in line and " remap 0 " not in line, line
