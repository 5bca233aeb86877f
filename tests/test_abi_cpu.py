"""CPU-side checks of the drop-in boundary: the C-ABI library builds, loads
without a GPU, exports every symbol include/detshare/ds.h declares, and fails
loudly (no fallback) when asked to create a domain with no GPU present."""
import ctypes
import os
import re

import pytest

from paper_2603_15042_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "detshare", "ds.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|int64_t)\s+(ds_\w+)\(", text, re.M)))


def test_header_and_binding_agree():
    assert sorted(_abi.EXPORTS) == header_functions()


def test_library_exports_every_declared_symbol():
    L = _abi.lib()
    for name in header_functions():
        assert hasattr(L, name), name


def test_status_names_follow_errc_order():
    L = _abi.lib()
    # errors.hpp:8-19 order
    names = ["Ok", "InvalidTier", "BindConflict", "DoubleBind", "CausalityViolation", "EventBudgetExceeded",
             "TraceViolation", "PlanMismatch", "InvalidSplit", "ParseError", "ConfigError"]
    for i, n in enumerate(names):
        assert L.ds_status_name(i).decode() == n
    assert L.ds_status_name(100).decode() == "CudaError"
    assert L.ds_abi_version() == 1


def test_args_struct_layout():
    assert ctypes.sizeof(_abi.ReduceArgs) == 48
    assert ctypes.sizeof(_abi.SgemmArgs) == 40
    assert ctypes.sizeof(_abi.Completion) == 48
    assert ctypes.sizeof(_abi.BlockRecord) == 32
    assert ctypes.sizeof(_abi.GemmArgs) == 448
    assert ctypes.sizeof(_abi.SplitkReduceArgs) == 48
    # field offsets pinned by static_asserts in bodies/decode.cuh, gemm_tc.cuh and collective.cuh
    assert ctypes.sizeof(_abi.GemvArgs) == 400
    want = {_abi.GemmArgs: {"K": 272, "bk": 296, "abandon": 304, "l2_hint": 308, "tiles": 312, "fuse_fold": 316, "tmC": 320},
            _abi.SplitkReduceArgs: {"splits": 36, "rows": 40},
            _abi.GemvArgs: {"out": 256, "N": 320, "dbg": 360, "w_packed": 368, "bm": 376, "sk": 384, "pair": 388, "pf_ahead": 392},
            _abi.AttnArgs: {"q": 256, "L": 288, "scale": 300, "dbg": 304, "kbase": 312, "l2_pf_kb": 328, "tc": 332},
            _abi.AllreduceArgs: {"out": 128, "outs": 136, "n": 200, "rank": 212, "chunk": 216}}
    for S, fields in want.items():
        for name, off in fields.items():
            assert getattr(S, name).offset == off, (S.__name__, name)


def test_domain_create_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2603_15042_b200.runtime import Domain
    with pytest.raises(_abi.DsError) as ei:
        Domain(0)
    assert ei.value.code in (100, 101)


def test_invalid_tier_rejected_before_device():
    # create_pool rejects tiers outside (0, 1] (types.cpp:91-96) — checked
    # after the device probe on a GPU box, so only the code path is exercised
    cfg = _abi.DomainConfig()
    cfg.n_tiers = 1
    cfg.tier_num[0] = 3
    cfg.tier_den[0] = 2
    h = ctypes.c_void_p()
    rc = _abi.lib().ds_domain_create(ctypes.byref(cfg), ctypes.byref(h))
    assert rc in (1, 101)


def test_plain_c_caller_links_and_runs(tmp_path):
    """The C ABI from C (examples/ds_cabi_demo.c): header + library only."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / "ds_demo"
    libdir = os.path.join(root, "paper_2603_15042_b200")
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-I" + os.path.join(root, "include"),
                    os.path.join(root, "examples", "ds_cabi_demo.c"), "-L" + libdir, "-ldetshare",
                    "-Wl,-rpath," + libdir, "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.splitlines()
    n = int(out[0].split()[1])
    assert n > 0 and "kernels" in out[0]
    where = [int(x) for x in out[1].split()[1:]]
    assert sorted(set(where)) == list(range(8))
    # metrics: TTFT p99 9000 ns; TPOT p50 = 10000/3 (exact); one TPOT above 3.5 us
    assert out[2] == "metrics ttft_p99 9000/1 tpot_p50 10000/3 tpot_violations 1"
    assert out[3].split("-> ")[1] in ("InvalidTier", "NoDevice")
