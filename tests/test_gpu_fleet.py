"""Fleet on a B200: global exception -> emergency migration of a running
coroutine to a standby device, and planned migration with eager / lazy
working-set copies and demand faults (csrc/fleet.cpp; reference
engine.cpp:563-672, 1095-1166).

The box has one GPU, so the "devices" are two domains on GPU 0 used one at a
time (the fleet runs one executor per physical GPU at a time and stops an
idle one before starting the next).  Copies are device-to-device on the copy
engines, exactly the path a peer copy takes between two GPUs.

Checked: every logical block of the interrupted launch runs exactly once
across the two devices (block logs), the launch resumes at its next unclaimed
block (ds_launch_from), and every output is bit-identical to plain-grid solo
runs of the same kernels on the same inputs."""
import time
from fractions import Fraction

import numpy as np
import pytest
import torch

from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.fleet import Fleet
from paper_2603_15042_b200.runtime import Domain, solo_launch

pytestmark = pytest.mark.gpu

F = Fraction


def _sgemm_inputs(n, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    A = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
    B = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
    return A, B


def _solo_sgemm(A, B):
    n = A.shape[0]
    C = torch.zeros(n, n, device="cuda")
    solo_launch(0, "sgemm", _abi.BODY_SGEMM, (n // 64, n // 64, 1), _abi.SgemmArgs(A.data_ptr(), B.data_ptr(),
                                                                                   C.data_ptr(), n, n, n, 0))
    torch.cuda.synchronize()
    return C


def _blocks(dom, tenant, grid):
    return [b.block for b in dom.block_log() if b.tenant == tenant and b.flags == 0 and b.seq == 0]


def test_global_exception_moves_running_coroutine_to_standby_bit_exact():
    n = 1024
    A, B = _sgemm_inputs(n, 3)
    C_solo = _solo_sgemm(A, B)
    D_solo = _solo_sgemm(C_solo, B)
    C = torch.zeros(n, n, device="cuda")
    D = torch.zeros(n, n, device="cuda")
    grid_spin = 3072
    spin = torch.zeros(grid_spin * 3, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    # both domains exist before any executor starts (domain creation runs a probe kernel)
    dom0 = Domain(0, tiers=[F(1, 2), F(1, 4), F(1, 4)], block_log_capacity=1 << 16)
    dom1 = Domain(0, tiers=[F(1, 4), F(1, 2), F(1)], block_log_capacity=1 << 16)
    with Fleet() as fl:
        d0 = fl.add_device(dom0, standby=False)
        d1 = fl.add_device(dom1, standby=True)
        ja = fl.add_job(d0, "train-a")
        jb = fl.add_job(d0, "train-b")
        rs = fl.add_region(ja, spin.data_ptr(), spin.numel() * 8)
        rA = fl.add_region(ja, A.data_ptr(), A.numel() * 4)
        rB = fl.add_region(ja, B.data_ptr(), B.numel() * 4)
        rC = fl.add_region(ja, C.data_ptr(), C.numel() * 4)
        rD = fl.add_region(ja, D.data_ptr(), D.numel() * 4)
        k_spin = fl.add_kernel(ja, "spin", _abi.BODY_SPIN, (grid_spin, 1, 1), _abi.SpinArgs(0, 400000),
                               relocs=[("out", rs, 0)], touched=[rs])
        k_c = fl.add_kernel(ja, "sgemm", _abi.BODY_SGEMM, (n // 64, n // 64, 1), _abi.SgemmArgs(0, 0, 0, n, n, n, 0),
                            relocs=[("A", rA, 0), ("B", rB, 0), ("C", rC, 0)], touched=[rA, rB, rC])
        k_d = fl.add_kernel(ja, "sgemm", _abi.BODY_SGEMM, (n // 64, n // 64, 1), _abi.SgemmArgs(0, 0, 0, n, n, n, 0),
                            relocs=[("A", rC, 0), ("B", rB, 0), ("C", rD, 0)], touched=[rC, rB, rD])
        # job b: a small spin on its own buffer, bound to a 1/4 pctx
        spin_b = torch.zeros(64 * 3, dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()
        rb = fl.add_region(jb, spin_b.data_ptr(), spin_b.numel() * 8)
        kb = fl.add_kernel(jb, "spin-b", _abi.BODY_SPIN, (64, 1, 1), _abi.SpinArgs(0, 1000000),
                           relocs=[("out", rb, 0)], touched=[rb])
        fl.bind(ja, 0)  # tier 1/2
        fl.bind(jb, 1)  # tier 1/4
        dom0.start()
        la = [fl.launch(ja, k) for k in (k_spin, k_c, k_d)]
        lb = fl.launch(jb, kb)
        time.sleep(0.003)  # the spin launch (3072 x 400 us on 148 lanes ~ 8.3 ms) is mid-way
        fl.global_exception(d0)
        for l in la:
            fl.wait(ja, l)
        ia, ib = fl.job(ja), fl.job(jb)
        migs = fl.migrations()
        ledger = fl.ledger()
        dom1.stop()
        blocks0 = _blocks(dom0, 0, grid_spin)
        blocks1 = _blocks(dom1, ia.tenant, grid_spin)
        D_got = np.empty((n, n), dtype=np.float32)
        spin_got = np.empty(grid_spin * 3, dtype=np.int64)
        fl.read_region(ja, rD, D_got)
        fl.read_region(ja, rs, spin_got)
        dom0.close()
        dom1.close()
    # job a: emergency-migrated to the standby's 1/2 pctx (smallest adequate tier)
    assert ia.status == 0 and ia.device == d1 and ia.pctx == 1, (ia.status, ia.device, ia.pctx)
    em = [m for m in migs if m.emergency]
    assert len(em) == 1 and em[0].job == ja and em[0].dst_device == d1 and em[0].dst_pctx == 1
    assert em[0].eager_bytes == sum(t.numel() * t.element_size() for t in (spin, A, B, C, D))
    # it resumed mid-launch: the spin launch's blocks ran exactly once across both devices
    assert em[0].resumed_launch == 0 and 0 < em[0].resumed_block < grid_spin, em[0].resumed_block
    assert sorted(blocks0 + blocks1) == list(range(grid_spin))
    assert max(blocks0) < em[0].resumed_block <= min(blocks1)
    # every block's record survived the move (written on device 0, copied, or written on device 1)
    rec = spin_got.reshape(grid_spin, 3)
    assert bool((rec[:, 1] > 0).all()) and bool((rec[:, 2] >= rec[:, 1]).all())
    # the SGEMM chain after the move is bit-identical to solo runs
    assert np.array_equal(D_got.view(np.int32), D_solo.cpu().numpy().view(np.int32))
    # job b: the only standby device now hosts live work -> stranded
    assert ib.status == 2
    assert ledger["emergency_migrations"] == 1 and ledger["stranded"] == 1


def test_planned_migration_eager_lazy_and_demand_faults_bit_exact():
    n = 1024
    A, B = _sgemm_inputs(n, 5)
    C_solo = _solo_sgemm(A, B)
    D_solo = _solo_sgemm(C_solo, B)
    C = torch.zeros(n, n, device="cuda")
    D = torch.zeros(n, n, device="cuda")
    torch.cuda.synchronize()
    dom0 = Domain(0, tiers=[F(1)], block_log_capacity=0)
    dom1 = Domain(0, tiers=[F(1, 2), F(1)], block_log_capacity=0)
    with Fleet() as fl:
        d0 = fl.add_device(dom0)
        d1 = fl.add_device(dom1)
        j = fl.add_job(d0, "train")
        rA = fl.add_region(j, A.data_ptr(), A.numel() * 4)
        rB = fl.add_region(j, B.data_ptr(), B.numel() * 4)
        rC = fl.add_region(j, C.data_ptr(), C.numel() * 4)
        rD = fl.add_region(j, D.data_ptr(), D.numel() * 4)
        k_c = fl.add_kernel(j, "sgemm", _abi.BODY_SGEMM, (n // 64, n // 64, 1), _abi.SgemmArgs(0, 0, 0, n, n, n, 0),
                            relocs=[("A", rA, 0), ("B", rB, 0), ("C", rC, 0)], touched=[rA, rB, rC])
        k_d = fl.add_kernel(j, "sgemm", _abi.BODY_SGEMM, (n // 64, n // 64, 1), _abi.SgemmArgs(0, 0, 0, n, n, n, 0),
                            relocs=[("A", rC, 0), ("B", rB, 0), ("C", rD, 0)], touched=[rC, rB, rD])
        fl.bind(j, 0)
        dom0.start()
        l0 = fl.launch(j, k_c)
        fl.wait(j, l0)
        # after K1 its regions are dirty and live on device 0; D was never touched
        assert fl.region(j, rC)[2] and not fl.region(j, rD)[2]
        # planned move with no queued kernel: eager = touched(next) = {}, lazy = dirty = {A, B, C}
        fl.migrate(j, d1, 1)
        m = fl.migrations()[-1]
        assert not m.emergency and m.eager_bytes == 0
        assert m.lazy_bytes == 3 * n * n * 4
        l1 = fl.launch(j, k_d)  # touches C, B (lazy or landed) and D (never on device 1: demand fault)
        fl.wait(j, l1)
        info = fl.job(j)
        ledger = fl.ledger()
        dom1.stop()
        D_got = np.empty((n, n), dtype=np.float32)
        fl.read_region(j, rD, D_got)
        dom0.close()
        dom1.close()
    assert info.device == d1 and info.pctx == 1
    assert ledger["demand_faults"] >= 1 and ledger["lazy_bytes"] == 3 * n * n * 4
    assert np.array_equal(D_got.view(np.int32), D_solo.cpu().numpy().view(np.int32))
