"""Immutable-launch-config equivalence on random scenarios (
reference check_immutable_equivalence, src/numlab/equivalence.cpp:56-95):
2-4 tenants share the GPU, each running a random program of reduction
kernels (random format, n, logical grid, seed) while the device rewrites the
SM quota at random claim counts; every result equals the reference's own
reduction_result (C restatement, pinned to the reference by the golden
fixtures), every tenant's transcript is its launch program unchanged, and
each launch ran every logical block exactly once."""
import random
from fractions import Fraction

import numpy as np
import pytest

from oracle import loader
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain

from test_gpu_executor import FMT, ReduceKernel

pytestmark = pytest.mark.gpu

SCENARIOS = 100


def test_random_scenarios_are_equivalent_to_solo():
    rnd = random.Random(2603)
    cn = loader.cnumlab()
    plans = []
    for sc in range(SCENARIOS):
        ntenant = rnd.randint(2, 4)
        prog = []
        for t in range(ntenant):
            for _ in range(rnd.randint(1, 3)):
                fmt = rnd.choice(["fp16", "bf16", "fp32"])
                n = rnd.choice([1, 7, 100, 1000, 4096, 10000])
                grid = rnd.choice([1, 2, 3, 16, 37, 64, 148, 300])
                prog.append((t, ReduceKernel(rnd.getrandbits(32), n, fmt, grid), fmt, n, grid))
        plans.append((ntenant, prog))
    # all device data exists before the executor starts
    with Domain(0, tiers=[Fraction(1)], block_log_capacity=1 << 22) as dom:
        dom.start()
        tenants = [dom.tenant(f"t{i}", _abi.BEST_EFFORT) for i in range(4)]
        N = dom.num_sms
        for sc, (ntenant, prog) in enumerate(plans):
            # random SM split between the scenario's tenants, then random
            # device-side rewrites at random claim counts of random launches
            cuts = sorted(rnd.sample(range(1, N), ntenant - 1))
            bounds = [0] + cuts + [N]
            owner = [-1] * N
            for i in range(ntenant):
                for s in range(bounds[i], bounds[i + 1]):
                    owner[s] = tenants[i]
            dom.quota_set(owner)
            dom.clear_logs()
            # one device-side quota rewrite at a random claim count of a random
            # launch, installed before the launches (triggers fire in order)
            nxt = {t: len(dom.transcript(tenants[t])) for t in range(ntenant)}
            kids = []
            for t, k, fmt, n, grid in prog:
                kids.append(dom.kernel(f"reduce/{fmt}/{n}", _abi.BODY_REDUCE_CHUNKS, (grid, 1, 1), k.args))
            dom.quota_triggers_reset()
            j = rnd.randrange(len(prog))
            tj = prog[j][0]
            sj = nxt[tj] + sum(1 for t, *_ in prog[:j] if t == tj)
            perm = tenants[:ntenant]
            dom.quota_at_claim(tenants[tj], sj, rnd.randint(0, max(0, prog[j][4] - 1)),
                               [perm[rnd.randrange(ntenant)] for _ in range(N)])
            seqs = []
            for (t, k, fmt, n, grid), kid in zip(prog, kids):
                seqs.append((t, kid, dom.launch(tenants[t], kid), k, fmt, n, grid))
            assert seqs[j][2] == sj
            for t, kid, s, k, fmt, n, grid in seqs:
                dom.wait(tenants[t], s, 60000)
            log = dom.block_log()
            for t, kid, s, k, fmt, n, grid in seqs:
                assert k.result() == reference_bits(cn, k, fmt, n, grid), (sc, fmt, n, grid)
                blocks = sorted(b.block for b in log if b.tenant == tenants[t] and b.seq == s)
                assert blocks == list(range(grid)), (sc, t, s)
            for i in range(ntenant):
                mine = [(kid, grid) for t, kid, s, k, fmt, n, grid in seqs if t == i]
                assert dom.transcript(tenants[i])[-len(mine):] == mine
            # the control words the triggers installed must not leak into the next scenario
            dom.quota_set([-1] * N)


def reference_bits(cn, k, fmt, n, grid):
    """reduction_result of the tenant's input (the C restatement of
    reduce_with_plan over balanced(n, grid), pinned to the reference)."""
    import ctypes
    if n == 0:
        return 0
    x = k.x.cpu().numpy().astype(np.uint32) & (0xFFFF if fmt != "fp32" else 0xFFFFFFFF)
    arr = (ctypes.c_uint32 * n)(*x.tolist())
    return cn.cn_reduce_bits(arr, n, FMT[fmt], grid, 0)
