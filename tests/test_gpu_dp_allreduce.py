"""DP training tenant's gradient all-reduce body (csrc/bodies/collective.cuh,
reduce-scatter + all-gather) on W virtual ranks = W tenants of one domain on
one B200 (the multi-GPU path differs only in where the peer pointers come
from).  Bit-exact against a rank-ordered fp32 sum rounded once to bf16,
identical on every rank, across epochs (flag-slot reuse), with ranks arriving
late, and with fewer chunks than ranks (ranks owning no chunk)."""
import time

import numpy as np
import pytest
import torch

from paper_2603_15042_b200 import _abi, dp
from paper_2603_15042_b200.runtime import Domain

pytestmark = pytest.mark.gpu


def expected(grads):
    acc = torch.zeros(grads[0].numel(), dtype=torch.float32)
    for g in grads:
        acc += g.cpu().float()
    return acc.to(torch.bfloat16)


@pytest.mark.parametrize("world,n,chunk", [(4, 1 << 20, 1 << 16), (3, 1000000, 1 << 15), (8, 65536, 8192),
                                           (1, 4096, 1024), (8, 24576, 8192)])
def test_allreduce_virtual_ranks_bit_exact(world, n, chunk):
    g = torch.Generator(device="cuda").manual_seed(world)
    flags = [torch.zeros(dp.FLAG_BYTES, dtype=torch.uint8, device="cuda") for _ in range(world)]
    outs = [[torch.zeros(n, dtype=torch.bfloat16, device="cuda") for _ in range(world)] for _ in range(3)]
    # all device data exists before the executor starts: no other kernel can
    # run beside the resident executor (it holds every SM)
    grads = [[((torch.rand(n, device="cuda", generator=g) * 2 - 1) * (r + 1)).to(torch.bfloat16)
              for r in range(world)] for _ in range(3)]
    torch.cuda.synchronize()
    with Domain(0, block_log_capacity=0) as dom:
        dom.start()
        ts = [dom.tenant(f"rank{r}", _abi.BEST_EFFORT) for r in range(world)]
        per = dom.num_sms // world
        owner = [ts[min(i // per, world - 1)] for i in range(dom.num_sms)]
        dom.quota_set(owner)
        for epoch in range(3):
            kids = []
            for r in range(world):
                a = dp.make_args([x.data_ptr() for x in grads[epoch]], [f.data_ptr() for f in flags],
                                 [o.data_ptr() for o in outs[epoch]], n, r, chunk)
                kids.append(dom.kernel("dp/allreduce", _abi.BODY_ALLREDUCE_P2P, dp.grid_for(n, chunk), a,
                                       phase=_abi.TRAINING))
            seqs = []
            for r in range(world):
                if epoch == 1 and r == world - 1:
                    time.sleep(0.05)  # a late rank: the others wait at the ready barrier
                seqs.append(dom.launch(ts[r], kids[r]))
            for r in range(world):
                dom.wait(ts[r], seqs[r], 30000)
    for epoch in range(3):
        want = expected(grads[epoch]).view(torch.int16).numpy()
        for r in range(world):
            assert np.array_equal(outs[epoch][r].cpu().view(torch.int16).numpy(), want), (epoch, r)
