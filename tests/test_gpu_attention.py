"""GQA decode attention body (mma.sync and tcgen05 paths) vs a plain torch
fp32 reference on the same bf16 inputs (tolerance: bf16 output rounding,
|err| <= 2^-7 |ref| + 2^-9)."""
import math

import pytest
import torch

from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import solo_launch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tc", [0, 1])
@pytest.mark.parametrize("L,S", [(96, 2), (1024, 2), (333, 3), (32, 1), (1000, 4), (1024, 1), (70, 1)])
def test_attention_matches_fp32_reference(L, S, tc):
    g = torch.Generator(device="cuda").manual_seed(L)
    Lmax = L + 5
    q = (torch.randn(32, 4096, device="cuda", generator=g)).to(torch.bfloat16)
    kc = (torch.randn(32, 8, Lmax, 128, device="cuda", generator=g)).to(torch.bfloat16)
    vc = (torch.randn(32, 8, Lmax, 128, device="cuda", generator=g)).to(torch.bfloat16)
    out = torch.zeros(32, 4096, device="cuda", dtype=torch.bfloat16)
    ws = torch.zeros(256 * S * 4 * 130, device="cuda")
    ctr = torch.zeros(256, device="cuda", dtype=torch.int32)
    rows = 32 * 8 * Lmax
    a = _abi.AttnArgs(_abi.tensor_map_kv(kc.data_ptr(), rows),
                      _abi.tensor_map_kv(vc.data_ptr(), rows),
                      q.data_ptr(), out.data_ptr(), ws.data_ptr(), ctr.data_ptr(), L, Lmax, S, 1.0 / math.sqrt(128), 0)
    a.tc = tc  # 1: S^T / O^T on tcgen05 with TMEM accumulators (lazy softmax rescale)
    solo_launch(0, "attn", _abi.BODY_ATTN_DECODE, (256 * S, 1, 1), a)
    torch.cuda.synchronize()
    Q = q.float().view(32, 8, 4, 128)
    s = torch.einsum("bhqd,bhpd->bhqp", Q, kc[:, :, :L].float()) / math.sqrt(128)
    ref = torch.einsum("bhqp,bhpd->bhqd", torch.softmax(s, -1), vc[:, :, :L].float()).reshape(32, 4096)
    err = (out.float() - ref).abs()
    assert bool((err <= ref.abs() * 2 ** -7 + 2 ** -9).all()), float(err.max())
    assert int(ctr.sum()) == 0
