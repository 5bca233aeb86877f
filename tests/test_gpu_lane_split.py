"""Lane split (ds_set_lane_split): a memory-bound owner (decode) on lane 0
and a compute-bound lend tenant (training) on lane 1 of the same SMs.  Both
results stay bit-identical to solo; the throughput trade-off is measured by
scripts/lane_split.py (profiles/r1_lane_split.json)."""
from fractions import Fraction

import numpy as np
import pytest
import torch

from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import DecodeConfig, DecodeModel
from gpu_util import sgemm_copies as _sgemm

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", [1, 2])
def test_lane_split_keeps_both_tenants_bit_exact(mode):
    """ds_set_lane_split: decode owns lane 0 of every SM, training runs on
    lane 1 of the same SMs; both results stay bit-identical to solo."""
    m = DecodeModel(DecodeConfig(layers=2, vocab=2048, L=96, attn_splits=2), seed=5)
    tok0 = m.tokens.clone()
    kc0 = [k.clone() for k in m.kc]
    vc0 = [v.clone() for v in m.vc]
    m.solo_step()
    torch.cuda.synchronize()
    solo_logits = m.logits.clone()
    m.tokens.copy_(tok0)
    for l in range(m.cfg.layers):
        m.kc[l].copy_(kc0[l])
        m.vc[l].copy_(vc0[l])
    m.logits.zero_()
    keep, sargs, grid = _sgemm(copies=3)
    Cs = keep[2]
    torch.cuda.synchronize()
    with Domain(0, tiers=[Fraction(1)], block_log_capacity=1 << 16) as dom:
        dom.start()
        td = dom.tenant("decode", _abi.LATENCY_CRITICAL)
        ts = dom.tenant("train", _abi.BEST_EFFORT)
        kids = m.register(dom)
        ks = [dom.kernel("sgemm", _abi.BODY_SGEMM, grid, a) for a in sargs[1:]]
        dom.set_lend(ts)
        dom.set_lane_split(mode)
        dom.quota_set([td] * dom.num_sms)
        seqs = [dom.launch(ts, k) for k in ks]
        last = None
        for k in kids:
            last = dom.launch(td, k)
        dom.wait(td, last, 30000)
        for s in seqs:
            dom.wait(ts, s, 60000)
        got_logits = m.logits.cpu()
        got = [C.cpu() for C in Cs]
        sms = {b.smid for b in dom.block_log() if b.tenant == ts}
        dom.set_lane_split(0)
    assert np.array_equal(got_logits.view(torch.int16).numpy(), solo_logits.cpu().view(torch.int16).numpy())
    ref = got[0].numpy().view(np.uint32)
    for C in got[1:]:
        assert np.array_equal(C.numpy().view(np.uint32), ref)
    assert len(sms) > 100  # training ran beside decode on (nearly) every SM
