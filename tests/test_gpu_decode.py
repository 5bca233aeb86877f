"""Decode tenant numerics: one Llama-3-shaped decode step (2 layers, reduced
vocab/KV for test time) on the native bodies vs a plain torch fp32 reference
of the same math with the same bf16 rounding points.  Tolerance: bf16
storage of every intermediate -> |err| <= 0.05 (|ref| + 1), mean <= 5e-3.
Then: the same step as a coroutine under quota changes is bit-identical to
the solo step."""
from fractions import Fraction

import numpy as np
import pytest
import torch

from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import DecodeConfig, DecodeModel, pick_split

pytestmark = pytest.mark.gpu


# (row slabs, GEMV grids): split-K defaults, 64-row slabs, and stream-K
# grids at the full GPU's and the 1/2 tier's lane counts
BM_VARIANTS = ["", "qkv:64,o:64,down:64,lm:64", "sk296", "qkv:64,o:64,down:64,lm:64/sk148"]
SK = {"sk296": "qkv:296,o:296,gu:296,down:296", "sk148": "qkv:148,o:148,gu:296,down:148"}


def small_model(bms=""):
    cfg = DecodeConfig(layers=2, vocab=2048, L=96, attn_splits=2)
    bm, _, g = bms.rpartition("/") if "/" in bms else (bms, "", "")
    if bm.startswith("sk"):
        bm, g = "", bm
    return DecodeModel(cfg, seed=5, bm_override=bm, g_override=SK.get(g, ""))


@pytest.mark.parametrize("bms", BM_VARIANTS)
def test_decode_step_matches_torch_reference(bms):
    m = small_model(bms)
    tok0 = m.tokens.clone()
    kc0 = [k.clone() for k in m.kc]
    vc0 = [v.clone() for v in m.vc]
    m.solo_step()
    torch.cuda.synchronize()
    ref_logits, ref_h, ref_tok = m.reference_step(tok0, kc0, vc0)
    got = m.logits.float()
    ref = ref_logits.float()
    err = (got - ref).abs() / (ref.abs() + 1)
    assert float(err.max()) <= 0.05, float(err.max())
    assert float(err.mean()) <= 5e-3, float(err.mean())
    herr = (m.H[m.cfg.layers % 2].float() - ref_h.float()).abs() / (ref_h.float().abs() + 1)
    assert float(herr.max()) <= 0.05
    # greedy sampling: the kernel's argmax of its own logits (ties -> lowest index)
    assert torch.equal(m.tokens.cpu(), m.logits.float().argmax(-1).to(torch.int32).cpu())
    # and the sampled token agrees with the reference wherever the top-2 margin exceeds the tolerance
    top2 = ref_logits.float().topk(2, -1).values
    clear = (top2[:, 0] - top2[:, 1]) > 0.1 * (top2[:, 0].abs() + 1)
    assert torch.equal(m.tokens.cpu()[clear.cpu()], ref_tok.cpu()[clear.cpu()])


@pytest.mark.parametrize("bms", BM_VARIANTS)
def test_decode_step_coroutine_bit_exact_vs_solo(bms):
    m = small_model(bms)
    tok0 = m.tokens.clone()
    kc0 = [k.clone() for k in m.kc]
    vc0 = [v.clone() for v in m.vc]
    m.solo_step()
    torch.cuda.synchronize()
    solo_logits = m.logits.clone()
    solo_h = m.H[m.cfg.layers % 2].clone()
    # reset state, then run the same step as a coroutine with quota changes
    m.tokens.copy_(tok0)
    for l in range(m.cfg.layers):
        m.kc[l].copy_(kc0[l])
        m.vc[l].copy_(vc0[l])
    m.logits.zero_()
    torch.cuda.synchronize()
    with Domain(0, tiers=[Fraction(1, 2), Fraction(1)], block_log_capacity=1 << 16) as dom:
        dom.start()
        t = dom.tenant("decode", _abi.LATENCY_CRITICAL)
        dom.quota_set(dom.mask(t, 0, dom.num_sms))
        kids = m.register(dom)
        dom.quota_at_claim(t, 3, 10, dom.mask(t, 0, 37))
        dom.quota_at_claim(t, 6, 5, dom.mask(t, 40, 90))
        dom.quota_at_claim(t, 9, 0, dom.mask(t, 0, dom.num_sms))
        last = None
        for k in kids:
            last = dom.launch(t, k)
        dom.wait(t, last)
        got_logits = m.logits.cpu()
        got_h = m.H[m.cfg.layers % 2].cpu()
        assert dom.transcript(t) == [(k, r[2][0]) for k, r in zip(kids, m.records)]
    assert np.array_equal(got_logits.view(torch.int16).numpy(), solo_logits.cpu().view(torch.int16).numpy())
    assert np.array_equal(got_h.view(torch.int16).numpy(), solo_h.cpu().view(torch.int16).numpy())


def test_full_decode_step_matches_torch_fp32_and_coroutine_bit_exact():
    """The headline decode tenant at full size: Llama-3-8B shapes (32 layers,
    vocab 128256, KV length 1024, batch 32).  Solo step vs the plain torch fp32
    restatement with bf16 rounding points: |err| <= 0.05 (|ref| + 1), mean
    <= 5e-3 (same tolerance as the 2-layer case; bf16 storage of every
    intermediate).  Then the same step as a coroutine on a quarter of the SMs
    with a mid-step change to all of them -- its gate_up projections as the
    two-slab-block variant -- is bit-identical to the solo step, and the
    device checksum body agrees with the host checksum."""
    from paper_2603_15042_b200.tenants import OutputChecksum
    m = DecodeModel(DecodeConfig(), seed=7)
    tok0 = m.tokens.clone()
    kc0 = [k.clone() for k in m.kc]
    vc0 = [v.clone() for v in m.vc]
    m.solo_step()
    torch.cuda.synchronize()
    solo_logits = m.logits.clone()
    ref_logits, ref_h, _ = m.reference_step(tok0, kc0, vc0)
    del kc0, vc0
    err = (solo_logits.float() - ref_logits.float()).abs() / (ref_logits.float().abs() + 1)
    assert float(err.max()) <= 0.05, float(err.max())
    assert float(err.mean()) <= 5e-3, float(err.mean())
    m.tokens.copy_(tok0)
    m.logits.zero_()
    ck = OutputChecksum(m.logits, cap=4, grid=32)
    torch.cuda.synchronize()
    with Domain(0, tiers=[Fraction(1)], block_log_capacity=0) as dom:
        t = dom.tenant("decode", _abi.LATENCY_CRITICAL)
        # the co-located variant (gate_up as two-slab blocks) against the
        # plain split-K solo step: bit-identical by construction
        kids = m.register_variant(dom, m.register(dom)) + [ck.register(dom, "decode/logits_checksum")]
        dom.start()
        dom.quota_set(dom.mask(t, 0, dom.num_sms // 4))
        dom.quota_at_claim(t, 80, 0, dom.mask(t, 0, dom.num_sms))
        last = None
        for k in kids:
            last = dom.launch(t, k)
        dom.wait(t, last, 120000)
        slots = ck.slots()
    assert torch.equal(m.logits.view(torch.int16), solo_logits.view(torch.int16))
    assert ck.of_seq(slots, last) == OutputChecksum.host(solo_logits)


def test_half_tier_variants_bit_exact_vs_solo():
    """gate_up as 112 two-slab blocks and the LM head as 7-slab blocks
    (register_variant: "gu_pair", "lm_multi") under mid-step quota changes
    equal the one-slab solo step bit for bit."""
    m = small_model()
    assert "gu_pair" in m.variant_records and "lm_multi" in m.variant_records
    tok0 = m.tokens.clone()
    kc0 = [k.clone() for k in m.kc]
    vc0 = [v.clone() for v in m.vc]
    m.solo_step()
    torch.cuda.synchronize()
    solo_logits, solo_act = m.logits.clone(), m.act.clone()
    m.tokens.copy_(tok0)
    for l in range(m.cfg.layers):
        m.kc[l].copy_(kc0[l])
        m.vc[l].copy_(vc0[l])
    m.logits.zero_()
    m.act.zero_()
    torch.cuda.synchronize()
    with Domain(0, tiers=[Fraction(1)], block_log_capacity=0) as dom:
        t = dom.tenant("decode", _abi.LATENCY_CRITICAL)
        kids = m.register_variant(dom, m.register(dom))
        dom.start()
        dom.quota_set(dom.mask(t, 0, 74))
        dom.quota_at_claim(t, 4, 30, dom.mask(t, 10, 50))
        last = None
        for k in kids:
            last = dom.launch(t, k)
        dom.wait(t, last)
    assert torch.equal(m.act.view(torch.int16), solo_act.view(torch.int16))
    assert torch.equal(m.logits.view(torch.int16), solo_logits.view(torch.int16))
