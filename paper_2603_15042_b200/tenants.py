"""Tenant workloads of the benchmark configs, built from the native bodies.

* ``DecodeModel`` — Llama-3-8B-shaped decode step, batch 32 (config 2): per
  layer RMSNorm-folded QKV projection (+ KV-cache append), GQA attention,
  O projection (+ residual), gate/up projection (+ SiLU*up), down projection
  (+ residual); final norm + LM head + argmax.  163 launches per decode step
  (embed with the RMS statistics of its rows, 5 per layer, LM head, argmax).
* ``TrainGemm`` — bf16 GEMM 8192^3 training step on tcgen05 (config 2).

Weights are random (synthetic data, no checkpoints); shapes are exactly the
named model's.  Device memory comes from torch (plumbing only).
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass
from typing import List

import torch

from . import _abi

SMS = 148
LANES = 2
WORKERS = SMS * LANES  # concurrent logical blocks (2 worker lanes per SM)


def pick_split(nb: int, kblocks: int, sms: int = WORKERS, max_s: int = 16, min_kb: int = 4, slack: float = 0.04) -> int:
    """K-split S for a GEMV with nb row slabs: the smallest S whose wave
    efficiency nblk / (ceil(nblk/sms)*sms) is within `slack` of the best,
    keeping >= min_kb k-blocks per block (fewer, larger blocks amortise the
    per-block pipeline fill)."""
    effs = {}
    for s in range(1, max_s + 1):
        if kblocks // s < min_kb:
            break
        n = nb * s
        effs[s] = n / (math.ceil(n / sms) * sms)
    best = max(effs.values())
    return min(s for s, e in effs.items() if e >= best - slack)


def pack_sw128(W: torch.Tensor, bm: int = 128) -> torch.Tensor:
    """[N, K] bf16 -> the SWIZZLE_128B shared-memory image of its [bm x 64]
    tiles, tile (slab, kblock) contiguous at ((slab * K/64) + kblock) * bm*128 B:
    within a tile, row r's 16-B chunk c is stored at chunk c ^ (r % 8)
    (exactly what a TMA SWIZZLE_128B load would place in smem)."""
    N, K = W.shape
    assert N % bm == 0 and K % 64 == 0
    t = W.reshape(N // bm, bm, K // 64, 8, 8).permute(0, 2, 1, 3, 4)  # [nb][kb][r][chunk][8]
    r = torch.arange(bm, device=W.device).view(bm, 1)
    c = torch.arange(8, device=W.device).view(1, 8)
    src = (c ^ (r % 8)).view(1, 1, bm, 8, 1).expand(t.shape[0], t.shape[1], bm, 8, 8)
    return torch.gather(t, 3, src).contiguous()


@dataclass
class DecodeConfig:
    layers: int = 32
    d: int = 4096
    n_q: int = 32
    n_kv: int = 8
    ffn: int = 14336
    vocab: int = 128256
    batch: int = 32
    L: int = 1024          # attended KV length (positions 0..L-1; the new token writes L-1)
    eps: float = 1e-5
    attn_splits: int = 1   # one block per (batch row, kv head): measured best (scripts/block_stats.py ASPLIT sweep)


def sk_contributors(nb: int, kb: int, G: int) -> int:
    """Stream-K GEMV plan (bodies/decode.cuh gemv_body, a.sk = 1): block t of
    G takes units [t U / G, (t+1) U / G) of the U = nb * kb (slab, k-block)
    units.  Returns the most blocks any slab is split across; a run must not
    exceed one slab's k-blocks (the body handles two pieces per block)."""
    U = nb * kb
    if not (1 <= G <= U) or -(-U // G) > kb:
        raise ValueError(f"stream-K grid {G} invalid for {nb} slabs x {kb} k-blocks")
    block_of = lambda u: ((u + 1) * G - 1) // U
    return max(block_of(n * kb + kb - 1) - block_of(n * kb) + 1 for n in range(nb))


class DecodeModel:
    def __init__(self, cfg: DecodeConfig = DecodeConfig(), device="cuda", seed: int = 0, split_override: str = "",
                 bm_override: str = "", pf_override: str = "", g_override: str = ""):
        assert cfg.batch == 32 and cfg.d == cfg.n_q * 128 and cfg.n_q == 4 * cfg.n_kv
        self.cfg = cfg
        c = cfg
        g = torch.Generator(device=device).manual_seed(seed)

        def w(n, k):
            return ((torch.rand(n, k, device=device, generator=g) * 2 - 1) / math.sqrt(k)).to(torch.bfloat16)

        self.kv_dim = c.n_kv * 128
        self.qkv_n = c.d + 2 * self.kv_dim
        self.Wqkv = [w(self.qkv_n, c.d) for _ in range(c.layers)]
        self.Wo = [w(c.d, c.d) for _ in range(c.layers)]
        self.Wgu = [w(2 * c.ffn, c.d) for _ in range(c.layers)]   # slabs of [64 gate | 64 up] rows
        self.Wd = [w(c.d, c.ffn) for _ in range(c.layers)]
        self.lm = w(c.vocab, c.d)
        self.embed = ((torch.rand(c.vocab, c.d, device=device, generator=g) * 2 - 1)).to(torch.bfloat16)
        self.tokens = torch.randint(0, c.vocab, (32,), device=device, generator=g, dtype=torch.int32)
        self.Lmax = c.L
        self.kc = [((torch.rand(32, c.n_kv, self.Lmax, 128, device=device, generator=g) * 2 - 1)).to(torch.bfloat16)
                   for _ in range(c.layers)]
        self.vc = [((torch.rand(32, c.n_kv, self.Lmax, 128, device=device, generator=g) * 2 - 1)).to(torch.bfloat16)
                   for _ in range(c.layers)]
        bf = torch.bfloat16
        self.H = [((torch.rand(32, c.d, device=device, generator=g) * 2 - 1)).to(bf), torch.zeros(32, c.d, device=device, dtype=bf)]
        self.h_mid = torch.zeros(32, c.d, device=device, dtype=bf)
        self.q = torch.zeros(32, c.d, device=device, dtype=bf)
        self.attn = torch.zeros(32, c.d, device=device, dtype=bf)
        self.act = torch.zeros(32, c.ffn, device=device, dtype=bf)
        self.logits = torch.zeros(32, c.vocab, device=device, dtype=bf)
        self.st0 = torch.zeros(1, 32, device=device)
        self.st_h = torch.zeros(c.d // 64, 32, device=device)    # per-slab partial RMS sums (64- or 128-row slabs)
        self.st_mid = torch.zeros(c.d // 64, 32, device=device)
        # split-K plans and workspaces
        self.S = {
            "qkv": pick_split(self.qkv_n // 128, c.d // 64),
            "o": pick_split(c.d // 128, c.d // 64),
            "gu": pick_split(2 * c.ffn // 128, c.d // 64),
            "down": pick_split(c.d // 128, c.ffn // 64),
            "lm": pick_split(c.vocab // 128, c.d // 64),
        }
        # measured on B200 (scripts/split_sweep.py, decode step at 74 and 148
        # SMs): every block pays ~8 us of prologue / partial exchange /
        # epilogue around its weight stream, so the fewest splits that still
        # fill the lanes win — no split at all for gate_up and the LM head
        self.S.update({"qkv": 3, "o": 4, "gu": 1, "down": 4, "lm": 1})
        split_override = split_override or os.environ.get("DS_SPLITS", "")
        if split_override:  # e.g. "o:4,down:5"
            for kv in split_override.split(","):
                k, v = kv.split(":")
                self.S[k] = int(v)
        # stream-K grids (bodies/decode.cuh gemv_body, a.sk): G equal runs of
        # (slab, k-block) units instead of nb x S blocks, so the grid can be a
        # multiple of the worker lanes at both the full GPU (296) and the
        # decode tenant's 1/2 tier (148); 0 = split-K S
        self.G = {"qkv": 0, "o": 0, "gu": 0, "down": 0, "lm": 0}
        for kv in filter(None, (g_override or os.environ.get("DS_GEMV_G", "")).split(",")):
            k, v = kv.split(":")
            self.G[k] = int(v)
        # attention products on tcgen05 (TMEM accumulators) instead of mma.sync
        self.attn_tc = int(os.environ.get("DS_ATTN_TC", "0"))
        # weight rows per slab (M of the swap-AB MMA): 128, or 64 for the small
        # projections (gate_up's SiLU pairing needs 128-row slabs)
        self.BM = {"qkv": 128, "o": 128, "gu": 128, "down": 128, "lm": 128}
        if bm_override:  # e.g. "o:64,qkv:64"
            for kv in bm_override.split(","):
                k, v = kv.split(":")
                self.BM[k] = int(v)
        assert self.BM["gu"] == 128
        # early start: KB of each block's operands past its smem ring that are
        # prefetched into L2 once the previous launch has streamed (its
        # epilogues run).  Measured (scripts/pf_sweep.py,
        # profiles/r2_l2_prefetch_sweep2.jsonl): 128 KB 4.72 vs 4.76 ms per step,
        # deeper prefetches lose (L2 thrash)
        self.PF = {"qkv": 128, "attn": 128, "o": 128, "gu": 128, "down": 128, "lm": 128}
        for kv in filter(None, (pf_override or os.environ.get("DS_L2PF", "")).split(",")):
            k, v = kv.split(":")
            self.PF[k] = int(v)
        shapes = {"qkv": (self.qkv_n, c.d), "o": (c.d, c.d), "gu": (2 * c.ffn, c.d), "down": (c.d, c.ffn),
                  "lm": (c.vocab, c.d)}
        ws_elems = max((sk_contributors(N // self.BM[k], K // 64, self.G[k]) if self.G[k] else self.S[k]) * N
                       for k, (N, K) in shapes.items()) * 32
        self.ws = torch.zeros(ws_elems, device=device)
        self.counters = torch.zeros(max(c.vocab, 2 * c.ffn) // 128 + 1, device=device, dtype=torch.int32)
        self.attn_ws = torch.zeros(256 * c.attn_splits * 4 * 130, device=device)
        self.attn_counters = torch.zeros(256, device=device, dtype=torch.int32)
        self.amax_ws = torch.zeros(32 * 16 * 2, device=device)
        self.amax_counters = torch.zeros(32, device=device, dtype=torch.int32)
        self._build_args()

    # ---- launch records ----
    def _gemv(self, W, X, N, K, S, mode, out, resid=None, stats_in=None, P_in=0, stats_out=None, l=None, bm=128,
              pf=0, G=0):
        if mode == _abi.GEMV_SILU_MUL:
            # slabs [64 gate | 64 up] -> rows interleaved gate/up (2i, 2i+1):
            # the SiLU pairing then stays inside a warp (bodies/decode.cuh)
            assert bm == 128 and (N // bm) % 2 == 0
            W = W.view(N // bm, 2, 64, K).transpose(1, 2).reshape(N, K)
            self._packed.append(W)  # keeps the permuted copy (tmW's base) alive
        Wp = pack_sw128(W, bm)
        self._packed.append(Wp)
        tmW = _abi.tensor_map_bf16(W.data_ptr(), N, K, bm)
        tmX = _abi.tensor_map_bf16(X.data_ptr(), 32, K, 32)
        a = _abi.GemvArgs()
        a.tmW, a.tmX = tmW, tmX
        a.out = out.data_ptr()
        a.resid = resid.data_ptr() if resid is not None else 0
        a.ws = self.ws.data_ptr()
        a.counters = self.counters.data_ptr()
        a.stats_in = stats_in.data_ptr() if stats_in is not None else 0
        a.stats_out = stats_out.data_ptr() if stats_out is not None else 0
        a.kcache = self.kc[l].data_ptr() if l is not None else 0
        a.vcache = self.vc[l].data_ptr() if l is not None else 0
        a.N, a.K, a.S, a.mode, a.P_in = N, K, S, mode, P_in
        a.eps = self.cfg.eps
        a.pos = self.cfg.L - 1
        a.Lmax = self.Lmax
        a.q_dim, a.kv_dim = self.cfg.d, self.kv_dim
        a.w_packed = Wp.data_ptr()
        a.bm = bm
        a.l2_pf_kb = pf
        # sliding L2 prefetch distance (k-blocks) ahead of the ring: DS_GEMV_PF_AHEAD (0 = off)
        a.pf_ahead = int(os.environ.get("DS_GEMV_PF_AHEAD", "0"))
        if G:
            sk_contributors(N // bm, K // 64, G)  # validates the plan
            a.sk = 1
            return a, (G, 1, 1)
        return a, ((N // bm) * S, 1, 1)

    def _build_args(self):
        c = self.cfg
        self.records = []  # (semantic_id, body, grid, args, bytes)
        # alternative records of the same step, by variant name: {record index: record}
        self.variant_records = {}
        self._packed = []  # pre-packed weights (the copies the GEMV bodies stream)
        # token gather + the input rows' RMS statistics in one launch
        ea = _abi.EmbedArgs(self.embed.data_ptr(), self.tokens.data_ptr(), self.H[0].data_ptr(), c.d, c.vocab,
                            self.st0.data_ptr())
        self.records.append(("decode/embed", _abi.BODY_EMBED, (32, 1, 1), ea, 32 * c.d * 2 * 2))
        for l in range(c.layers):
            hin, hout = self.H[l % 2], self.H[(l + 1) % 2]
            st_in, p_in = (self.st0, 1) if l == 0 else (self.st_h, c.d // self.BM["down"])
            a, g = self._gemv(self.Wqkv[l], hin, self.qkv_n, c.d, self.S["qkv"], _abi.GEMV_QKV, self.q,
                              stats_in=st_in, P_in=p_in, l=l, bm=self.BM["qkv"], pf=self.PF["qkv"],
                              G=self.G["qkv"])
            self.records.append((f"decode/qkv", _abi.BODY_GEMV_BF16, g, a, self.qkv_n * c.d * 2))
            rows = 32 * c.n_kv * self.Lmax
            at = _abi.AttnArgs(_abi.tensor_map_kv(self.kc[l].data_ptr(), rows),
                               _abi.tensor_map_kv(self.vc[l].data_ptr(), rows), self.q.data_ptr(),
                               self.attn.data_ptr(), self.attn_ws.data_ptr(), self.attn_counters.data_ptr(), c.L,
                               self.Lmax, c.attn_splits, 1.0 / math.sqrt(128))
            at.kbase, at.vbase, at.l2_pf_kb = self.kc[l].data_ptr(), self.vc[l].data_ptr(), self.PF["attn"]
            at.tc = self.attn_tc
            self.records.append(("decode/attn", _abi.BODY_ATTN_DECODE, (256 * c.attn_splits, 1, 1), at,
                                 2 * 32 * c.n_kv * c.L * 128 * 2))
            a, g = self._gemv(self.Wo[l], self.attn, c.d, c.d, self.S["o"], _abi.GEMV_RESID, self.h_mid, resid=hin,
                              stats_out=self.st_mid, bm=self.BM["o"], pf=self.PF["o"], G=self.G["o"])
            self.records.append(("decode/o", _abi.BODY_GEMV_BF16, g, a, c.d * c.d * 2))
            a, g = self._gemv(self.Wgu[l], self.h_mid, 2 * c.ffn, c.d, self.S["gu"], _abi.GEMV_SILU_MUL, self.act,
                              stats_in=self.st_mid, P_in=c.d // self.BM["o"], pf=self.PF["gu"], G=self.G["gu"])
            self.records.append(("decode/gate_up", _abi.BODY_GEMV_BF16, g, a, 2 * c.ffn * c.d * 2))
            if not self.G["gu"] and self.S["gu"] == 1:
                # the same projection as two-slab blocks (bit-identical: every
                # slab is still one block's k-ordered accumulation)
                ap = _abi.GemvArgs.from_buffer_copy(a)
                ap.pair = 2
                self.variant_records.setdefault("gu_pair", {})[len(self.records) - 1] = (
                    "decode/gate_up", _abi.BODY_GEMV_BF16, (g[0] // 2, 1, 1), ap, 2 * c.ffn * c.d * 2)
            a, g = self._gemv(self.Wd[l], self.act, c.d, c.ffn, self.S["down"], _abi.GEMV_RESID, hout,
                              resid=self.h_mid, stats_out=self.st_h, bm=self.BM["down"], pf=self.PF["down"],
                              G=self.G["down"])
            self.records.append(("decode/down", _abi.BODY_GEMV_BF16, g, a, c.d * c.ffn * 2))
        hfin = self.H[c.layers % 2]
        a, g = self._gemv(self.lm, hfin, c.vocab, c.d, self.S["lm"], _abi.GEMV_STORE, self.logits,
                          stats_in=self.st_h, P_in=c.d // self.BM["down"], bm=self.BM["lm"], pf=self.PF["lm"],
                          G=self.G["lm"])
        self.records.append(("decode/lm_head", _abi.BODY_GEMV_BF16, g, a, c.vocab * c.d * 2))
        if not self.G["lm"] and self.S["lm"] == 1 and self.BM["lm"] == 128:
            # the LM head as 7-slab blocks (144 blocks: one wave on 148 lanes, one continuous
            # 7 MB stream per lane); bit-identical to the one-slab record
            am = _abi.GemvArgs.from_buffer_copy(a)
            am.pair = 7
            self.variant_records.setdefault("lm_multi", {})[len(self.records) - 1] = (
                "decode/lm_head", _abi.BODY_GEMV_BF16, (-(-(c.vocab // 128) // 7), 1, 1), am, c.vocab * c.d * 2)
        chunks = max(1, min(4, c.vocab // 2048))  # 128 blocks: one wave; every block pays a claim + ticket
        am = _abi.ArgmaxArgs(self.logits.data_ptr(), self.tokens.data_ptr(), self.amax_ws.data_ptr(),
                             self.amax_counters.data_ptr(), c.vocab, chunks)
        self.records.append(("decode/argmax", _abi.BODY_ARGMAX, (32 * chunks, 1, 1), am, 32 * c.vocab * 2))

    @property
    def weight_bytes(self) -> int:
        return sum(r[4] for r in self.records if r[1] == _abi.BODY_GEMV_BF16)

    @property
    def step_bytes(self) -> int:
        """Algorithmic HBM bytes per decode step: weights + KV cache read
        (activations are O(MB) and L2-resident)."""
        return sum(r[4] for r in self.records)

    def register(self, dom, phase=_abi.DECODE) -> List[int]:
        return [dom.kernel(sid, body, grid, args, phase=phase) for sid, body, grid, args, _ in self.records]

    HALF_TIER = "gu_pair,lm_multi"

    def register_variant(self, dom, ids: List[int], names: str = HALF_TIER, phase=_abi.DECODE) -> List[int]:
        """The step's kernel ids with the named variants' records registered in
        place of the base ones (other ids shared; names comma-separated).
        "gu_pair": gate_up as 112 two-slab blocks — one wave at the decode
        tenant's 1/2 tier (148 worker lanes) where the 224 one-slab blocks
        need two; "lm_multi": the LM head as 144 seven-slab blocks.  Outputs
        are bit-identical to the base step."""
        out = list(ids)
        for name in filter(None, names.split(",")):
            for i, (sid, body, grid, args, _) in self.variant_records.get(name, {}).items():
                out[i] = dom.kernel(sid, body, grid, args, phase=phase)
        return out

    def prefill_records(self, prompt_tokens: int = 256):
        """A prompt's prefill on the same weights: per layer the four
        projection GEMMs over `prompt_tokens` rows (tcgen05 GEMM body; the
        weights [N][K] are already the K-major B operand).  Activations are
        synthetic (one shared input / output buffer), so this prices and
        schedules prefill without modelling attention over the prompt.
        Returns (records, flops)."""
        c = self.cfg
        P = (prompt_tokens + 127) // 128 * 128
        dev = self.q.device
        self.pf_x = (torch.rand(P, max(c.d, c.ffn), device=dev) * 2 - 1).to(torch.bfloat16)
        self.pf_y = torch.zeros(P, max(self.qkv_n, 2 * c.ffn, c.d), device=dev, dtype=torch.bfloat16)
        recs, flops = [], 0.0
        for l in range(c.layers):
            for name, W in (("qkv", self.Wqkv[l]), ("o", self.Wo[l]), ("gate_up", self.Wgu[l]), ("down", self.Wd[l])):
                N, K = W.shape
                # row-major views with the GEMM's own row pitch (x: [P][K], y: [P][N])
                x = self.pf_x.view(-1)[: P * K].view(P, K)
                y = self.pf_y.view(-1)[: P * N].view(P, N)
                ga = _abi.gemm_args(x.data_ptr(), W.data_ptr(), y.data_ptr(), P, N, K, group_m=4)
                recs.append((f"prefill/{name}", _abi.BODY_GEMM_BF16, _abi.gemm_grid(P, N), ga, 2.0 * P * N * K))
                flops += 2.0 * prompt_tokens * N * K
        return recs, flops

    def solo_step(self, device: int = 0):
        from .runtime import solo_launch
        for sid, body, grid, args, _ in self.records:
            solo_launch(device, sid, body, grid, args)

    # ---- plain torch fp32 reference of the same step (numerics tests) ----
    @torch.no_grad()
    def reference_step(self, tokens: torch.Tensor, kc, vc):
        """fp32 torch restatement of one step; returns (logits, h_final, next tokens)."""
        c = self.cfg
        bf = torch.bfloat16
        h = self.embed[tokens.long()].clone()
        kc = [k.clone() for k in kc]
        vc = [v.clone() for v in vc]
        for l in range(c.layers):
            r = torch.rsqrt(h.float().pow(2).sum(-1) / c.d + c.eps)
            qkv = (h.float() @ self.Wqkv[l].float().t()) * r[:, None]
            q = qkv[:, :c.d].to(bf)
            kc[l][:, :, c.L - 1] = qkv[:, c.d:c.d + self.kv_dim].to(bf).view(32, c.n_kv, 128)
            vc[l][:, :, c.L - 1] = qkv[:, c.d + self.kv_dim:].to(bf).view(32, c.n_kv, 128)
            Q = q.float().view(32, c.n_kv, 4, 128)
            K = kc[l][:, :, :c.L].float()
            V = vc[l][:, :, :c.L].float()
            s = torch.einsum("bhqd,bhpd->bhqp", Q, K) / math.sqrt(128)
            o = torch.einsum("bhqp,bhpd->bhqd", torch.softmax(s, -1), V)
            attn = o.reshape(32, c.d).to(bf)
            hmid = (h.float() + attn.float() @ self.Wo[l].float().t()).to(bf)
            r2 = torch.rsqrt(hmid.float().pow(2).sum(-1) / c.d + c.eps)
            gu = (hmid.float() @ self.Wgu[l].float().t()) * r2[:, None]
            gu = gu.view(32, -1, 2, 64)
            act = (torch.nn.functional.silu(gu[:, :, 0]) * gu[:, :, 1]).reshape(32, c.ffn).to(bf)
            h = (hmid.float() + act.float() @ self.Wd[l].float().t()).to(bf)
        rf = torch.rsqrt(h.float().pow(2).sum(-1) / c.d + c.eps)
        logits = ((h.float() @ self.lm.float().t()) * rf[:, None]).to(bf)
        return logits, h, logits.float().argmax(-1).to(torch.int32)


class OutputChecksum:
    """Per-launch checksum of an output buffer (DS_BODY_CHECKSUM): appended
    to a record, launch seq writes slot seq % cap, so every co-located launch
    of a long run can be compared with a plain-grid solo run of the same
    inputs.  value = sum_i w_i * (2i + 1) mod 2^64 over the buffer's 32-bit
    words w_i (integer: independent of scheduling)."""

    def __init__(self, buf: torch.Tensor, cap: int = 16384, grid: int = 64):
        self.buf, self.cap, self.grid = buf, cap, grid
        self.n_words = buf.numel() * buf.element_size() // 4
        self.partials = torch.zeros(cap * grid, dtype=torch.int64, device=buf.device)
        self.args = _abi.ChecksumArgs(buf.data_ptr(), self.partials.data_ptr(), self.n_words, cap, 0)

    def register(self, dom, semantic_id: str, phase=_abi.OTHER) -> int:
        return dom.kernel(semantic_id, _abi.BODY_CHECKSUM, (self.grid, 1, 1), self.args, phase=phase)

    def slots(self):
        """uint64 checksum per slot (device partials summed on the host)."""
        import numpy as np
        p = self.partials.cpu().numpy().view(np.uint64).reshape(self.cap, self.grid)
        with np.errstate(over="ignore"):
            return p.sum(axis=1, dtype=np.uint64)

    def of_seq(self, slots, seq: int) -> int:
        return int(slots[seq % self.cap])

    @staticmethod
    def host(buf: torch.Tensor) -> int:
        """The same checksum computed on the host (numpy, independent of the body)."""
        import numpy as np
        w = buf.contiguous().reshape(-1).cpu().view(torch.int32).numpy().view(np.uint32).astype(np.uint64)
        m = 2 * np.arange(w.size, dtype=np.uint64) + 1
        with np.errstate(over="ignore"):
            return int((w * m).sum(dtype=np.uint64))


class TrainGemm:
    """One training-step contraction: C = A . B^T, bf16 in, fp32 accumulate."""

    def __init__(self, M=8192, N=8192, K=8192, device="cuda", seed=1):
        g = torch.Generator(device=device).manual_seed(seed)
        self.M, self.N, self.K = M, N, K
        self.A = (torch.rand(M, K, device=device, generator=g) * 2 - 1).to(torch.bfloat16)
        self.B = (torch.rand(N, K, device=device, generator=g) * 2 - 1).to(torch.bfloat16)
        self.C = torch.zeros(M, N, device=device, dtype=torch.bfloat16)
        # 32-row tile groups: the ~296 concurrently claimed tiles share A/B
        # panels in L2 (scripts/perf_gemm.py GM sweep)
        self.args = _abi.gemm_args(self.A.data_ptr(), self.B.data_ptr(), self.C.data_ptr(), M, N, K, group_m=32)
        self.grid = _abi.gemm_grid(M, N)
        self.flops = 2.0 * M * N * K

    def register(self, dom, phase=_abi.TRAINING, abandon: bool = False) -> int:
        args = self.args
        if abandon:
            args = _abi.gemm_args(self.A.data_ptr(), self.B.data_ptr(), self.C.data_ptr(), self.M, self.N, self.K,
                                  group_m=32, abandon=True)
        return dom.kernel("train/gemm_bf16", _abi.BODY_GEMM_BF16, self.grid, args, phase=phase)


# ---------------------------------------------------------------------------
# Config 4: ResNet-50-shaped training kernel stream
# ---------------------------------------------------------------------------
def resnet50_convs(batch: int = 128, image: int = 224):
    """The 53 convolutions + FC of ResNet-50 (v1.5: stride on the 3x3) as
    (name, Cin, Cout, k, H_in, H_out) with H the square spatial size."""
    convs = [("conv1", 3, 64, 7, image, image // 2)]
    h = image // 4  # after the stride-2 max-pool
    cin = 64
    for stage, (width, blocks) in enumerate(((64, 3), (128, 4), (256, 6), (512, 3))):
        out = width * 4
        for blk in range(blocks):
            stride = 2 if (blk == 0 and stage > 0) else 1
            ho = h // stride
            nm = f"s{stage + 2}b{blk}"
            convs.append((nm + "_1x1a", cin, width, 1, h, h))
            convs.append((nm + "_3x3", width, width, 3, h, ho))
            convs.append((nm + "_1x1b", width, out, 1, ho, ho))
            if blk == 0:
                convs.append((nm + "_proj", cin, out, 1, h, ho))
            cin = out
            h = ho
    return convs


def _round(x: int, m: int) -> int:
    return (x + m - 1) // m * m


def resnet50_gemms(batch: int = 128, image: int = 224):
    """Implicit-GEMM shapes of one training iteration (forward, data-gradient
    and weight-gradient of every conv + the FC layer), in execution order:
    forward front to back, then backward back to front (wgrad before dgrad).
    Each entry (name, M, N, K) with true (unpadded) sizes; conv1's dgrad (the
    input-image gradient) is not computed, as in any training framework."""
    convs = resnet50_convs(batch, image)
    fwd, bwd = [], []
    for name, ci, co, k, hi, ho in convs:
        fwd.append((name + "/fwd", batch * ho * ho, co, ci * k * k))
    fwd.append(("fc/fwd", batch, 1000, 2048))
    bwd.append(("fc/wgrad", 1000, 2048, batch))
    bwd.append(("fc/dgrad", batch, 2048, 1000))
    for name, ci, co, k, hi, ho in reversed(convs):
        bwd.append((name + "/wgrad", co, ci * k * k, batch * ho * ho))
        if name != "conv1":
            bwd.append((name + "/dgrad", batch * hi * hi, ci, co * k * k))
    return fwd + bwd


def plan_gemm(M: int, N: int, K: int, workers: int = WORKERS, wide: bool = None):
    """Tile width and split-K for a padded GEMM: the widest tile giving >= one
    wave of logical blocks; else (wide) the widest tile whose split-K still
    fills a wave with >= 8 k-blocks per split -- wider tiles re-read the A
    panel from L2 fewer times -- or the narrowest that divides N; split K
    while the grid is short of a wave and every split keeps >= 8 k-blocks."""
    if wide is None:
        wide = os.environ.get("DS_RESNET_WIDE", "0") != "0"
    Mp, Kp = _round(M, 128), _round(K, 64)
    Np = _round(N, 64)
    choices = [bn for bn in (256, 128, 64) if Np % bn == 0]
    full = [b for b in choices if (Mp // 128) * (Np // b) >= workers]
    fill = [b for b in choices if (Mp // 128) * (Np // b) * ((Kp // 64) // 8) >= workers]
    bn = full[0] if full else (fill[0] if wide and fill else choices[-1])
    tiles = (Mp // 128) * (Np // bn)
    splits = 1
    if tiles < workers:
        splits = max(1, min(256, -(-workers // tiles), (Kp // 64) // 8))
    return Mp, Np, Kp, bn, splits


def plan_tiles(Mp: int, Np: int, Kp: int, bn: int, splits: int, workers: int = WORKERS, max_tiles: int = 8):
    """Multi-tile blocks for the tall, short-K GEMMs of the stream (gemm_multi):
    with no split-K, K <= 1152 (at most 18 k-blocks per tile, where the
    per-block overhead rivals the tile's bytes) and at least two waves of
    tiles, T consecutive raster tiles per block with T chosen to leave >= 2
    blocks per worker lane (load balance), capped at max_tiles.  The tile
    narrows to 128 columns (two TMEM accumulators per lane), only for
    K <= 256 (profiles/r2_resnet_multi_tile_ab.txt: past that the second
    read of each A panel costs more than the block overhead saved).  Returns
    (bn, T); T = 1 keeps the one-tile record."""
    if splits > 1 or Kp > 1152 or max_tiles < 2:
        return bn, 1
    if bn > 128 and Kp > 256:  # narrowing re-reads A from L2 twice; measured slower past K = 256
        return bn, 1
    bn2 = min(bn, 128)
    if Np % bn2:
        return bn, 1
    tiles = (Mp // 128) * (Np // bn2)
    T = min(max_tiles, tiles // (2 * workers))
    return (bn2, T) if T >= 2 else (bn, 1)


class ResNetStream:
    """One ResNet-50 training iteration (batch 128, 224^2, bf16) as a stream of
    tcgen05 GEMM launches (+ split-K folds), one per conv pass.  Operands are
    padded to tile multiples and share three arenas (contents are synthetic;
    shapes, flops and launch order are ResNet-50's)."""

    def __init__(self, batch: int = 128, image: int = 224, device="cuda", seed: int = 2, max_tiles=None):
        self.gemms = resnet50_gemms(batch, image)
        self.batch = batch
        self.flops = sum(2.0 * M * N * K for _, M, N, K in self.gemms)  # algorithmic (unpadded)
        # each GEMM may run as C or C^T (operands swapped): take the
        # orientation with the smaller padded output (e.g. weight gradients
        # with 64 output channels would waste half of every 128-row tile)
        def orient(M, N):
            pad = lambda m, n: _round(m, 128) * _round(n, 64)  # noqa: E731
            return (N, M) if pad(N, M) < pad(M, N) else (M, N)
        self.gemms = [(name,) + orient(M, N) + (K,) for name, M, N, K in self.gemms]
        plans = [plan_gemm(M, N, K) for _, M, N, K in self.gemms]
        # measured per-GEMM (tile width, split-K) for the split-K GEMMs
        # (scripts/autotune_resnet.py -> resnet_plan.json); DS_RESNET_TUNED=0 ignores it
        tuned_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "resnet_plan.json")
        self._tuned_tiles = {}
        if os.environ.get("DS_RESNET_TUNED", "1") != "0" and os.path.exists(tuned_path):
            import json
            tuned = json.load(open(tuned_path))
            for i, (name, M, N, K) in enumerate(self.gemms):
                t = tuned.get(name)
                Mp, Np, Kp, bn, sp = plans[i]
                if t and Np % t["bn"] == 0 and (t["splits"] == 1 or (Kp // 64) // t["splits"] >= 1):
                    plans[i] = (Mp, Np, Kp, int(t["bn"]), int(t["splits"]))
                    self._tuned_tiles[name] = int(t.get("tiles", 0))
        self.padded_flops = sum(2.0 * Mp * Np * Kp for Mp, Np, Kp, _, _ in plans)
        a_el = max(Mp * Kp for Mp, Np, Kp, _, _ in plans)
        b_el = max(Np * Kp for Mp, Np, Kp, _, _ in plans)
        c_el = max(Mp * Np for Mp, Np, Kp, _, _ in plans)
        ws_el = max((_abi.splitk_ws_elems(Mp, Np, bn, s) if s > 1 else 0) for Mp, Np, Kp, bn, s in plans)
        g = torch.Generator(device=device).manual_seed(seed)
        self.A = (torch.rand(a_el, device=device, generator=g) * 2 - 1).to(torch.bfloat16)
        self.B = (torch.rand(b_el, device=device, generator=g) * 2 - 1).to(torch.bfloat16)
        self.C = torch.zeros(c_el, device=device, dtype=torch.bfloat16)
        self.ws = torch.zeros(max(1, ws_el), device=device, dtype=torch.float32)
        self.records = []  # (semantic_id, body, grid, args, flops)
        # multi-tile blocks for the tall short-K GEMMs (max tiles per block;
        # DS_RESNET_TILES=1 keeps every GEMM on one-tile blocks)
        max_t = int(os.environ.get("DS_RESNET_TILES", "4")) if max_tiles is None else max_tiles
        fold_wide = os.environ.get("DS_RESNET_FOLD_WIDE", "1") != "0"
        # split-K GEMMs with at most fuse_max splits fold inside the GEMM (the
        # last-arriving split of each tile), each with a private workspace so
        # its at-rest tickets are never overwritten by another GEMM's partials
        fuse_max = int(os.environ.get("DS_RESNET_FUSE_FOLD", "0"))
        self._fold_ws = []
        self.tiles = []
        for (name, M, N, K), (Mp, Np, Kp, bn, s) in zip(self.gemms, plans):
            tt = self._tuned_tiles.get(name, 0)
            bn, T = (bn, tt) if tt else plan_tiles(Mp, Np, Kp, bn, s, max_tiles=max_t)
            self.tiles.append((bn, T))
            # true extents: the TMA loads never read the tile padding (conv1's
            # K = 147 of 192, its 147 weight-gradient rows of 256, FC's 1000)
            fuse = 1 < s <= fuse_max
            ws_ptr = self.ws.data_ptr() if s > 1 else 0
            if fuse:
                w = torch.zeros(_abi.splitk_ws_elems(Mp, Np, bn, s) + _abi.fold_tickets(Mp, Np, bn), device=device)
                self._fold_ws.append(w)
                ws_ptr = w.data_ptr()
            ga = _abi.gemm_args(self.A.data_ptr(), self.B.data_ptr(), self.C.data_ptr(), Mp, Np, Kp, bn=bn,
                                splits=s, ws=ws_ptr, tiles=T, fuse_fold=fuse,
                                valid=None if os.environ.get("DS_RESNET_PADDED") else (M, N, K))
            self.records.append((f"resnet/{name}", _abi.BODY_GEMM_BF16, _abi.gemm_grid(Mp, Np, bn, s, T), ga,
                                 2.0 * M * N * K))
            if s > 1 and not fuse:
                rows = _abi.fold_rows(Mp, Np, bn, WORKERS) if fold_wide else 16
                ra, rg = _abi.splitk_reduce(self.ws.data_ptr(), self.C.data_ptr(), Mp, Np, Kp, 16, bn, s, rows)
                self.records.append((f"resnet/{name}/fold", _abi.BODY_SPLITK_REDUCE, rg, ra, 0.0))
        self.plans = plans

    def register(self, dom, phase=_abi.TRAINING) -> List[int]:
        return [dom.kernel(sid, body, grid, args, phase=phase) for sid, body, grid, args, _ in self.records]

    def bound_s(self, tflops: float, hbm_gbs: float) -> float:
        """Roofline lower bound of one iteration: per GEMM (true sizes) the
        larger of flops / bf16 peak and (A + B + C) bytes / HBM peak, summed.
        Most of the stream's GEMMs are HBM-bound at batch 128 (K = 64..576
        against M = 100k..1.6M rows), so this is the honest denominator."""
        return sum(max(2.0 * M * N * K / (tflops * 1e12), 2.0 * (M * K + N * K + M * N) / (hbm_gbs * 1e9))
                   for _, M, N, K in self.gemms)
