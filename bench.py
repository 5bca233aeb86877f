"""Benchmark: BASELINE config 2 on B200 — two tenants on one GPU.

  decode tenant  : Llama-3-8B-shaped decode step, batch 32, KV length 1024,
                   bf16, 163 launches/step (HBM-bound; tcgen05 swap-AB GEMV)
  training tenant: bf16 GEMM 8192^3 per iteration on tcgen05/TMEM

A *step* = one decode request of T tokens arriving while the training tenant
runs continuously.  Both sharing policies run the same kernels through the
same coroutine executor:
  tpot-first : spatial SM quotas (reference TpotFirstPolicy) + idle-SM lending
  temporal   : time slicing, full GPU per quantum (reference TemporalBaselinePolicy)

value = P99 TPOT (ms) under tpot-first (reference metric: TPOT per request =
(last decode finish - first decode finish) / (tokens - 1), nearest-rank P99,
proj/src/io/metrics.cpp:9-52).  Lower is better.  Device timing is
%globaltimer on record completions (the executor is one persistent kernel, so
CUDA events cannot bracket sub-regions of it); bit-exactness vs solo is checked
on the step outputs.
"""
from __future__ import annotations

import argparse
import bisect
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from fractions import Fraction

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "co-located P99 TPOT + train throughput vs time-slicing; bit-exact vs solo"
UNIT = "ms (P99 TPOT, decode tenant)"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")


def log(*a):
    print(f"[bench {time.strftime('%H:%M:%S')}]", *a, file=sys.stderr, flush=True)


def nearest_rank(samples, pct):
    """metrics.cpp:9-16: k = ceil(pct/100 * n), 1-indexed."""
    s = sorted(samples)
    k = max(1, (pct * len(s) + 99) // 100)
    return s[k - 1]


def p99_tpot_ms(outcomes, check=None):
    """P99 TPOT through the runtime's ds_compute_metrics (the reference's
    compute_metrics over device timestamps); cross-checked against the
    Python nearest rank of the same samples."""
    from paper_2603_15042_b200.metrics import compute_metrics
    m = compute_metrics(outcomes, makespan_ns=1)
    v = float(m["tpot"]["p99"]) / 1e6
    if check is not None:
        assert abs(v - nearest_rank(check, 99)) < 1e-9, (v, nearest_rank(check, 99))
    return v


def ncu_traffic(kernel):
    """dram__bytes_read+write per launch of this body from the committed ncu
    capture (profiles/r1_ncu_summary.json), or None."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "r1_ncu_summary.json")))["kernels"]
        key = {"decode/attn": "attn", "decode/gate_up": "gate_up", "decode/lm_head": "lm_head",
               "train/gemm_bf16": "gemm"}.get(kernel)
        return int(d[key]["traffic_bytes"]) if key in d else None
    except Exception:
        return None


def load_peaks():
    try:
        p = json.load(open(PEAKS_PATH))
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_gpu{gpu}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def _guarded(fn):
    """A run that raises must not leave its policy engine polling a domain
    that is about to be stopped and destroyed: stop the feeder thread, stop
    and close the engine, reset the control word, then re-raise."""
    def w(self, *a, **k):
        self._cur_eng = self._cur_stop = self._cur_th = None
        try:
            return fn(self, *a, **k)
        except BaseException:
            if self._cur_stop is not None:
                self._cur_stop.set()
            if self._cur_th is not None:
                self._cur_th.join(timeout=10)
            if self._cur_eng is not None:
                try:
                    self._cur_eng.stop()
                    self._cur_eng.close()
                except Exception:
                    pass
            try:
                self.dom.set_lend(-1)
                self.dom.quota_set([-1] * self.dom.num_sms)
            except Exception:
                pass
            raise
    w.__name__ = fn.__name__
    w.__doc__ = fn.__doc__
    return w


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
class Colocation:
    def __init__(self, device, tokens_per_req, kv_len, layers=32, decode_sat=Fraction(1, 2), slo_x=8.0,
                 tiers=(Fraction(1, 4), Fraction(3, 4), Fraction(1)), prefill_mix=False, abandon=False):
        import torch
        from paper_2603_15042_b200 import _abi
        from paper_2603_15042_b200.runtime import Domain
        from paper_2603_15042_b200.tenants import DecodeConfig, DecodeModel, TrainGemm
        self.torch, self._abi = torch, _abi
        self.device = device
        torch.cuda.set_device(device)
        self.T = tokens_per_req
        self.model = DecodeModel(DecodeConfig(L=kv_len, layers=layers), device=f"cuda:{device}")
        self.decode_sat = decode_sat
        self.slo_x = slo_x
        self.train = TrainGemm(device=f"cuda:{device}")
        # prefill mix (config 4b): a second chat stream (its own model state)
        # and both streams' prefill GEMM records, built before the executor
        # owns the SMs
        self.model2 = None
        if prefill_mix:
            self.model2 = DecodeModel(DecodeConfig(L=kv_len, layers=layers), device=f"cuda:{device}", seed=1)
            self.pf_recs = [self.model.prefill_records(256), self.model2.prefill_records(256)]
        torch.cuda.synchronize()
        # pool: decode binds 3/4 (smallest tier >= its fair share 1/2), training 1/4;
        # idle SMs are lent to training.  (With a 1/2 tier, the reference
        # SLO-aware rule can defer a bound decode forever once it predicts a
        # TPOT miss: upgrades count the vctx's own tier — SURVEY 8-appendix #2.)
        self.tiers = [Fraction(t) for t in tiers]
        self.dom = Domain(device, tiers=self.tiers, block_log_capacity=int(os.environ.get("DS_BENCH_BLOG", "0")),
                          lend_idle_sms=True)
        self.t_dec = self.dom.tenant("decode", _abi.LATENCY_CRITICAL)
        self.t_trn = self.dom.tenant("train", _abi.BEST_EFFORT)
        self.dec_kernels = self.model.register(self.dom)
        # optional: the step as TPOT-First would run it on its 1/2 tier, with
        # gate_up as two-slab and the LM head as seven-slab blocks (one wave
        # each on 148 worker lanes; bit-identical outputs).  Measured co-located
        # (profiles/r2_half_tier_variants_ab.txt): gate_up two-slab +0.18 ms
        # P50 TPOT, LM head seven-slab neutral — off by default
        hv = os.environ.get("DS_HALF_VARIANTS", "0")
        self.dec_kernels_half = self.model.register_variant(self.dom, self.dec_kernels, "" if hv == "0" else hv)
        self.gemm_kernel = self.train.register(self.dom)
        # parity evidence at full size: a per-launch checksum of the decode
        # step's logits and of the training GEMM's C, appended to the records
        # of the pinned run (run(pin=True)) and compared with plain-grid solo
        # runs of the same inputs after the executor stops (pin_check)
        from paper_2603_15042_b200.tenants import OutputChecksum
        self.ck_logits = OutputChecksum(self.model.logits, cap=16384, grid=32)
        self.ck_C = OutputChecksum(self.train.C, cap=32768, grid=64)
        self.k_ck_logits = self.ck_logits.register(self.dom, "decode/logits_checksum", phase=_abi.DECODE)
        self.k_ck_C = self.ck_C.register(self.dom, "train/C_checksum", phase=_abi.TRAINING)
        # optionally the same GEMM with sub-block yields (tiles give up within
        # a few k-blocks when revoked; bit-identical results), per run
        self.gemm_kernel_plain = self.gemm_kernel
        self.gemm_kernel_abandon = None
        if abandon:
            self.dom.set_abandonable(self.t_trn)
            self.gemm_kernel_abandon = self.train.register(self.dom, abandon=True)
        self.resnet = None
        if self.model2 is not None:
            self.t_dec2 = self.dom.tenant("decode2", _abi.LATENCY_CRITICAL)
            self.dec2_kernels = self.model2.register(self.dom)
            self.pf_kernels = [[self.dom.kernel(sid, body, grid, args, phase=_abi.PREFILL)
                                for sid, body, grid, args, _ in recs] for recs, _ in self.pf_recs]
        self.dom.start()

    def add_resnet(self):
        """Config 4 training tenant: the ResNet-50-shaped kernel stream."""
        from paper_2603_15042_b200.tenants import ResNetStream
        self.resnet = ResNetStream(device=f"cuda:{self.device}")
        self.t_res = self.dom.tenant("resnet", self._abi.BEST_EFFORT)
        self.res_kernels = self.resnet.register(self.dom)
        dom = self.dom
        dom.quota_set(dom.mask(self.t_res, 0, dom.num_sms))
        for _ in range(2):
            for k in self.res_kernels:
                last = dom.launch(self.t_res, k)
        dom.wait(self.t_res, last)
        cs = [c for c in dom.poll(1 << 20) if c.tenant == self.t_res]
        n = len(self.res_kernels)
        self.res_iter_ns = cs[-1].t_end - cs[-n].t_first_claim
        dom.quota_set([-1] * dom.num_sms)
        return self.res_iter_ns / 1e6

    @_guarded
    def run_bursty(self, policy, arrivals_ns, tokens, step_ns, quantum_ms=5.0, tpot_slo_ns=0, ttft_slo_ns=0):
        """Config 4: bursty decode requests (arrivals from the reference's
        gen_burst) co-located with the ResNet-50 training stream.  Returns
        per-request TTFT / TPOT / latency, SLO violation rates (metrics.cpp
        definitions) and training images/s."""
        from paper_2603_15042_b200.runtime import Engine
        _abi, dom = self._abi, self.dom
        lend = self.t_res if policy != "temporal" else -1
        eng = Engine(dom, policy=policy, quantum_ns=int(quantum_ms * 1e6), lend_tenant=lend, fair_handover=True)
        jd = eng.add_job(self.t_dec, _abi.LATENCY_CRITICAL)
        jt = eng.add_job(self.t_res, _abi.BEST_EFFORT)
        dom.set_lend(lend)
        self._cur_eng = eng
        eng.start()
        stop = threading.Event()
        self._cur_stop = stop
        train_recs = []

        def trainer():
            outstanding = []
            while not stop.is_set():
                while len(outstanding) < 2:
                    r = eng.submit(jt, self.res_kernels, "resnet/iter", _abi.TRAINING, grid_size=len(self.res_kernels),
                                   base_hint_ns=self.res_iter_ns, saturation=Fraction(1))
                    outstanding.append(r)
                    train_recs.append(r)
                outstanding = [r for r in outstanding if eng.record(r).state != 2]
                time.sleep(0.0005)

        th = threading.Thread(target=trainer, daemon=True)
        self._cur_th = th
        th.start()
        time.sleep(0.05)
        t0 = eng.now() + 10_000_000
        tpot_slo = tpot_slo_ns or int(self.slo_x * step_ns)
        ttft_slo = ttft_slo_ns or int(4 * self.slo_x * step_ns)
        reqs = []
        for i, a in enumerate(arrivals_ns):
            while eng.now() < t0 + a:
                time.sleep(0.0001)
            arr = eng.now()
            recs = [eng.submit(jd, self.dec_kernels, "decode/step", _abi.DECODE, grid_size=len(self.dec_kernels),
                               request=i, decode_index=k, request_arrival_ns=arr, ttft_ns=ttft_slo, tpot_ns=tpot_slo,
                               base_hint_ns=step_ns, saturation=self.decode_sat) for k in range(tokens)]
            reqs.append((arr, recs))
        for _, recs in reqs:
            eng.wait(recs[-1], timeout_ms=120000)
        stop.set()
        th.join()
        for r in train_recs:
            eng.wait(r)
        out = []
        for arr, recs in reqs:
            inf = [eng.record(r) for r in recs]
            out.append({"ttft_ms": (inf[0].finish_host_ns - arr) / 1e6,
                        "tpot_ms": (inf[-1].t_end - inf[0].t_end) / (tokens - 1) / 1e6,
                        "latency_ms": (inf[-1].finish_host_ns - arr) / 1e6,
                        "w0": inf[0].t_first_claim, "w1": inf[-1].t_end})
        w0 = min(o["w0"] for o in out)
        w1 = max(o["w1"] for o in out)
        iters = 0.0
        for ti in (eng.record(r) for r in train_recs):
            a, b = ti.t_first_claim, ti.t_end
            if b > a:
                iters += max(0, min(b, w1) - max(a, w0)) / (b - a)
        counters = eng.counters()
        eng.stop()
        eng.close()
        dom.set_lend(-1)
        dom.quota_set([-1] * dom.num_sms)
        win_s = (w1 - w0) * 1e-9
        return {"requests": len(out), "p99_tpot_ms": round(nearest_rank([o["tpot_ms"] for o in out], 99), 3),
                "p99_ttft_ms": round(nearest_rank([o["ttft_ms"] for o in out], 99), 3),
                "p99_latency_ms": round(nearest_rank([o["latency_ms"] for o in out], 99), 3),
                "train_images_per_s": round(iters * self.resnet.batch / win_s, 1),
                "train_tflops": round(iters * self.resnet.flops / win_s / 1e12, 1),
                "tpot_slo_violation_rate": round(sum(o["tpot_ms"] * 1e6 > tpot_slo for o in out) / len(out), 4),
                "ttft_slo_violation_rate": round(sum(o["ttft_ms"] * 1e6 > ttft_slo for o in out) / len(out), 4),
                "slo_ms": {"tpot": tpot_slo / 1e6, "ttft": ttft_slo / 1e6},
                "window_ms": round(win_s * 1e3, 1), "engine_counters": counters}

    def close(self):
        self.dom.stop()  # the registered records stay valid for solo replays

    def release(self):
        self.dom.close()

    # solo calibration through the executor with the whole GPU
    def solo(self, steps):
        dom, _abi = self.dom, self._abi
        dom.quota_set(dom.mask(self.t_dec, 0, dom.num_sms))
        for _ in range(2):
            for k in self.dec_kernels:
                last = dom.launch(self.t_dec, k)
        dom.wait(self.t_dec, last)
        dom.poll(1 << 16)
        for _ in range(steps):
            for k in self.dec_kernels:
                last = dom.launch(self.t_dec, k)
        dom.wait(self.t_dec, last)
        cs = [c for c in dom.poll(1 << 20) if c.tenant == self.t_dec]
        n = len(self.dec_kernels)
        ends = [cs[(i + 1) * n - 1].t_end for i in range(steps)]
        step_ns = [(ends[i] - ends[i - 1]) for i in range(1, steps)]
        # per-kernel device time: the launch's full span, first claim to last
        # retire (it includes the early-start window in which its blocks
        # stream weights while the previous launch finishes, so it is never
        # shorter than the kernel's share of the step)
        per_kernel = {}
        for i, c in enumerate(cs):
            sid = self.model.records[i % n][0]
            per_kernel.setdefault(sid, []).append(c.t_end - c.t_first_claim)
        dom.quota_set(dom.mask(self.t_trn, 0, dom.num_sms))
        for _ in range(3):
            last = dom.launch(self.t_trn, self.gemm_kernel)
        dom.wait(self.t_trn, last)
        dom.poll(1 << 16)
        n_gemm = 20
        for _ in range(n_gemm):
            last = dom.launch(self.t_trn, self.gemm_kernel)
        dom.wait(self.t_trn, last)
        gs = [c for c in dom.poll(1 << 16) if c.tenant == self.t_trn]
        # throughput over back-to-back launches (consecutive GEMMs overlap at
        # the launch boundary through early start): span / launches
        gemm_ms = (gs[-1].t_end - gs[0].t_first_claim) / 1e6 / n_gemm
        self.gemm_ns = gemm_ms * 1e6
        dom.quota_set([-1] * dom.num_sms)
        return {"decode_step_ms": statistics.median(step_ns) / 1e6, "gemm_ms": gemm_ms,
                "per_kernel_ns": {k: statistics.mean(v) for k, v in per_kernel.items()},
                "per_kernel_launches": {k: len(v) // steps for k, v in per_kernel.items()}}

    @_guarded
    def run(self, policy, requests, warmup, solo, e2e=False, quantum_ms=5.0, pin=False):
        """Co-located run: returns per-request TPOT (ms), training TFLOP/s in
        the timed window, and engine counters.

        e2e: the host token loop — every step's input tokens go H2D from
        pinned host memory and the sampled tokens come back D2H.
        pin: every decode record also checksums its logits and every training
        record its C (DS_BODY_CHECKSUM, one slot per launch); the step inputs
        and launch sequence numbers are kept for pin_check()."""
        from paper_2603_15042_b200.runtime import Engine
        _abi, torch = self._abi, self.torch
        from paper_2603_15042_b200.metrics import RequestOutcome
        dom = self.dom
        lend = self.t_trn if policy != "temporal" and os.environ.get("DS_BENCH_LEND", "1") != "0" else -1
        eng = Engine(dom, policy=policy, quantum_ns=int(quantum_ms * 1e6), lend_tenant=lend, fair_handover=True)
        jd = eng.add_job(self.t_dec, _abi.LATENCY_CRITICAL)
        jt = eng.add_job(self.t_trn, _abi.BEST_EFFORT)
        dom.set_lend(lend)
        step_ns = int(solo["decode_step_ms"] * 1e6)
        gemm_ns = int(solo["gemm_ms"] * 1e6)
        tpot_slo = int(self.slo_x * step_ns)
        ttft_slo = int(2 * self.slo_x * step_ns)
        period = int(2 * self.T * step_ns)  # decode busy ~50% of the time when solo
        half = policy == "tpot-first" and self.decode_sat <= Fraction(1, 2)
        base = self.dec_kernels_half if half else self.dec_kernels
        dec_kernels = base + ([self.k_ck_logits] if pin else [])
        trn_kernels = [self.gemm_kernel] + ([self.k_ck_C] if pin else [])
        self._cur_eng = eng
        eng.start()
        stop = threading.Event()
        self._cur_stop = stop
        train_recs = []

        def trainer():
            # keep 2 training iterations queued at all times
            outstanding = []
            while not stop.is_set():
                while len(outstanding) < 2:
                    r = eng.submit(jt, trn_kernels, "train/gemm_bf16", _abi.TRAINING, grid_size=2048,
                                   base_hint_ns=gemm_ns, saturation=Fraction(1, 4))
                    outstanding.append(r)
                    train_recs.append(r)
                outstanding = [r for r in outstanding if eng.record(r).state != 2]
                time.sleep(0.0002)

        th = threading.Thread(target=trainer, daemon=True)
        self._cur_th = th
        th.start()
        time.sleep(0.05)
        pinned_tok = torch.zeros(32, dtype=torch.int32).pin_memory()
        pinned_tok.copy_(self.model.tokens)  # contiguous D2H (copy engine): the first step's input
        results = []
        pin_steps = []  # (request, step, input tokens, record)
        t_next = eng.now() + period // 4
        log(f"run {policy} e2e={e2e} pin={pin}: {warmup}+{requests} requests, period {period/1e6:.2f} ms, "
            f"step {step_ns/1e6:.2f} ms")
        for req in range(warmup + requests):
            # open-loop arrival at a fixed period
            while eng.now() < t_next:
                time.sleep(0.0002)
            arrival = eng.now()
            recs = []
            host_tok_times = []
            for tok in range(self.T):
                if e2e:
                    # host buffers: H2D the step input tokens, D2H the sampled tokens
                    self.model.tokens.copy_(pinned_tok, non_blocking=True)
                    torch.cuda.current_stream().synchronize()
                tok_in = pinned_tok.clone() if pin else None
                r = eng.submit(jd, dec_kernels, "decode/step", _abi.DECODE, grid_size=len(self.dec_kernels),
                               request=req, decode_index=tok, request_arrival_ns=arrival, ttft_ns=ttft_slo,
                               tpot_ns=tpot_slo, base_hint_ns=step_ns, saturation=self.decode_sat)
                recs.append(r)
                if pin:
                    pin_steps.append((req, tok, tok_in, r))
                if e2e:
                    eng.wait(r)
                    pinned_tok.copy_(self.model.tokens, non_blocking=True)
                    torch.cuda.current_stream().synchronize()
                    host_tok_times.append(time.perf_counter_ns())
            try:
                eng.wait(recs[-1], timeout_ms=60000)
            except Exception:
                log("TIMEOUT", policy, "req", req, eng.counters(), [eng.record(r).state for r in recs])
                log(dom.debug())
                raise
            infos = [eng.record(r) for r in recs]
            firsts = infos[0].t_end
            lasts = infos[-1].t_end
            tpot = (lasts - firsts) / (self.T - 1) / 1e6
            ttft = (infos[0].t_end - infos[0].t_first_claim) / 1e6
            e2e_tpot = ((host_tok_times[-1] - host_tok_times[0]) / (self.T - 1) / 1e6) if e2e else None
            gaps = [(infos[i + 1].t_first_claim - infos[i].t_end) / 1e3 for i in range(self.T - 1)]
            steps_ms = [(i.t_end - i.t_first_claim) / 1e6 for i in infos[1:]]
            if req % 10 == 9 or req < 2:
                log(f"  req {req}: tpot {tpot:.3f} ms (step {statistics.mean(steps_ms):.3f} ms, "
                    f"host gap {statistics.mean(gaps):.1f} us)")
            results.append({"tpot_ms": tpot, "first_ms": ttft, "t0": infos[0].t_first_claim, "t1": lasts,
                            "outcome": RequestOutcome(arrival=infos[0].t_first_claim, first_decode_finish=firsts,
                                                      last_finish=lasts, output_tokens=self.T),
                            "gap_us": statistics.mean(gaps), "step_ms": statistics.mean(steps_ms),
                            "e2e_tpot_ms": e2e_tpot, "preempted": sum(i.preempted for i in infos)})
            t_next = arrival + period
        stop.set()
        th.join()
        # drain training
        for r in train_recs:
            eng.wait(r)
        timed = results[warmup:]
        w0 = timed[0]["t0"]
        w1 = timed[-1]["t1"]
        tinfos = [eng.record(r) for r in train_recs]
        # training work inside the window: completed GEMMs weighted by overlap
        done_flop = 0.0
        gemm_durs = []
        for ti in tinfos:
            a, b = ti.t_first_claim, ti.t_end
            if b <= a:
                continue
            ov = max(0, min(b, w1) - max(a, w0))
            done_flop += self.train.flops * ov / (b - a)
            gemm_durs.append(b - a)
        pin_data = None
        if pin:
            pin_data = {"steps": [(q, k, t, eng.record(r).last_seq) for q, k, t, r in pin_steps],
                        "train": [(ti.t_first_claim, ti.t_end, ti.last_seq) for ti in tinfos],
                        "request_starts": [r["t0"] for r in results],
                        "logit_slots": self.ck_logits.slots(), "C_slots": self.ck_C.slots()}
        counters = eng.counters()
        ledger = eng.ledger()
        # normalized throughput (add_normalization, metrics.cpp:81-102): per
        # job, exclusive span / shared span over the timed window; exclusive
        # spans from the measured solo durations of the same work (training:
        # its completed GEMMs back to back; decode: the same request starts,
        # each request T solo steps)
        from paper_2603_15042_b200.runtime import add_normalization
        tw = [ti for ti in tinfos if ti.t_first_claim >= w0 and ti.t_end <= w1]
        norm = None
        if tw:
            t_shared = (min(t.t_first_claim for t in tw), max(t.t_end for t in tw))
            t_solo = (0, int(len(tw) * gemm_ns))
            starts = [r["t0"] for r in timed]
            d_shared = (starts[0], w1)
            d_solo = (starts[0], starts[-1] + self.T * step_ns)
            vals, agg = add_normalization([d_shared, t_shared], [d_solo, t_solo])
            norm = {"decode": round(float(vals[0]), 4), "train": round(float(vals[1]), 4), "aggregate": round(agg, 4)}
        eng.stop()
        eng.close()
        dom.set_lend(-1)
        dom.quota_set([-1] * dom.num_sms)
        return {"tpot_ms": [r["tpot_ms"] for r in timed], "e2e_tpot_ms": [r["e2e_tpot_ms"] for r in timed],
                "ledger": ledger, "normalized_throughput": norm,
                "outcomes": [r["outcome"] for r in timed],
                "kernels_completed": len(timed) * self.T * len(self.dec_kernels) + len(tw),
                "train_launches": len(train_recs),
                "gap_us": statistics.mean(r["gap_us"] for r in timed),
                "step_ms": statistics.mean(r["step_ms"] for r in timed),
                "window_ms": (w1 - w0) / 1e6, "train_tflops": done_flop / ((w1 - w0) * 1e-9) / 1e12,
                "counters": counters, "gemm_ms_median": statistics.median(gemm_durs) / 1e6 if gemm_durs else None,
                "pin": pin_data}

    @_guarded
    def run_prefill_mix(self, policy, arrivals, tokens, step_ns, prefill_ns, tpot_slo_ns, ttft_slo_ns, quantum_ms=5.0):
        """Config 4b: two chat streams (requests alternate between them), each
        request a prefill record (256 prompt tokens: 128 tcgen05 GEMMs) then
        `tokens` decode steps, beside the training GEMM.  This is where
        TPOT-First differs from the default policy: a prefill is admitted only
        if the running decodes keep their TPOT (policies.cpp:184-204)."""
        from paper_2603_15042_b200.runtime import Engine
        _abi, dom = self._abi, self.dom
        lend = self.t_trn if policy != "temporal" else -1
        eng = Engine(dom, policy=policy, quantum_ns=int(quantum_ms * 1e6), lend_tenant=lend, fair_handover=True)
        jobs = [eng.add_job(self.t_dec, _abi.LATENCY_CRITICAL), eng.add_job(self.t_dec2, _abi.LATENCY_CRITICAL)]
        jt = eng.add_job(self.t_trn, _abi.BEST_EFFORT)
        dec = [self.dec_kernels, self.dec2_kernels]
        dom.set_lend(lend)
        self._cur_eng = eng
        eng.start()
        stop = threading.Event()
        self._cur_stop = stop
        train_recs = []

        def trainer():
            outstanding = []
            while not stop.is_set():
                while len(outstanding) < 2:
                    r = eng.submit(jt, [self.gemm_kernel], "train/gemm_bf16", _abi.TRAINING, grid_size=2048,
                                   base_hint_ns=int(self.gemm_ns), saturation=Fraction(1, 4))
                    outstanding.append(r)
                    train_recs.append(r)
                outstanding = [r for r in outstanding if eng.record(r).state != 2]
                time.sleep(0.0005)

        th = threading.Thread(target=trainer, daemon=True)
        self._cur_th = th
        th.start()
        time.sleep(0.05)
        t0 = eng.now() + 10_000_000
        reqs = []
        for i, (a, stream) in enumerate(arrivals):
            while eng.now() < t0 + a:
                time.sleep(0.0001)
            arr = eng.now()
            j = jobs[stream]
            pf = eng.submit(j, self.pf_kernels[stream], "prefill/default", _abi.PREFILL, grid_size=1, request=i,
                            request_arrival_ns=arr, ttft_ns=ttft_slo_ns, tpot_ns=tpot_slo_ns, base_hint_ns=prefill_ns,
                            saturation=Fraction(9, 10))
            recs = [eng.submit(j, dec[stream], "decode/step", _abi.DECODE, grid_size=len(dec[stream]), request=i,
                               decode_index=k, request_arrival_ns=arr, ttft_ns=ttft_slo_ns, tpot_ns=tpot_slo_ns,
                               base_hint_ns=step_ns, saturation=self.decode_sat) for k in range(tokens)]
            reqs.append((arr, pf, recs))
        try:
            for _, _, recs in reqs:
                eng.wait(recs[-1], timeout_ms=120000)
            stop.set()
            th.join()
            for r in train_recs:
                eng.wait(r, timeout_ms=120000)
        except Exception:
            log("TIMEOUT prefill mix", policy, eng.counters(),
                [(eng.record(pf).state, [eng.record(r).state for r in recs]) for _, pf, recs in reqs],
                [eng.record(r).state for r in train_recs])
            log(dom.debug())
            raise
        out = []
        for arr, pf, recs in reqs:
            inf = [eng.record(r) for r in recs]
            out.append({"ttft_ms": (inf[0].finish_host_ns - arr) / 1e6,  # first decode completion (metrics.cpp:46)
                        "tpot_ms": (inf[-1].t_end - inf[0].t_end) / (tokens - 1) / 1e6,
                        "w0": eng.record(pf).t_first_claim, "w1": inf[-1].t_end})
        w0, w1 = min(o["w0"] for o in out), max(o["w1"] for o in out)
        done = 0.0
        for ti in (eng.record(r) for r in train_recs):
            a, b = ti.t_first_claim, ti.t_end
            if b > a:
                done += self.train.flops * max(0, min(b, w1) - max(a, w0)) / (b - a)
        counters = eng.counters()
        eng.stop()
        eng.close()
        dom.set_lend(-1)
        dom.quota_set([-1] * dom.num_sms)
        tp, tt = [o["tpot_ms"] for o in out], [o["ttft_ms"] for o in out]
        return {"requests": len(out), "p99_tpot_ms": round(nearest_rank(tp, 99), 3),
                "p99_ttft_ms": round(nearest_rank(tt, 99), 3),
                "tpot_slo_violation_rate": round(sum(x * 1e6 > tpot_slo_ns for x in tp) / len(tp), 4),
                "ttft_slo_violation_rate": round(sum(x * 1e6 > ttft_slo_ns for x in tt) / len(tt), 4),
                "train_tflops": round(done / ((w1 - w0) * 1e-9) / 1e12, 1), "engine_counters": counters}

    def solo_kernel_times(self, steps=3):
        """After the executor stopped: every decode kernel as a plain-grid
        solo launch (ds_solo_launch) in step order on one stream, each
        bracketed by CUDA events on that stream (serialised like the ncu
        launch list; every launch streams its own layer's weights, so the L2
        holds none of them).  Returns {sid: mean us}, and the sum per step."""
        torch, m = self.torch, self.model
        stream = torch.cuda.current_stream()
        times = {}
        for it in range(steps + 1):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(m.records) + 1)]
            # hold the stream while the host enqueues the step, so no event
            # pair includes host launch latency
            torch.cuda._sleep(100_000_000)
            ev[0].record(stream)
            # registered records: device-resident args, no host sync per launch
            for i, k in enumerate(self.dec_kernels):
                self.dom.solo(k, stream.cuda_stream)
                ev[i + 1].record(stream)
            torch.cuda.synchronize()
            if it == 0:
                continue  # warm-up
            for i, (sid, _, _, _, _) in enumerate(m.records):
                times.setdefault(sid, []).append(ev[i].elapsed_time(ev[i + 1]) * 1e3)
        per = {k: statistics.mean(v) for k, v in times.items()}
        step_us = sum(per[sid] for sid, _, _, _, _ in m.records)
        return per, step_us

    def pin_check(self, pin, requests=5):
        """After the executor stopped: replay decode steps of the pinned
        co-located run as plain-grid solo launches (ds_solo_launch, the
        exclusive baseline) from the same input tokens, and one solo training
        GEMM, and compare with the co-located launches' checksums.
        Checked: every step of the last `requests` timed requests (logits),
        and every training iteration whose checksum slot survived (C),
        counting those a decode request started during (revoked mid-flight:
        the decode tenant took SMs the GEMM was running on)."""
        import numpy as np
        from paper_2603_15042_b200 import _abi
        from paper_2603_15042_b200.runtime import solo_launch
        from paper_2603_15042_b200.tenants import OutputChecksum
        torch, m = self.torch, self.model
        steps = pin["steps"]
        last_req = max(q for q, _, _, _ in steps)
        sel = [x for x in steps if x[0] > last_req - requests]
        max_seq = max(s for _, _, _, s in steps)
        dec_ok, dec_n = True, 0
        for q, k, tok_in, seq in sel:
            if seq <= max_seq - self.ck_logits.cap:
                continue  # slot reused by a later step
            m.tokens.copy_(tok_in)
            m.solo_step(self.device)
            torch.cuda.synchronize()
            want = OutputChecksum.host(m.logits)
            got = self.ck_logits.of_seq(pin["logit_slots"], seq)
            dec_ok &= (want == got)
            dec_n += 1
        # one solo GEMM of the same operands into a separate output
        C_solo = torch.zeros_like(self.train.C)
        a = _abi.gemm_args(self.train.A.data_ptr(), self.train.B.data_ptr(), C_solo.data_ptr(), self.train.M,
                           self.train.N, self.train.K, group_m=32)
        solo_launch(self.device, "train/gemm_bf16", _abi.BODY_GEMM_BF16, self.train.grid, a)
        torch.cuda.synchronize()
        want_c = OutputChecksum.host(C_solo)
        c_final_equal = bool(torch.equal(C_solo.view(torch.int16), self.train.C.view(torch.int16)))
        tr = pin["train"]
        max_tseq = max(s for _, _, s in tr)
        starts = sorted(pin["request_starts"])
        gemm_ok, gemm_n, revoked = True, 0, 0
        for t0, t1, seq in tr:
            if seq <= max_tseq - self.ck_C.cap:
                continue
            gemm_ok &= (self.ck_C.of_seq(pin["C_slots"], seq) == want_c)
            gemm_n += 1
            i = bisect.bisect_right(starts, t0)
            if i < len(starts) and starts[i] < t1:
                revoked += 1
        return {"decode_logits_equal": bool(dec_ok), "decode_steps_checked": dec_n,
                "gemm_C_equal": bool(gemm_ok) and c_final_equal, "gemm_launches_checked": gemm_n,
                "gemm_launches_revoked_midflight": revoked,
                "how": "co-located launches' per-launch checksums (DS_BODY_CHECKSUM) vs plain-grid ds_solo_launch "
                       "replays of the same inputs (host checksum); decode: every step of the last "
                       f"{requests} timed requests of the e2e run; training: every iteration of that run",
                "ok": bool(dec_ok and gemm_ok and c_final_equal and dec_n > 0 and gemm_n > 0)}


def reference_sim(solo, requests, tokens, policy="tpot-first", scale=1, slo_x=8.0):
    """Time the reference simulator (corosim SimEngine, oracle/_ref) on the
    same two-tenant scenario, time unit = 1 us, calibrated with the measured
    solo durations and the GPU arm's SLOs (TPOT slo_x x step, TTFT twice
    that).  Returns (simulated P99 TPOT ms, wall s, events).

    Bandwidth demands sum to 1 (decode 0.75 + training 0.25): with an
    oversubscribed HBM (sum > 1) the reference's own work-conservation check
    `assert(run.work_done == k.base_duration)` (src/engine/engine.cpp:838)
    fails for this scenario — see DESIGN.md "Reference quirks"."""
    from oracle import loader
    step_us = max(1, int(solo["decode_step_ms"] * 1000))
    gemm_us = max(1, int(solo["gemm_ms"] * 1000))
    period_us = 2 * tokens * step_us
    n_req = requests * scale
    recs = [{"arrival_time": "0", "job_id": "train", "kind": "training",
             "iterations": int(n_req * period_us / gemm_us) + 4, "priority": "best_effort", "profile": "gemm"}]
    for r in range(n_req):
        recs.append({"arrival_time": str(period_us // 4 + r * period_us), "job_id": "chat", "kind": "inference",
                     "prompt_tokens": 8, "output_tokens": tokens, "priority": "latency_critical",
                     "slo": {"ttft": str(int(2 * slo_x * step_us)), "tpot": str(int(slo_x * step_us))}})
    sc = {"devices": [{"tiers": ["0.25", "0.5", "0.75", "1"]}], "policy": policy,
          "policy_params": {"quantum": "5000"},
          "segments_per_kernel": 16, "event_budget": 100000000,
          "profiles": {"inference": {"default": {"decode_cost": str(step_us), "prefill_cost_per_token": "1",
                                                 "decode_saturation": "0.75", "decode_mem_bound": "0.8",
                                                 "decode_bw_demand": "0.75", "decode_grid": 163}},
                       "training": {"gemm": {"iteration_cost": str(gemm_us), "saturation": "0.25",
                                             "mem_bound": "0.1", "bw_demand": "0.25", "grid": 2048}}},
          "workload": {"records": recs}}
    out = json.loads(loader.ref_simulate(json.dumps(sc)))
    p99 = out["metrics"]["tpot"].get("p99")
    return (float(p99) / 1000.0 if p99 is not None else None), out["wall_ns"] / 1e9, out["events"]


def cpu_baseline_leg(solo, requests, tokens, budget_s=10.0):
    """The reference's CPU implementation of the path — the corosim
    simulator (oracle/_ref, compiled from the reference sources) — timed on
    this host's core on the same two-tenant scenario, scaled until it does
    ~budget_s of CPU work.  value = wall ms it spends per simulated decode
    step (token); its own prediction of the P99 TPOT is reported beside it."""
    scale = 1
    p99, wall, ev = reference_sim(solo, requests, tokens, scale=scale)
    while wall < budget_s / 2 and scale < 4096:
        scale = max(scale + 1, int(scale * min(16.0, budget_s / max(wall, 1e-3))))
        p99, wall, ev = reference_sim(solo, requests, tokens, scale=scale)
    steps = requests * scale * tokens
    return {"value": round(wall * 1e3 / steps, 5), "unit": "ms wall per simulated decode step (1 core)",
            "cores": 1, "kind": "reference",
            "sample": f"corosim SimEngine::simulate (oracle/_ref, compiled from the reference) of the config-2 "
                      f"tpot-first scenario: {requests * scale} requests x {tokens} tokens beside the training "
                      f"GEMM stream, {ev} events in {wall:.2f} s wall",
            "sim_predicted_p99_tpot_ms": p99,
            "note": "the reference models the decode step (slowdown model, speed.cpp:5-12) instead of computing it; "
                    "its predicted TPOT is calibrated with this run's measured solo durations"}


def _ref_timed(sc, reps_budget_s=2.0, equivalence=False):
    """simulate (and optionally check_immutable_equivalence) of one reference
    scenario, repeated until ~reps_budget_s of CPU work; per-run wall time."""
    from oracle import loader
    text = json.dumps(sc)
    runs, wall, out, eq = 0, 0.0, None, None
    while runs == 0 or (wall < reps_budget_s and runs < 20):
        out = json.loads(loader.ref_simulate(text))
        wall += out["wall_ns"] / 1e9
        if equivalence:
            eq = json.loads(loader.ref_equivalence(text))
            wall += eq["wall_ns"] / 1e9
        runs += 1
    return out, eq, wall / runs, runs


def cpu_reference_configs(c1_solo_us, step_us, gemm_us, resnet_iter_us):
    """the reference simulator (oracle/_ref, 1 host core) timed
    on each config's scenario beside the GPU numbers.  Time unit 1 us,
    calibrated with the measured B200 durations."""
    import multiprocessing
    out = {}
    # config 1: one SGEMM kernel (256 logical blocks, a yield point per
    # block); a soft hang at 30% is detected (3x prediction) and the kernel
    # is quarantined 1 -> 1/4 mid-run: the reference's quota change
    c1 = max(1, int(c1_solo_us))
    sc1 = {"devices": [{"tiers": ["0.25", "1"]}], "policy": "slo-aware", "segments_per_kernel": 256,
           "hang_detection": True,
           "faults": [{"kind": "soft_hang", "pctx": 1, "time": str(int(0.3 * c1)), "stretch": "10"}],
           "profiles": {"training": {"sgemm": {"iteration_cost": str(c1), "saturation": "1", "mem_bound": "0.1",
                                               "grid": 256}}},
           "workload": {"records": [{"arrival_time": "0", "job_id": "sgemm", "kind": "training", "iterations": 1,
                                     "priority": "best_effort", "profile": "sgemm"}]}}
    r, eq, per, runs = _ref_timed(sc1, equivalence=True)
    out["config1"] = {"wall_us_per_run": round(per * 1e6, 1), "runs": runs, "cores": 1,
                      "equivalent": eq["equivalent"], "kernels_completed": r["kernels_completed"],
                      "sim_preemptions": r["preemptions"],
                      "what": "simulate + check_immutable_equivalence (J+1 runs) of the SGEMM scenario"}
    # config 3: periodic switching between two tenants (temporal policy with
    # quantum = period); the model's preempt ledger beside the measured yields
    rows = []
    for period in (50, 200, 1000, 5000):
        sc3 = {"devices": [{"tiers": ["0.25", "1"]}], "policy": "temporal", "policy_params": {"quantum": str(period)},
               "segments_per_kernel": 16,
               "profiles": {"training": {"g": {"iteration_cost": str(gemm_us), "saturation": "1", "grid": 2048}}},
               "workload": {"records": [
                   {"arrival_time": "0", "job_id": "a", "kind": "training", "iterations": 8, "priority": "best_effort",
                    "profile": "g"},
                   {"arrival_time": "0", "job_id": "b", "kind": "training", "iterations": 8, "priority": "best_effort",
                    "profile": "g"}]}}
        r, _, per, runs = _ref_timed(sc3, reps_budget_s=0.5)
        ov = r["metrics"].get("overheads", {})
        rows.append({"period_us": period, "wall_us_per_run": round(per * 1e6, 1), "runs": runs,
                     "preemptions": ov.get("preemptions"), "preempt_total_us": ov.get("preempt_total"),
                     "migrations": ov.get("migrations"), "ctx_switches": ov.get("ctx_switches")})
    out["config3"] = {"cores": 1, "sweep": rows,
                      "what": "temporal-policy scenario per period (the reference has no quota timer; its "
                              "time-sliced owner change is the closest periodic switch). It shows 0 preemptions: "
                              "a bound holder keeps the full tier across quanta (SURVEY 8-appendix #1)"}
    # config 4: the ResNet-50 training stream (one kernel per iteration at the
    # measured iteration time) beside bursty decode (same gen_burst stream)
    from paper_2603_15042_b200 import workload as wl
    reqs = wl.gen_burst(0.5, 4.0, 2.0, 20.0, 60.0, wl.RequestTemplate(output_tokens=4), seed=0)
    unit = 50_000  # us per trace time unit, as the GPU leg
    recs = [{"arrival_time": "0", "job_id": "resnet", "kind": "training",
             "iterations": int(60 * unit / max(1, resnet_iter_us)) + 2, "priority": "best_effort",
             "profile": "resnet"}]
    for i, q in enumerate(reqs):
        recs.append({"arrival_time": str(int(q.arrival_q * unit // 10**9)), "job_id": "chat", "kind": "inference",
                     "prompt_tokens": 8, "output_tokens": 4, "priority": "latency_critical",
                     "slo": {"ttft": "150000", "tpot": str(3 * step_us)}})
    sc4 = {"devices": [{"tiers": ["0.25", "0.5", "0.75", "1"]}], "policy": "tpot-first", "segments_per_kernel": 16,
           "event_budget": 100000000,
           "profiles": {"inference": {"default": {"decode_cost": str(step_us), "prefill_cost_per_token": "1",
                                                  "decode_saturation": "0.75", "decode_mem_bound": "0.8",
                                                  "decode_bw_demand": "0.75", "decode_grid": 163}},
                        "training": {"resnet": {"iteration_cost": str(resnet_iter_us), "saturation": "0.25",
                                                "mem_bound": "0.3", "bw_demand": "0.25", "grid": 161}}},
           "workload": {"records": recs}}
    r, _, per, runs = _ref_timed(sc4, reps_budget_s=2.0)
    tp = r["metrics"]["tpot"].get("p99")
    out["config4"] = {"wall_ms_per_run": round(per * 1e3, 2), "runs": runs, "cores": 1, "requests": len(reqs),
                      "sim_p99_tpot_ms": float(tp) / 1000 if tp is not None else None, "events": r["events"]}
    # config 5: one 8-device engine with the 16-tenant mix, and 8 per-device
    # engines on 8 threads (ctypes releases the GIL inside the call)
    def mix(devs, jobs_per_dev):
        recs = []
        for j in range(jobs_per_dev * devs):
            if j % 2 == 0:
                for r_ in range(8):
                    recs.append({"arrival_time": str(1000 + r_ * 8 * step_us * 2), "job_id": f"chat{j}",
                                 "kind": "inference", "prompt_tokens": 8, "output_tokens": 8,
                                 "priority": "latency_critical", "slo": {"ttft": str(8 * step_us), "tpot": str(3 * step_us)}})
            else:
                recs.append({"arrival_time": "0", "job_id": f"train{j}", "kind": "training", "iterations": 100,
                             "priority": "best_effort", "profile": "gemm"})
        recs.sort(key=lambda x: int(x["arrival_time"]))
        return {"devices": [{"tiers": ["0.25", "0.5", "0.75", "1"]} for _ in range(devs)], "policy": "tpot-first",
                "segments_per_kernel": 16, "event_budget": 100000000,
                "profiles": {"inference": {"default": {"decode_cost": str(step_us), "prefill_cost_per_token": "1",
                                                       "decode_saturation": "0.5", "decode_grid": 163}},
                             "training": {"gemm": {"iteration_cost": str(gemm_us), "saturation": "0.5",
                                                   "grid": 2048}}},
                "workload": {"records": recs}}
    r, _, per, runs = _ref_timed(mix(8, 2), reps_budget_s=2.0)
    from concurrent.futures import ThreadPoolExecutor
    import time as _t
    t0 = _t.perf_counter()
    with ThreadPoolExecutor(8) as ex:
        list(ex.map(lambda _: _ref_timed(mix(1, 2), reps_budget_s=0.0), range(8)))
    par = _t.perf_counter() - t0
    out["config5"] = {"one_engine_8_devices_ms": round(per * 1e3, 2), "runs": runs, "events": r["events"],
                      "eight_engines_on_8_threads_ms": round(par * 1e3, 2), "nproc": multiprocessing.cpu_count(),
                      "cores": 8}
    return out


def config4b_leg(co, args, solo):
    """Two chat streams with prefill (256-token prompts) + the training GEMM:
    TPOT-First vs the reference default (slo-aware) vs time slicing, in P99
    TPOT / TTFT and SLO violation rates (the paper's TPOT-First comparison,
    PAPER.md:457-458)."""
    from paper_2603_15042_b200 import workload as wl
    dom, _abi = co.dom, co._abi
    # prefill's solo duration on the whole GPU (predictor hint)
    dom.quota_set(dom.mask(co.t_dec, 0, dom.num_sms))
    for _ in range(2):
        for k in co.pf_kernels[0]:
            last = dom.launch(co.t_dec, k)
    dom.wait(co.t_dec, last)
    cs = [c for c in dom.poll(1 << 20) if c.tenant == co.t_dec]
    n = len(co.pf_kernels[0])
    prefill_ns = cs[-1].t_end - cs[-n].t_first_claim
    dom.quota_set([-1] * dom.num_sms)
    step_ns = int(solo["decode_step_ms"] * 1e6)
    reqs = wl.gen_burst(0.5, 4.0, 2.0, 20.0, args.burst_units, wl.RequestTemplate(output_tokens=4, streams=2), seed=1)
    arrivals = [(int(r.arrival_q * 50.0 * 1e-3), r.stream) for r in reqs]
    # TPOT SLO 3x the solo step: with tighter SLOs the reference SLO-aware
    # rule (inherited by TPOT-First) defers a bound decode forever once it
    # predicts a miss it cannot fix at its tier
    tpot_slo, ttft_slo = 3 * step_ns, 150_000_000
    log(f"config 4b: {len(arrivals)} requests over 2 streams, prefill solo {prefill_ns / 1e6:.2f} ms")
    res = {p: co.run_prefill_mix(p, arrivals, 4, step_ns, prefill_ns, tpot_slo, ttft_slo, quantum_ms=args.quantum_ms)
           for p in ("tpot-first", "slo-aware", "temporal")}
    return {"workload": "config 4b: two chat streams (batch-32 Llama-3-8B-shaped decode each; requests alternate, "
                        "gen_burst arrivals) with 256-token prefill (128 tcgen05 GEMMs) before 4 decode steps, "
                        "beside the bf16 GEMM 8192^3 training tenant",
            "prefill_solo_ms": round(prefill_ns / 1e6, 3), "slo_ms": {"tpot": tpot_slo / 1e6, "ttft": ttft_slo / 1e6},
            "tpot_first": res["tpot-first"], "slo_aware": res["slo-aware"], "temporal": res["temporal"]}


def config4_leg(co, args, solo, peaks):
    """Config 4: the ResNet-50-shaped training stream co-located with bursty
    decode requests (gen_burst arrivals), TPOT-First vs time slicing."""
    from paper_2603_15042_b200 import workload as wl
    res_ms = co.add_resnet()
    unit_ms = 50.0
    reqs = wl.gen_burst(0.5, 4.0, 2.0, 20.0, args.burst_units, wl.RequestTemplate(output_tokens=4), seed=0)
    arrivals = [int(r.arrival_q * unit_ms * 1e-3) for r in reqs]  # arrival_q = round(t*1e9) -> ns
    step_ns = int(solo["decode_step_ms"] * 1e6)
    log(f"config 4: {len(arrivals)} bursty requests, resnet solo iter {res_ms:.2f} ms")
    # SLOs tight enough to separate the policies: TPOT 3x the solo decode
    # step, TTFT 150 ms (the paper's TPOT-First-vs-Default comparison is in
    # SLO violation rates)
    slo = dict(tpot_slo_ns=3 * step_ns, ttft_slo_ns=150_000_000)
    c4 = {p: co.run_bursty(p, arrivals, 4, step_ns, quantum_ms=args.quantum_ms, **slo)
          for p in ("tpot-first", "slo-aware", "temporal")}
    return {"workload": "config 4: ResNet-50-shaped training stream (53 convs + FC, fwd/dgrad/wgrad = 161 "
                        "tcgen05 GEMMs + split-K folds per iteration, batch 128, 224^2, bf16) co-located with "
                        "bursty decode requests (4 tokens each)",
            "arrivals": f"gen_burst(base 0.5, burst 4.0, burst_duration 2, period 20, duration "
                        f"{args.burst_units}) x {unit_ms} ms/unit (trace.cpp:204-232), seed 0",
            "resnet_solo_iter_ms": round(res_ms, 3),
            "resnet_solo_images_per_s": round(co.resnet.batch / (res_ms * 1e-3), 1),
            "roofline": {"bound": "tensor", "kernel": "train/resnet50 iteration (161 GEMMs + folds)",
                         "achieved": round(co.resnet.flops / (res_ms * 1e-3) / 1e12, 1),
                         "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                         "frac": round(co.resnet.flops / (res_ms * 1e-3) / 1e12 / peaks["bf16_tflops"], 4),
                         "padded_frac": round(co.resnet.padded_flops / (res_ms * 1e-3) / 1e12 / peaks["bf16_tflops"], 4),
                         "stream_bound_ms": round(co.resnet.bound_s(peaks["bf16_tflops"], peaks["hbm_gbs"]) * 1e3, 3),
                         "frac_of_stream_bound": round(co.resnet.bound_s(peaks["bf16_tflops"], peaks["hbm_gbs"]) * 1e3
                                                       / res_ms, 4),
                         "what": "algorithmic (unpadded) conv/FC flops of one fwd+dgrad+wgrad iteration over its "
                                 "solo time on the executor (full GPU); padded_frac counts the flops of the "
                                 "128-row-tiled GEMMs actually issued; stream_bound_ms sums per GEMM "
                                 "max(flops / bf16 peak, bytes / HBM peak) (most of the stream is HBM-bound)"},
            "tpot_first": c4["tpot-first"], "slo_aware": c4["slo-aware"], "temporal": c4["temporal"]}


def decode_roofline(co, solo, solo_us, solo_step_us, peaks, peaks_src):
    """HBM roofline of the decode tenant.

    Per kernel: algorithmic bytes per launch / the kernel's mean duration as a
    plain-grid solo launch timed with CUDA events on its stream (solo_us:
    serialised in step order, like the ncu launch list, so shares of the step
    agree with profiles/).  The dominant kernel (largest share of the step) is
    the line's roofline.  Beside it: the same kernels' full spans inside the
    executor (first claim -> last retire, %globaltimer; spans of consecutive
    launches overlap through early start), and the whole step on the executor
    at 148 SMs (algorithmic bytes per step / step time)."""
    m = co.model
    kn, nl = solo["per_kernel_ns"], solo["per_kernel_launches"]
    bytes_by = {sid: b for sid, _, _, _, b in m.records}
    table = {}
    for sid in solo_us:
        gbs = bytes_by[sid] / (solo_us[sid] * 1e3)  # bytes/ns = GB/s
        table[sid] = {"launches_per_step": nl[sid], "bytes": bytes_by[sid], "solo_us": round(solo_us[sid], 2),
                      "gbs": round(gbs, 1), "frac": round(gbs / peaks["hbm_gbs"], 4),
                      "share_of_solo_step": round(solo_us[sid] * nl[sid] / solo_step_us, 4),
                      "executor_span_us": round(kn[sid] / 1e3, 2)}
    top = max(table, key=lambda k: table[k]["share_of_solo_step"])
    step_gbs = m.step_bytes / (solo["decode_step_ms"] * 1e6)
    return {"bound": "hbm", "kernel": top, "achieved": table[top]["gbs"], "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": table[top]["frac"], "traffic": ncu_traffic(top), "algorithmic_bytes": bytes_by[top],
            "peak_source": peaks_src,
            "timing": "mean duration of the kernel as a plain-grid solo launch, CUDA events on its stream, "
                      "launches serialised in decode-step order (the ncu launch-list setting)",
            "step": {"bytes": m.step_bytes, "executor_ms": round(solo["decode_step_ms"], 4),
                     "gbs": round(step_gbs, 1), "frac": round(step_gbs / peaks["hbm_gbs"], 4),
                     "solo_serialised_ms": round(solo_step_us / 1e3, 4),
                     "floor_ms": round(m.step_bytes / peaks["hbm_gbs"] / 1e6, 4)},
            "per_kernel": table}


def paired_report(a, b):
    from paper_2603_15042_b200 import metrics as M
    from paper_2603_15042_b200 import report as R

    def one(run):
        m = M.compute_metrics(run["outcomes"], makespan_ns=int(run["window_ms"] * 1e6),
                              kernels_completed=run.get("kernels_completed", 0))
        n = run.get("normalized_throughput")
        return R.metrics_to_json(m, run["ledger"], {0: Fraction(str(n["decode"])), 1: Fraction(str(n["train"]))} if n else None)

    return R.compare(one(a), one(b), "config2", "tpot-first", "config2", "temporal")


def gpu_arm(args, rank, world):
    import torch
    dev = int(os.environ.get("LOCAL_RANK", rank))
    peaks, peaks_src = load_peaks()
    log("building tenants")
    co = Colocation(dev, args.tokens, args.kv_len, layers=args.layers, decode_sat=Fraction(args.decode_sat),
                    slo_x=args.slo_x, tiers=[Fraction(t) for t in args.tiers.split(",")],
                    prefill_mix=not args.no_config4b)
    solo = co.solo(steps=max(3, args.warmup))
    log("solo", {k: v for k, v in solo.items() if k != "per_kernel_ns" and k != "per_kernel_launches"})
    if args.only_config4b:
        try:
            r = config4b_leg(co, args, solo)
        except Exception as e:
            r = {"error": repr(e)}
        co.close()
        print(json.dumps({"config4b": r}))
        sys.exit(0)
    # one bench step = args.rps requests (P99 over steps x rps samples)
    n_req, n_warm = args.steps * args.rps, args.warmup * args.rps
    with ClockSampler(dev) as clk:
        sp = co.run("tpot-first", n_req, n_warm, solo)
        tm = co.run("temporal", n_req, n_warm, solo, quantum_ms=args.quantum_ms)
    clocks = clk.summary()
    # time slicing with a finer quantum (lower latency, more switches): the
    # comparison must not hinge on one quantum choice
    tm_fine = co.run("temporal", args.steps * 2, args.warmup, solo, quantum_ms=args.quantum_ms / 5)
    # the end-to-end run through the host token loop is also the pinned run:
    # every decode step's logits and every training GEMM's C checksummed
    e2e = co.run("tpot-first", n_req, n_warm, solo, e2e=True, pin=True)
    config4b = None
    if not args.no_config4b:
        try:
            config4b = config4b_leg(co, args, solo)
        except Exception as e:  # an auxiliary leg must not cost the headline line
            config4b = {"error": repr(e)}
    config4 = None
    if not args.no_config4:
        try:
            config4 = config4_leg(co, args, solo, peaks)
        except Exception as e:  # an auxiliary leg must not cost the headline line
            config4 = {"error": repr(e)}
    co.close()
    exact = co.pin_check(e2e["pin"])
    log("bit-exact vs solo:", exact)
    solo_us, solo_step_us = co.solo_kernel_times()
    co.release()
    p99 = p99_tpot_ms(sp["outcomes"], sp["tpot_ms"])
    p99_tm = p99_tpot_ms(tm["outcomes"], tm["tpot_ms"])
    p99_e2e = nearest_rank(e2e["e2e_tpot_ms"], 99)
    m = co.model
    roof = decode_roofline(co, solo, solo_us, solo_step_us, peaks, peaks_src)
    gemm_tf = co.train.flops / (solo["gemm_ms"] * 1e6) / 1e3  # flop/ns -> TFLOP/s
    out = {
        "metric": METRIC, "value": round(p99, 4), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(sp["window_ms"] / args.steps, 3), "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights, random tokens)",
        "config": {"workload": "config 2: Llama-3-8B-shaped decode (batch 32, KV 1024, 32 layers) + bf16 GEMM "
                               "8192^3 training tenant on 1 B200", "policy": "tpot-first (+idle-SM lending)",
                   "baseline_policy": f"temporal (time slicing, quantum {args.quantum_ms} ms)", "tiers": args.tiers,
                   "decode_saturation": args.decode_sat, "step": f"{args.rps} decode requests",
                   "tokens_per_request": args.tokens, "requests_timed": n_req, "requests_warmup": n_warm,
                   "global_batch": 32, "seq_len": args.kv_len, "parallelism": f"independent domain per GPU x{world}",
                   "l2": "inputs larger than L2 (15 GB weights + 4.3 GB KV per step, 384 MB GEMM operands)"},
        "solo": {"decode_step_ms": round(solo["decode_step_ms"], 4), "gemm_ms": round(solo["gemm_ms"], 4),
                 "gemm_tflops": round(gemm_tf, 1)},
        "bit_exact_vs_solo": exact["ok"],
        "bit_exact_detail": exact,
        "tpot_distribution_ms": {name: {"p50": round(nearest_rank(v, 50), 4), "p90": round(nearest_rank(v, 90), 4),
                                        "p99": round(nearest_rank(v, 99), 4), "mean": round(statistics.mean(v), 4),
                                        "n": len(v)}
                                 for name, v in (("tpot_first", sp["tpot_ms"]), ("temporal", tm["tpot_ms"]))},
        "engine_counters": sp["counters"],
        "ledger": {"tpot_first": sp["ledger"], "temporal": tm["ledger"],
                   "what": "OverheadLedger from device %globaltimer stamps summed over worker lanes (ns): "
                           "ctx_switch = lane gap between tenants, preempt = control install -> retire of the "
                           "block a revoked lane was running, migration = control install -> a lane's first "
                           "block of its new tenant"},
        "normalized_throughput": {"tpot_first": sp["normalized_throughput"],
                                  "temporal": tm["normalized_throughput"]},
        "e2e": {"value": round(p99_e2e, 4), "unit": UNIT,
                "h2d_bytes_per_step": 32 * 4 * args.tokens * args.rps,
                "d2h_bytes_per_step": 32 * 4 * args.tokens * args.rps,
                "how": "host token loop: per decode step, H2D of the 32 input tokens from pinned memory and D2H "
                       "of the 32 sampled tokens; TPOT from host clocks after each D2H"},
        "roofline": roof,
        "roofline_gemm": {"bound": "tensor", "kernel": "train/gemm_bf16", "achieved": round(gemm_tf, 1),
                          "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                          "frac": round(gemm_tf / peaks["bf16_tflops"], 4), "peak_source": peaks_src,
                          "traffic": ncu_traffic("train/gemm_bf16"), "algorithmic_bytes": 3 * 8192 * 8192 * 2},
        "clocks": clocks,
        # logical launches through the executor in the timed tpot-first run:
        # decode kernels of every step + training GEMM launches
        "gpu_launches": len(m.records) * (n_req + n_warm) * args.tokens + sp.get("train_launches", 0),
        "config4": config4,
        "config4b": config4b,
        # corosim compare (tools/corosim.cpp:99-123) of the two timed runs, in
        # the reference's metrics_to_json schema (times in device ns)
        "compare": paired_report(sp, tm),
    }
    tail = {
        "host_gap_us": round(sp["gap_us"], 1),
        "train_tflops": round(sp["train_tflops"], 1),
        "timeslice": {"p99_tpot_ms": round(p99_tm, 4), "train_tflops": round(tm["train_tflops"], 1),
                      "quantum_ms": args.quantum_ms,
                      "fine_quantum": {"quantum_ms": args.quantum_ms / 5,
                                       "p99_tpot_ms": round(nearest_rank(tm_fine["tpot_ms"], 99), 4),
                                       "train_tflops": round(tm_fine["train_tflops"], 1)}},
    }
    return out, tail, solo


def config1_leg(dev):
    """Config 1: one unmodified SGEMM 1024^3 (fp32 FFMA, 64x64 logical tiles,
    k-ascending fma chain) as a GPU coroutine with a mid-kernel SM-quota change
    (100% -> 25% at 30% of claimed blocks -> 100% at 60%), bit-exact vs its
    solo launch; solo and coroutine device times."""
    import numpy as np
    import torch
    from paper_2603_15042_b200 import _abi
    from paper_2603_15042_b200.runtime import Domain
    M = N = K = 1024
    g = torch.Generator(device=f"cuda:{dev}").manual_seed(1)
    A = torch.rand(M, K, device=f"cuda:{dev}", generator=g) * 2 - 1
    B = torch.rand(K, N, device=f"cuda:{dev}", generator=g) * 2 - 1
    C_solo = torch.zeros(M, N, device=f"cuda:{dev}")
    C_co = torch.zeros(M, N, device=f"cuda:{dev}")
    grid = (N // 64, M // 64, 1)
    a_solo = _abi.SgemmArgs(A.data_ptr(), B.data_ptr(), C_solo.data_ptr(), M, N, K, 0)
    a_co = _abi.SgemmArgs(A.data_ptr(), B.data_ptr(), C_co.data_ptr(), M, N, K, 0)
    with Domain(dev, block_log_capacity=1 << 14) as dom:
        # solo: the same body as a plain grid on a stream (registered args, no per-launch setup)
        ks = dom.kernel("sgemm/solo", _abi.BODY_SGEMM, grid, a_solo)
        stream = torch.cuda.current_stream().cuda_stream
        for _ in range(3):
            dom.solo(ks, stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            dom.solo(ks, stream)
        e1.record()
        torch.cuda.synchronize()
        solo_ms = e0.elapsed_time(e1) / 5
        dom.start()
        t = dom.tenant("sgemm", _abi.BEST_EFFORT)
        dom.quota_set(dom.mask(t, 0, dom.num_sms))
        kid = dom.kernel("sgemm", _abi.BODY_SGEMM, grid, a_co)
        nblk = grid[0] * grid[1]
        for _ in range(2):
            s = dom.launch(t, kid)
        dom.wait(t, s)
        dom.clear_logs()
        dom.poll(1 << 16)
        dom.quota_at_claim(t, s + 1, int(0.3 * nblk), dom.mask(t, 0, dom.num_sms // 4))
        dom.quota_at_claim(t, s + 1, int(0.6 * nblk), dom.mask(t, 0, dom.num_sms))
        s = dom.launch(t, kid)
        dom.wait(t, s)
        c = [x for x in dom.poll(1 << 16) if x.tenant == t][-1]
        blocks = sorted(b.block for b in dom.block_log() if b.tenant == t and b.seq == s)
        switches = len(dom.switch_log())
    exact = bool(np.array_equal(C_co.cpu().numpy().view(np.uint32), C_solo.cpu().numpy().view(np.uint32)))
    co_ms = (c.t_end - c.t_first_claim) / 1e6
    flop = 2.0 * M * N * K
    try:  # measured on this device, no executor resident
        ffma_peak, ffma_src = _abi.measure_ffma_peak(dev), "measured: ds_measure_ffma_peak (8 independent fp32 fma chains per thread, 4 x 256 threads per SM, CUDA events)"
    except Exception as e:  # noqa: BLE001
        ffma_peak, ffma_src = 148 * 128 * 2 * 1.965e9 / 1e12, f"nominal 148 SMs x 128 lanes x 2 x 1965 MHz ({e})"
    ach = flop / (min(solo_ms, co_ms) * 1e-3) / 1e12
    return {"workload": "config 1: SGEMM 1024^3 fp32 (64x64 logical tiles, 256 blocks) as one coroutine, quota "
                        "100% -> 25% at 30% of claimed blocks -> 100% at 60%",
            "bit_exact_vs_solo": exact, "all_blocks_once": blocks == list(range(nblk)),
            "solo_ms": round(solo_ms, 4), "coroutine_ms": round(co_ms, 4), "ctl_switch_records": switches,
            "roofline": {"bound": "fp32 FFMA", "achieved": round(ach, 2), "peak": round(ffma_peak, 1),
                         "unit": "TFLOP/s", "frac": round(ach / ffma_peak, 4),
                         "peak_source": ffma_src}}


def config3_leg(dev):
    """Config 3: SM-quota migration sweep.  The device timer flips a tenant
    between all SMs and a quarter of them every 50 us .. 5 ms; yield / drain
    / grant latency (us) and lost throughput from the device switch log, for
    5-us logical blocks and for the training GEMM's 128x256 tiles; plus the
    host -> device control round trip."""
    import torch
    from paper_2603_15042_b200 import _abi, migration as mg
    from paper_2603_15042_b200.runtime import Domain
    from paper_2603_15042_b200.tenants import TrainGemm
    # 16384 x 16384 x 8192 (~4 ms at the full quota): flips every 50 us .. 5 ms
    # (at 5 ms the launch sees at most one flip);
    # 128x256 tiles (the throughput choice) and 128x64 tiles (4x shorter
    # logical blocks: the latency choice)
    gemm = TrainGemm(M=16384, N=16384, K=8192, device=f"cuda:{dev}", seed=5)
    narrow = _abi.gemm_args(gemm.A.data_ptr(), gemm.B.data_ptr(), gemm.C.data_ptr(), 16384, 16384, 8192, bn=64)
    # the same 128x256 tiles with sub-block yields (abandon within ~4 k-blocks, re-run)
    yielding = _abi.gemm_args(gemm.A.data_ptr(), gemm.B.data_ptr(), gemm.C.data_ptr(), 16384, 16384, 8192,
                              group_m=32, abandon=True)
    spilling = _abi.gemm_args(gemm.A.data_ptr(), gemm.B.data_ptr(), gemm.C.data_ptr(), 16384, 16384, 8192,
                              group_m=32, abandon=2)
    torch.cuda.synchronize()
    rows = []
    with Domain(dev, tiers=[Fraction(1)], block_log_capacity=0, lend_idle_sms=False) as dom:
        t = dom.tenant("migrating", _abi.BEST_EFFORT)
        dom.set_abandonable(t)
        nspin = int(2 * 148 * 2 * 30000 / 5 / 8)  # ~30 ms of 5-us blocks at full quota
        spin = mg.spin_kernel(dom, 5, nspin)
        gk = gemm.register(dom)
        gn = dom.kernel("train/gemm_bf16/bn64", _abi.BODY_GEMM_BF16, _abi.gemm_grid(16384, 16384, 64), narrow,
                        phase=_abi.TRAINING)
        gy = dom.kernel("train/gemm_bf16/abandon", _abi.BODY_GEMM_BF16, gemm.grid, yielding, phase=_abi.TRAINING)
        gsp = dom.kernel("train/gemm_bf16/spill", _abi.BODY_GEMM_BF16, gemm.grid, spilling, phase=_abi.TRAINING)
        dom.start()
        base = mg.run(dom, t, spin, 0)
        for p in (50, 200, 1000, 5000):
            rows.append(dict(unit="spin 5 us", period_us=p, **mg.summarize(mg.run(dom, t, spin, p), base["blocks_per_s"])))
        gemm_rows = {}
        for name, k, tile_flop in (("gemm tile 128x256x8192", gk, 2 * 128 * 256 * 8192),
                                   ("gemm tile 128x64x8192", gn, 2 * 128 * 64 * 8192),
                                   ("gemm tile 128x256x8192 abandonable (restart)", gy, 2 * 128 * 256 * 8192),
                                   ("gemm tile 128x256x8192 abandonable (spill + resume)", gsp, 2 * 128 * 256 * 8192)):
            gbase = mg.run(dom, t, k, 0)
            gemm_rows[name] = {"unflipped_tflops": round(gbase["blocks_per_s"] * tile_flop / 1e12, 1),
                               "block_us": round(1e6 / gbase["blocks_per_s"] * 2 * 148, 1)}
            for p in (50, 200, 1000, 5000):  # 50 us .. 5 ms
                rows.append(dict(unit=name, period_us=p, **mg.summarize(mg.run(dom, t, k, p), gbase["blocks_per_s"])))
        rtt = [x / 1e3 for x in dom.ctl_roundtrip(100)]
    return {"workload": "config 3: quota flips 100% <-> 25% of the SMs by the device timer (no host round trip)",
            "sweep": rows, "gemm_tiles": gemm_rows,
            "host_device_ctl_roundtrip_us": {"p50": round(mg.pct(rtt, .5), 2), "p99": round(mg.pct(rtt, .99), 2)},
            # a host (policy) driven quota change: half the measured round trip
            # (host write -> device install; the ack returns the other half)
            # plus the device-measured grant (install -> the new owner's first
            # block on a granted SM, 5-us blocks)
            "host_driven_migration_us": {
                "p50": round(mg.pct(rtt, .5) / 2 + rows[0]["grant_us_p50"], 2),
                "what": "ctl round trip p50 / 2 (one way, upper bound) + device grant p50 of the 50-us-period row"}}


def config5_leg(args, rank, world, dev, gather_fn):
    """Config 5: the 16-tenant mix (8 decode + 8 training) partitioned over
    the ranks by the native workload-aware placement, plus one data-parallel
    training tenant spanning every rank (GEMM 4096^3 -> gradient all-reduce
    body over peer memory).  Each rank runs its tenants under TPOT-First for
    a fixed window; returns this rank's throughputs and TPOT samples."""
    import torch
    from paper_2603_15042_b200 import _abi, dp
    from paper_2603_15042_b200.placement import config5_mix, place
    from paper_2603_15042_b200.runtime import Domain, Engine
    from paper_2603_15042_b200.tenants import DecodeConfig, DecodeModel, TrainGemm
    mix = config5_mix()
    where = place(mix, world, mem_cap_gb=150.0)
    mine = [mix[i] for i, d in enumerate(where) if d == rank]
    # the only collective of the leg (IPC handle exchange) comes first, before
    # any large allocation that could fail on one rank
    dpg = dp.DpGroup(dev, 4096 * 4096, rank, world, gather_fn)
    dec = [(spec, DecodeModel(DecodeConfig(L=args.kv_len, layers=spec.size), device=f"cuda:{dev}", seed=i))
           for i, spec in enumerate(mine) if spec.kind == "decode"]
    trn = [(spec, TrainGemm(M=spec.size, N=spec.size, K=spec.size, device=f"cuda:{dev}", seed=i))
           for i, spec in enumerate(mine) if spec.kind == "train"]
    dp_gemm = TrainGemm(M=4096, N=4096, K=4096, device=f"cuda:{dev}", seed=99)
    dp_gemm.args = _abi.gemm_args(dp_gemm.A.data_ptr(), dp_gemm.B.data_ptr(), dpg.grad, 4096, 4096, 4096)
    torch.cuda.synchronize()
    tiers = [Fraction(1, 16)] * 8 + [Fraction(1, 8)] * 4 + [Fraction(1, 4)] * 2 + [Fraction(1, 2), Fraction(1)]
    dom = Domain(dev, tiers=tiers, block_log_capacity=0, lend_idle_sms=True)
    td = [(dom.tenant(sp.name, _abi.LATENCY_CRITICAL), m.register(dom), m) for sp, m in dec]
    tt = [(dom.tenant(sp.name, _abi.BEST_EFFORT), [g.register(dom)], g) for sp, g in trn]
    t_dp = dom.tenant("dp_train", _abi.BEST_EFFORT)
    dp_kernels = [dom.kernel("train/dp_gemm", _abi.BODY_GEMM_BF16, dp_gemm.grid, dp_gemm.args, phase=_abi.TRAINING),
                  dpg.register(dom)]
    dom.start()
    eng = Engine(dom, policy="tpot-first", lend_tenant=tt[0][0] if tt else t_dp, fair_handover=True)
    jobs_d = [(eng.add_job(t, _abi.LATENCY_CRITICAL), ks, m) for t, ks, m in td]
    jobs_t = [(eng.add_job(t, _abi.BEST_EFFORT), ks, g.flops) for t, ks, g in tt]
    j_dp = eng.add_job(t_dp, _abi.BEST_EFFORT)
    jobs_t.append((j_dp, dp_kernels, dp_gemm.flops))
    # every rank runs the same number of DP iterations (the all-reduce is a
    # rendezvous: an extra iteration on one rank would wait for its peers)
    dp_submitted = [0]
    dom.set_lend(tt[0][0] if tt else t_dp)
    eng.start()
    T = 4
    step_hint = 2_000_000
    live_d = {j: None for j, _, _ in jobs_d}
    live_t = {j: [] for j, _, _ in jobs_t}
    done_reqs, train_done = [], []
    t_end = time.time() + args.c5_seconds
    req_id = 0
    last_log = time.time()
    while time.time() < t_end:
        if time.time() - last_log > 1.0:
            last_log = time.time()
            log(f"config 5 rank {rank}: {len(done_reqs)} requests, {len(train_done)} train iters, dp "
                f"{dp_submitted[0]}", eng.counters())
        for j, ks, m in jobs_d:
            cur = live_d[j]
            if cur is None or eng.record(cur[-1]).state == 2:
                if cur is not None:
                    done_reqs.append((j, cur))
                live_d[j] = [eng.submit(j, ks, "decode/step", _abi.DECODE, grid_size=len(ks), request=req_id,
                                        decode_index=k, tpot_ns=50_000_000, ttft_ns=200_000_000,
                                        base_hint_ns=step_hint, saturation=Fraction(1, 2)) for k in range(T)]
                req_id += 1
        for j, ks, fl in jobs_t:
            out = [r for r in live_t[j] if eng.record(r).state != 2]
            train_done += [(r, fl) for r in live_t[j] if r not in out]
            while len(out) < 2 and (j != j_dp or dp_submitted[0] < args.c5_dp_iters):
                dp_submitted[0] += j == j_dp
                out.append(eng.submit(j, ks, "train/iter", _abi.TRAINING, grid_size=len(ks), base_hint_ns=step_hint,
                                      saturation=Fraction(1, 4)))
            live_t[j] = out
        time.sleep(0.0005)
    # drain: decode requests in flight, then the rest of the DP program (other
    # trainers stop submitting, so every tenant gets SMs), then the trainers;
    # bounded so a starved tenant cannot hang the bench
    deadline = time.time() + args.c5_drain_s
    log(f"config 5 rank {rank}: window over, draining (dp {dp_submitted[0]}/{args.c5_dp_iters})")

    def settle(r):
        while eng.record(r).state != 2:
            if time.time() > deadline:
                return False
            time.sleep(0.0005)
        return True

    incomplete = 0
    for j, cur in live_d.items():
        if cur is not None:
            if settle(cur[-1]):
                done_reqs.append((j, cur))
            else:
                incomplete += 1
    while dp_submitted[0] < args.c5_dp_iters and time.time() < deadline:
        out = [r for r in live_t[j_dp] if eng.record(r).state != 2]
        train_done += [(r, dp_gemm.flops) for r in live_t[j_dp] if r not in out]
        if len(out) < 2:
            out.append(eng.submit(j_dp, dp_kernels, "train/iter", _abi.TRAINING, grid_size=2, base_hint_ns=step_hint,
                                  saturation=Fraction(1, 4)))
            dp_submitted[0] += 1
        live_t[j_dp] = out
        time.sleep(0.0005)
    for j, rs in live_t.items():
        fl = next(f for jj, _, f in jobs_t if jj == j)
        for r in rs:
            if settle(r):
                train_done.append((r, fl))
            else:
                incomplete += 1
    if incomplete:
        log(f"config 5 rank {rank}: {incomplete} records incomplete at the drain deadline", eng.counters())
    tpots, tokens, t0, t1 = [], 0, None, None
    for j, recs in done_reqs:
        inf = [eng.record(r) for r in recs]
        tpots.append((inf[-1].t_end - inf[0].t_end) / (T - 1) / 1e6)
        tokens += T * 32  # batch 32 sequences per step
        t0 = inf[0].t_first_claim if t0 is None else min(t0, inf[0].t_first_claim)
        t1 = inf[-1].t_end if t1 is None else max(t1, inf[-1].t_end)
    flop = sum(fl for _, fl in train_done)
    for r, _ in train_done:
        i = eng.record(r)
        t0 = i.t_first_claim if t0 is None else min(t0, i.t_first_claim)
        t1 = i.t_end if t1 is None else max(t1, i.t_end)
    counters = eng.counters()
    if incomplete:
        dpg.abort()  # a starved DP iteration must not keep peers' blocks waiting
    eng.stop()
    eng.close()
    dom.stop()
    dom.close()
    win = (t1 - t0) * 1e-9 if t0 is not None else 1.0
    counters["incomplete_records"] = incomplete
    return {"rank": rank, "tenants": [s.name for s in mine] + ["dp_train"], "tpot_ms": tpots,
            "decode_tokens_per_s": tokens / win, "train_tflops": flop / win / 1e12, "window_s": win,
            "train_iters": len(train_done), "requests": len(done_reqs), "dp_iters": dp_submitted[0],
            "engine_counters": counters}


def aggregate_config5(parts):
    tp = [x for p in parts for x in p["tpot_ms"]]
    return {"workload": "config 5: 16 synthetic tenants (8 Llama-3-8B-shaped decode, 2-8 layers, batch 32, KV "
                        "1024; 8 bf16 GEMM trainers 2048^3-8192^3) placed over the GPUs by ds_place_tenants, plus "
                        "one data-parallel GEMM 4096^3 tenant with the peer-memory gradient all-reduce body; "
                        "TPOT-First per GPU",
            "n_gpus": len(parts), "placement": {p["rank"]: p["tenants"] for p in parts},
            "decode_tokens_per_s": round(sum(p["decode_tokens_per_s"] for p in parts), 1),
            "train_tflops": round(sum(p["train_tflops"] for p in parts), 1),
            "p99_tpot_ms": round(nearest_rank(tp, 99), 3) if tp else None,
            "requests": sum(p["requests"] for p in parts), "train_iters": sum(p["train_iters"] for p in parts),
            "dp_iters_submitted": [p["dp_iters"] for p in parts],
            "incomplete_records": sum(p["engine_counters"].get("incomplete_records", 0) for p in parts)}


def aggregate_ranks(vals):
    """Whole-job line from per-rank lines (independent domains, weak scaling):
    latency metrics take the worst rank, throughputs sum, timing is the max
    over ranks."""
    out = dict(vals[0])
    out["value"] = max(v["value"] for v in vals)
    out["train_tflops"] = round(sum(v["train_tflops"] for v in vals), 1)
    out["e2e"] = dict(vals[0]["e2e"])
    out["e2e"]["value"] = max(v["e2e"]["value"] for v in vals)
    out["ms_per_step"] = max(v["ms_per_step"] for v in vals)
    out["timeslice"] = {"p99_tpot_ms": max(v["timeslice"]["p99_tpot_ms"] for v in vals),
                        "train_tflops": round(sum(v["timeslice"]["train_tflops"] for v in vals), 1)}
    out["bit_exact_vs_solo"] = all(v["bit_exact_vs_solo"] for v in vals)
    out["gpu_launches"] = sum(v["gpu_launches"] for v in vals)
    out["n_gpus"] = len(vals)
    # every rank's own numbers (each GPU ran its own domain: evidence that all
    # of them were busy, and the spread behind the worst-rank value)
    out["per_rank"] = [{"rank": i, "value": v["value"], "train_tflops": v["train_tflops"],
                        "gpu_launches": v["gpu_launches"], "ms_per_step": v["ms_per_step"],
                        "bit_exact_vs_solo": v["bit_exact_vs_solo"]} for i, v in enumerate(vals)]
    return out


def gather_ranks(out, world):
    import torch.distributed as dist
    vals = [None] * world
    dist.all_gather_object(vals, out)
    return aggregate_ranks(vals)


def reference_arm(args, world):
    """bench.py --impl reference: the reference's own CPU implementation of
    the path — the corosim simulator (oracle/_ref, built from the reference
    sources) — timed on this host on the config-2 scenario.  A step simulates
    `rps` decode requests of `tokens` tokens beside the training GEMM stream;
    its per-token value is the wall time the CPU path spends per decode token.
    value = nearest-rank P99 over the timed steps.  The engine is
    single-threaded by construction (engine.hpp:149-151) and TPOT is a
    latency, so extra host threads would not lower it: 1 core."""
    solo, calib = {"decode_step_ms": 3.0, "gemm_ms": 0.78}, "nominal B200 floors: 3.0 ms/decode step, 0.78 ms/GEMM"
    for name in ("r2_bench_latest.json", "r1_bench_latest.json"):
        try:
            rec = json.load(open(os.path.join(ROOT, "profiles", name)))["solo"]
            solo = {"decode_step_ms": float(rec["decode_step_ms"]), "gemm_ms": float(rec["gemm_ms"])}
            calib = (f"solo durations measured on B200 (profiles/{name}): "
                     f"{solo['decode_step_ms']} ms/decode step, {solo['gemm_ms']} ms/GEMM")
            break
        except Exception:
            continue
    try:
        per_tok, p99s, evs = [], [], 0
        for i in range(args.warmup + args.steps):
            p99, wall, ev = reference_sim(solo, args.rps, args.tokens)
            if i >= args.warmup:
                per_tok.append(wall * 1e3 / (args.rps * args.tokens))
                p99s.append(p99)
                evs = ev
        v = nearest_rank(per_tok, 99)
        return {"impl": "reference", "metric": METRIC, "value": round(v, 5), "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": round(statistics.median(per_tok) * args.rps * args.tokens, 4),
                "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "rational (exact)",
                "data": "synthetic",
                "config": {"workload": "config 2 scenario (decode requests + training GEMM stream, tpot-first) in the "
                                       "reference simulator (corosim SimEngine::simulate, oracle/_ref)",
                           "step": f"{args.rps} decode requests x {args.tokens} tokens", "calibration": calib,
                           "tpot": "CPU wall ms the reference path spends per decode token (it models the decode "
                                   "step, it does not compute it)"},
                "sim_predicted_p99_tpot_ms": p99s[-1],
                "cpu_baseline": {"value": round(v, 5), "unit": UNIT, "cores": 1, "kind": "reference",
                                 "sample": f"{args.rps} requests x {args.tokens} tokens per step, {evs} events"},
                "e2e": {"value": round(v, 5), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    except Exception as e:  # reference library missing on this host
        return {"impl": "reference", "unavailable": f"reference simulator not built: {e}"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--tokens", type=int, default=8)
    ap.add_argument("--rps", type=int, default=10, help="decode requests per bench step (P99 over steps x rps)")
    ap.add_argument("--kv-len", type=int, default=1024)
    ap.add_argument("--quantum-ms", type=float, default=5.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--decode-sat", default="1/2", help="decode compute saturation (tier wanted)")
    ap.add_argument("--slo-x", type=float, default=8.0, help="TPOT SLO as a multiple of the solo step")
    ap.add_argument("--no-config13", action="store_true", help="skip the config 1 / config 3 legs")
    ap.add_argument("--no-config5", action="store_true", help="skip the config 5 (16-tenant placement) leg")
    ap.add_argument("--c5-seconds", type=float, default=3.0, help="config 5 run window per rank")
    ap.add_argument("--c5-dp-iters", type=int, default=40, help="config 5 data-parallel tenant iterations")
    ap.add_argument("--c5-drain-s", type=float, default=30.0, help="config 5 drain deadline")
    ap.add_argument("--only-config5", action="store_true", help="run the config 5 leg alone (debug)")
    ap.add_argument("--no-config4b", action="store_true", help="skip the two-stream prefill mix leg")
    ap.add_argument("--only-config4b", action="store_true", help="run the two-stream prefill mix leg alone (debug)")
    ap.add_argument("--no-config4", action="store_true", help="skip the config 4 (ResNet + bursty decode) leg")
    ap.add_argument("--burst-units", type=float, default=60.0, help="config 4 trace duration (units of 50 ms)")
    ap.add_argument("--tiers", default="1/4,1/2,3/4,1", help="pctx pool tiers (create_pool; SPEC.md:65 pool)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if world > 1:
        import datetime
        import torch.distributed as dist
        # host-side plumbing only (line aggregation, DP handle exchange); a
        # bounded timeout so a failed rank cannot hang the others forever
        dist.init_process_group("gloo", timeout=datetime.timedelta(minutes=10))
    if args.impl == "reference":
        if rank != 0:
            return
        print(json.dumps(reference_arm(args, world)))
        return
    if args.only_config5:
        out, tail, solo = {}, {}, None
    else:
        out, tail, solo = gpu_arm(args, rank, world)
        # the latest solo calibration (the reference arm reads it)
        if rank == 0:
            try:
                json.dump({"solo": out["solo"], "roofline": out["roofline"]},
                          open(os.path.join(ROOT, "profiles", "r2_bench_latest.json"), "w"), indent=1)
            except Exception:
                pass
    if world > 1 and not args.only_config5:
        out = gather_ranks(dict(out, **tail), world)
        tail = {k: out.pop(k) for k in ("host_gap_us", "train_tflops", "timeslice")}
    if not args.no_config13 and not args.only_config5:
        import torch
        torch.cuda.empty_cache()
        dev = int(os.environ.get("LOCAL_RANK", rank))
        log("config 1 and 3 legs")
        try:
            c1 = config1_leg(dev)
        except Exception as e:  # an auxiliary leg must not cost the headline line
            c1 = {"error": repr(e)}
        try:
            c3 = config3_leg(dev)
        except Exception as e:
            c3 = {"error": repr(e)}
        if rank == 0:
            out["config1"], out["config3"] = c1, c3
    if not args.no_config5:
        import torch
        torch.cuda.empty_cache()
        dev = int(os.environ.get("LOCAL_RANK", rank))

        def gather(obj):
            if world == 1:
                return [obj]
            import torch.distributed as dist
            res = [None] * world
            dist.all_gather_object(res, obj)
            return res

        log("config 5 leg")
        try:
            part = config5_leg(args, rank, world, dev, gather)
        except Exception as e:
            part = {"rank": rank, "error": repr(e)}
        parts = gather(part)
        errors = [p["error"] for p in parts if "error" in p]
        c5 = {"error": errors} if errors else aggregate_config5(parts)
        if rank == 0:
            out["config5"] = c5
    if rank == 0:
        if not args.no_cpu_baseline and solo is not None:
            try:
                out["cpu_baseline"] = cpu_baseline_leg(solo, args.rps, args.tokens)
            except Exception as e:
                out["cpu_baseline"] = {"value": None, "unavailable": str(e)}
            # the reference simulator on every other config's scenario
            try:
                c1 = out.get("config1") or {}
                c4 = out.get("config4") or {}
                refs = cpu_reference_configs(
                    c1_solo_us=1000 * float(c1.get("solo_ms", 0.1)),
                    step_us=max(1, int(1000 * solo["decode_step_ms"])), gemm_us=max(1, int(1000 * solo["gemm_ms"])),
                    resnet_iter_us=max(1, int(1000 * float(c4.get("resnet_solo_iter_ms", 10.0)))))
                for k, v in refs.items():
                    if isinstance(out.get(k), dict):
                        out[k]["cpu_reference"] = v
                    else:
                        out.setdefault("cpu_reference", {})[k] = v
            except Exception as e:
                out["cpu_reference_error"] = repr(e)
        # the time-slicing comparator and training throughput last, so a
        # truncated tail of the line still carries them
        out.update(tail)
        print(json.dumps(out))


if __name__ == "__main__":
    main()
