"""Python view of one GPU sharing domain over the C ABI (tests, bench, smoke).

Names follow the reference: a *tenant* is the reference's JobSpec/vctx, a
*kernel* is the immutable Kernel launch record, a *pctx* is a quota-tier
physical context, and bind/unbind/migrate/preempt are the binding-table and
rck_flag operations (include/corosim/core/types.hpp:19-137,
src/engine/engine.cpp:620-806).
"""
from __future__ import annotations

import atexit
import ctypes
import weakref
from fractions import Fraction
from typing import Iterable, List, Optional, Sequence, Tuple

from . import _abi
from ._abi import check, check_engine, lib


_LIVE: "weakref.WeakSet[Domain]" = weakref.WeakSet()


@atexit.register
def _stop_live_domains():
    for d in list(_LIVE):
        try:
            d.stop()
            d.close()
        except Exception:
            pass


class Domain:
    def __init__(self, device: int = 0, tiers: Sequence[Fraction] = (Fraction(1),), ring_capacity: int = 1024,
                 block_log_capacity: int = 1 << 20, lend_idle_sms: bool = True, executor_smem: int = 0):
        cfg = _abi.DomainConfig()
        cfg.device = device
        cfg.n_tiers = len(tiers)
        for i, t in enumerate(tiers):
            t = Fraction(t)
            cfg.tier_num[i] = t.numerator
            cfg.tier_den[i] = t.denominator
        cfg.ring_capacity = ring_capacity
        cfg.block_log_capacity = block_log_capacity
        cfg.lend_idle_sms = int(lend_idle_sms)
        cfg.executor_smem = executor_smem
        h = ctypes.c_void_p()
        check(lib().ds_domain_create(ctypes.byref(cfg), ctypes.byref(h)))
        self.h = h
        self.device = device
        self.tiers = [Fraction(t) for t in tiers]
        n = ctypes.c_int()
        check(lib().ds_num_sms(self.h, ctypes.byref(n)))
        self.num_sms = n.value
        self._args_keep = []
        # a script that dies with the persistent executor still resident would
        # hang process teardown (the CUDA context waits for the kernel): stop
        # it at interpreter exit
        _LIVE.add(self)

    # -- lifecycle --
    def close(self):
        if self.h:
            lib().ds_domain_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        try:
            self.stop()
        finally:
            self.close()

    def start(self):
        check(lib().ds_start(self.h))

    def stop(self):
        if self.h:
            check(lib().ds_stop(self.h))

    # -- registration --
    def tenant(self, name: str, priority: int = _abi.BEST_EFFORT) -> int:
        d = _abi.TenantDesc(name.encode(), priority)
        out = ctypes.c_int()
        check(lib().ds_tenant_register(self.h, ctypes.byref(d), ctypes.byref(out)))
        return out.value

    def kernel(self, semantic_id: str, body: int, grid: Tuple[int, int, int], args: ctypes.Structure,
               phase: int = _abi.OTHER, request: int = -1, decode_index: int = -1, block_threads: int = 256) -> int:
        desc = make_desc(semantic_id, body, grid, args, phase, request, decode_index, block_threads)
        self._args_keep.append(args)
        out = ctypes.c_int()
        check(lib().ds_kernel_register(self.h, ctypes.byref(desc), ctypes.byref(out)))
        return out.value

    # -- launches --
    def launch(self, tenant: int, kernel: int, tag: int = 0) -> int:
        seq = ctypes.c_uint64()
        check(lib().ds_launch(self.h, tenant, kernel, tag, ctypes.byref(seq)))
        return seq.value

    def launch_atomized(self, tenant: int, kernel: int, tier: Fraction, tag: int = 0) -> int:
        tier = Fraction(tier)
        seq = ctypes.c_uint64()
        check(lib().ds_launch_atomized(self.h, tenant, kernel, tag, tier.numerator, tier.denominator,
                                       ctypes.byref(seq)))
        return seq.value

    def wait(self, tenant: int, seq: int, timeout_ms: int = 60000):
        check(lib().ds_wait_tenant(self.h, tenant, seq, timeout_ms))

    # -- local exceptions (apply_local_exception, engine.cpp:1049-1083) --
    def fault_inject(self, tenant: int, code: int = _abi.FAULT_INJECTED):
        check(lib().ds_fault_inject(self.h, tenant, code))

    def tenant_fault(self, tenant: int) -> Optional[dict]:
        """None while healthy, else the first fault: {code, block, seq,
        first_failed, t} (launches >= first_failed never complete intact)."""
        f = _abi.FaultInfo()
        check(lib().ds_tenant_fault(self.h, tenant, ctypes.byref(f)))
        if not f.code:
            return None
        return {"code": f.code, "block": f.block, "seq": f.seq, "first_failed": f.first_failed, "t": f.t_ns}

    def poll(self, cap: int = 4096) -> List[_abi.Completion]:
        arr = (_abi.Completion * cap)()
        n = ctypes.c_int()
        check(lib().ds_poll(self.h, arr, cap, ctypes.byref(n)))
        return [arr[i] for i in range(n.value)]

    # -- arbiter --
    def bind(self, tenant: int, pctx: int):
        check(lib().ds_bind(self.h, tenant, pctx))

    def unbind(self, tenant: int):
        check(lib().ds_unbind(self.h, tenant))

    def migrate(self, tenant: int, pctx: int):
        check(lib().ds_migrate(self.h, tenant, pctx))

    def preempt(self, pctx: int):
        check(lib().ds_preempt(self.h, pctx))

    def bound_pctx(self, tenant: int) -> int:
        out = ctypes.c_int()
        check(lib().ds_bound_pctx(self.h, tenant, ctypes.byref(out)))
        return out.value

    def _arr(self, xs: Optional[Iterable[int]]):
        if xs is None:
            return None
        xs = list(xs)
        assert len(xs) == self.num_sms
        return (ctypes.c_int32 * self.num_sms)(*xs)

    def quota_set(self, owner: Sequence[int], lender: Optional[Sequence[int]] = None):
        check(lib().ds_quota_set(self.h, self._arr(owner), self._arr(lender), self.num_sms))

    def quota_at_claim(self, tenant: int, seq: int, block: int, owner: Sequence[int],
                       lender: Optional[Sequence[int]] = None):
        check(lib().ds_quota_at_claim(self.h, tenant, seq, block, self._arr(owner), self._arr(lender),
                                      self.num_sms))

    def set_abandonable(self, tenant: int, enable: bool = True):
        """Blocks of abandonable bodies (GEMM with abandon=True) yield within
        a k-block when revoked and re-run from scratch (before start())."""
        check(lib().ds_tenant_abandonable(self.h, tenant, int(enable)))

    def ledger(self) -> dict:
        """OverheadLedger measured on the device since ds_start (ns)."""
        l = _abi.Ledger()
        check(lib().ds_ledger_get(self.h, ctypes.byref(l)))
        return ledger_dict(l)

    def kernel_info(self, kernel: int) -> _abi.KernelInfo:
        out = _abi.KernelInfo()
        check(lib().ds_kernel_info_get(self.h, kernel, ctypes.byref(out)))
        return out

    def verify_kernels(self) -> int:
        """-1 if every kernel record is intact, else the first mutated kernel id."""
        bad = ctypes.c_int(-1)
        rc = lib().ds_verify_kernels(self.h, ctypes.byref(bad))
        if rc not in (0, _abi.RECORD_MUTATED):
            check(rc)
        return bad.value

    def set_drain_exit(self, enable: bool = True, deadline_ms: int = 0):
        """Before start(): the executor exits by itself once every launch
        enqueued so far (launches may be issued before start) completed, or
        after deadline_ms.  For profilers that serialise kernel launches."""
        check(lib().ds_set_drain_exit(self.h, int(enable), deadline_ms))

    def set_lane_split(self, mode: int):
        """0 off; 1: owned SMs run the lend tenant on lane 1 (lane 0: owner,
        then lend tenant); 2: lane 0 runs the owner only."""
        check(lib().ds_set_lane_split(self.h, mode))

    def quota_triggers_reset(self):
        check(lib().ds_quota_triggers_reset(self.h))

    def quota_periodic(self, period_ns: int, owner_a, owner_b, lender_a=None, lender_b=None):
        check(lib().ds_quota_periodic(self.h, period_ns, self._arr(owner_a), self._arr(lender_a),
                                      self._arr(owner_b), self._arr(lender_b), self.num_sms))

    def set_lend(self, tenant: int):
        check(lib().ds_set_lend(self.h, tenant))

    def mask(self, tenant: int, first: int, count: int, default: int = -1) -> List[int]:
        """Owner vector giving SM slots [first, first+count) to tenant."""
        return [tenant if first <= i < first + count else default for i in range(self.num_sms)]

    # -- observation --
    def stats(self) -> _abi.Stats:
        s = _abi.Stats()
        check(lib().ds_stats_get(self.h, ctypes.byref(s)))
        return s

    def transcript(self, tenant: int) -> List[Tuple[int, int]]:
        n = ctypes.c_int()
        check(lib().ds_transcript(self.h, tenant, None, None, 0, ctypes.byref(n)))
        k = (ctypes.c_int32 * max(1, n.value))()
        g = (ctypes.c_uint32 * max(1, n.value))()
        check(lib().ds_transcript(self.h, tenant, k, g, n.value, ctypes.byref(n)))
        return [(k[i], g[i]) for i in range(n.value)]

    def logical_progress(self, tenant: int) -> int:
        out = ctypes.c_int64()
        check(lib().ds_logical_progress(self.h, tenant, ctypes.byref(out)))
        return out.value

    def _log(self, fn, rec):
        n = ctypes.c_int64()
        check(fn(self.h, None, 0, ctypes.byref(n)))
        arr = (rec * max(1, n.value))()
        check(fn(self.h, arr, n.value, ctypes.byref(n)))
        return [arr[i] for i in range(n.value)]

    def block_log(self):
        return self._log(lib().ds_block_log, _abi.BlockRecord)

    def switch_log(self):
        return self._log(lib().ds_switch_log, _abi.SwitchRecord)

    def ctl_log(self):
        return self._log(lib().ds_ctl_log, _abi.CtlRecord)

    def clear_logs(self):
        check(lib().ds_clear_logs(self.h))

    def globaltimer(self) -> int:
        out = ctypes.c_uint64()
        check(lib().ds_globaltimer(self.h, ctypes.byref(out)))
        return out.value

    def ctl_roundtrip(self, n: int = 100) -> List[int]:
        arr = (ctypes.c_uint64 * n)()
        check(lib().ds_ctl_roundtrip(self.h, n, arr))
        return list(arr)

    def debug(self) -> str:
        buf = ctypes.create_string_buffer(1 << 16)
        check(lib().ds_debug_dump(self.h, buf, len(buf)))
        return buf.value.decode()

    def smids(self) -> List[int]:
        arr = (ctypes.c_int * self.num_sms)()
        n = ctypes.c_int()
        check(lib().ds_smids(self.h, arr, self.num_sms, ctypes.byref(n)))
        return list(arr)

    def solo(self, kernel: int, stream: int = 0):
        check(lib().ds_solo_launch_registered(self.h, kernel, ctypes.c_void_p(stream)))


def make_desc(semantic_id, body, grid, args, phase=_abi.OTHER, request=-1, decode_index=-1, block_threads=256):
    gx, gy, gz = (tuple(grid) + (1, 1, 1))[:3]
    return _abi.KernelDesc(semantic_id.encode(), body, gx, gy, gz, block_threads,
                           ctypes.cast(ctypes.pointer(args), ctypes.c_void_p), ctypes.sizeof(args), phase,
                           request, decode_index)


def solo_launch(device: int, semantic_id: str, body: int, grid, args, stream: int = 0):
    """Run a body standalone as a plain grid (exclusive_baseline)."""
    desc = make_desc(semantic_id, body, grid, args)
    check(lib().ds_solo_launch(device, ctypes.byref(desc), ctypes.c_void_p(stream)))


_LIVE_ENGINES: "weakref.WeakSet[Engine]" = weakref.WeakSet()


@atexit.register  # registered after the domain hook, so it runs first (LIFO)
def _stop_live_engines():
    for e in list(_LIVE_ENGINES):
        try:
            e.stop()
            e.close()
        except Exception:
            pass


class UserPolicy:
    """A Python policy handed to the engine through the C-ABI vtable
    (ds_engine_create_with_policy; the reference's Policy virtuals,
    policy.hpp:97-126).  Hooks get a ``PolicyView``-shaped snapshot and a
    launch context and return ``(kind, target)`` with kind one of
    _abi.DISPATCH_DIRECT / DISPATCH_REMAP / DISPATCH_DEFER / PREEMPT /
    NO_ACTION.  The engine validates every decision (apply_decision,
    engine.cpp:688-754): an illegal one becomes Defer + policy_errors."""

    name = "user"

    def on_launch(self, view, launch):
        return (_abi.DISPATCH_DEFER, -1)

    def on_completion(self, view, launch):
        return (_abi.NO_ACTION, -1)

    def on_congestion(self, view, launch):
        return (_abi.DISPATCH_DEFER, -1)

    def launch_order_key(self, launch) -> int:
        return 0

    def next_review_time(self, view):
        return None


class _NS:
    def __init__(self, **kw):
        self.__dict__.update(kw)

    def __repr__(self):
        return f"{type(self).__name__}({self.__dict__})"


def view_from_c(v: _abi.View) -> _NS:
    """ds_view -> a PolicyView-shaped object (tiers as Fractions, times in ns)."""
    pctxs = []
    for i in range(v.n_pctx):
        p = v.pctx[i]
        pctxs.append(_NS(id=p.id, device=p.device, tier=Fraction(p.tier_num, p.tier_den), standby=bool(p.standby),
                         available=bool(p.available), bound=None if p.bound < 0 else p.bound,
                         running_kernel=p.running_kernel if p.has_running else None,
                         running_semantic_id=(p.running_semantic_id or b"").decode(), running_grid=p.running_grid,
                         running_remaining=p.running_remaining_ns, running_phase=p.running_phase,
                         running_priority=p.running_priority))
    vctxs = [_NS(id=x.id, priority=x.priority, quarantined=bool(x.quarantined), bound=bool(x.bound), pending=x.pending,
                 head_phase=x.head_phase, decoding=bool(x.decoding)) for x in (v.vctx[i] for i in range(v.n_vctx))]
    return _NS(now=v.now_ns, pctxs=pctxs, vctxs=vctxs,
               bound_tier_sums={d: Fraction(v.bound_tier_sum_num[d], v.bound_tier_sum_den[d])
                                for d in range(v.n_devices)},
               min_tiers={d: Fraction(v.min_tier_num[d], v.min_tier_den[d]) for d in range(v.n_devices)},
               active_vctx_count=v.active_vctx_count, predictor=v.predictor)


def launch_from_c(c: _abi.LaunchCtx) -> _NS:
    return _NS(vctx=c.vctx, has_kernel=bool(c.has_kernel), kernel_id=c.kernel_id,
               semantic_id=(c.semantic_id or b"").decode(), grid_size=c.grid_size, base_hint_ns=c.base_hint_ns,
               saturation=Fraction(c.sat_num, c.sat_den) if c.sat_den else Fraction(1), phase=c.phase,
               decode_index=c.decode_index, request=c.request, arrival_ns=c.arrival_ns,
               request_arrival_ns=c.request_arrival_ns,
               slo=(c.ttft_ns, c.tpot_ns) if c.has_slo else None, pool_exhausted=bool(c.pool_exhausted))


def predict(predictor, semantic_id: str, grid: int, hint_ns: Optional[int] = None) -> int:
    """DurationPredictor::predict of a view's predictor (valid inside a hook)."""
    out = ctypes.c_int64()
    check(lib().ds_predictor_predict(predictor, semantic_id.encode(), grid, 0 if hint_ns is None else 1,
                                     hint_ns or 0, ctypes.byref(out)))
    return out.value


def _vtable_for(policy: UserPolicy):
    """ctypes vtable whose hooks call the Python policy (kept alive by the engine object)."""
    def wrap(fn):
        def hook(user, view, launch, out):
            try:
                k, t = fn(view_from_c(view.contents), launch_from_c(launch.contents))
                out[0] = _abi.Decision(int(k), int(t))
            except Exception:  # no exceptions across the ABI: an illegal decision
                out[0] = _abi.Decision(-1, -1)
        return _abi.HOOK(hook)

    def order(user, launch):
        try:
            return int(policy.launch_order_key(launch_from_c(launch.contents)))
        except Exception:
            return 0

    def review(user, view, t):
        try:
            r = policy.next_review_time(view_from_c(view.contents))
        except Exception:
            r = None
        if r is None:
            return 0
        t[0] = int(r)
        return 1

    vt = _abi.PolicyVtable()
    keep = [wrap(policy.on_launch), wrap(policy.on_completion), wrap(policy.on_congestion),
            _abi.ORDER_KEY(order), _abi.REVIEW(review), _abi.DESTROY(0)]
    name = str(getattr(policy, "name", "user")).encode()
    vt.name = name
    vt.on_launch, vt.on_completion, vt.on_congestion, vt.launch_order_key, vt.next_review_time, vt.destroy = keep
    return vt, keep + [name]


def builtin_decide(policy: str, hook: int, view: _abi.View, launch: _abi.LaunchCtx, quantum_ns: int = 0):
    """A built-in policy's hook over a C view (ds_builtin_decide): (kind, target)."""
    d = _abi.Decision()
    check(lib().ds_builtin_decide(policy.encode(), hook, ctypes.byref(view), ctypes.byref(launch), quantum_ns,
                                  ctypes.byref(d)))
    return d.kind, d.target


def seeded_values(seed: int, n: int, fmt: int) -> List[int]:
    """seeded_values (equivalence.cpp:7-17): raw bit patterns (fmt 0 fp16, 1 bf16, 2 fp32)."""
    out = (ctypes.c_uint32 * max(1, n))()
    check(lib().ds_seeded_values(seed, n, fmt, out))
    return list(out[:n])


def round_to(fmt: int, x: float) -> int:
    out = ctypes.c_uint32()
    check(lib().ds_round_to(fmt, x, ctypes.byref(out)))
    return out.value


def add_normalization(shared, solo):
    """add_normalization (metrics.cpp:81-102) over [(first_arrival_ns, last_finish_ns) or None] per job:
    ([Fraction per job], aggregate float)."""
    n = len(shared)
    a = (_abi.JobSpan * max(1, n))()
    b = (_abi.JobSpan * max(1, n))()
    for i in range(n):
        for arr, x in ((a, shared[i]), (b, solo[i])):
            if x is not None:
                arr[i] = _abi.JobSpan(int(x[0]), int(x[1]), 1, 0)
    num = (ctypes.c_int64 * max(1, n))()
    den = (ctypes.c_int64 * max(1, n))()
    agg = ctypes.c_double()
    check(lib().ds_add_normalization(a, b, n, num, den, ctypes.byref(agg)))
    return [Fraction(num[i], den[i]) for i in range(n)], agg.value


def ledger_dict(l: _abi.Ledger) -> dict:
    return {n: getattr(l, n) for n, _ in _abi.Ledger._fields_}


class Engine:
    """SimEngine-like dispatch loop over one domain (C++ engine thread).

    Jobs map 1:1 to tenants; ``submit`` is the reference's kernel arrival of a
    launch record that runs as the listed registered kernels.  ``policy`` is a
    built-in name or a UserPolicy object (SimEngine(Scenario,
    std::unique_ptr<Policy>), engine.hpp:155)."""

    def __init__(self, dom: Domain, policy="tpot-first", quantum_ns: int = 5_000_000, alpha: float = 0.3,
                 cold_start_ns: int = 1_000_000_000, release_on_idle: bool = True, fair_handover: bool = True,
                 lend_tenant: int = -1, assignments=None, hang_detection: bool = False, hang_threshold: float = 3.0,
                 capture_log: bool = False, reset_delay_ns: int = 0):
        cfg = _abi.EngineConfig()
        cfg.reset_delay_ns = reset_delay_ns
        cfg.hang_detection = int(hang_detection)
        cfg.hang_threshold = hang_threshold
        cfg.capture_log = int(capture_log)
        user = None if isinstance(policy, str) else policy
        cfg.policy = policy.encode() if user is None else b""
        cfg.quantum_ns = quantum_ns
        cfg.alpha = alpha
        cfg.cold_start_ns = cold_start_ns
        cfg.release_on_idle = int(release_on_idle)
        cfg.fair_handover = int(fair_handover)
        cfg.lend_tenant = lend_tenant
        assignments = assignments or {}
        cfg.n_assignments = len(assignments)
        for i, (v, p) in enumerate(assignments.items()):
            cfg.assign_vctx[i] = v
            cfg.assign_pctx[i] = p
        h = ctypes.c_void_p()
        self._keep = []
        if user is None:
            check_engine(lib().ds_engine_create(dom.h, ctypes.byref(cfg), ctypes.byref(h)))
        else:
            vt, keep = _vtable_for(user)
            self._keep += keep + [vt, user]
            check_engine(lib().ds_engine_create_with_policy(dom.h, ctypes.byref(cfg), ctypes.byref(vt), None,
                                                            ctypes.byref(h)))
        self.h = h
        self.dom = dom
        _LIVE_ENGINES.add(self)

    def add_job(self, tenant: int, priority: int) -> int:
        out = ctypes.c_int()
        check_engine(lib().ds_engine_add_job(self.h, tenant, priority, ctypes.byref(out)))
        return out.value

    def submit(self, job: int, kernels: Sequence[int], semantic_id: str, phase: int = _abi.OTHER, grid_size: int = 1,
               request: int = -1, decode_index: int = -1, arrival_ns: int = 0, request_arrival_ns: int = 0,
               ttft_ns: int = 0, tpot_ns: int = 0, base_hint_ns: int = 0, saturation: Fraction = Fraction(1)) -> int:
        arr = (ctypes.c_int32 * len(kernels))(*kernels)
        sat = Fraction(saturation)
        d = _abi.RecordDesc(semantic_id.encode(), grid_size, arr, len(kernels), phase, request, decode_index,
                            arrival_ns, request_arrival_ns, ttft_ns, tpot_ns, base_hint_ns, sat.numerator,
                            sat.denominator)
        out = ctypes.c_uint64()
        check_engine(lib().ds_engine_submit(self.h, job, ctypes.byref(d), ctypes.byref(out)))
        return out.value

    def start(self):
        check_engine(lib().ds_engine_start(self.h))

    def stop(self):
        if self.h:
            check_engine(lib().ds_engine_stop(self.h))

    def close(self):
        if self.h:
            lib().ds_engine_destroy(self.h)
            self.h = None

    def now(self) -> int:
        out = ctypes.c_int64()
        check_engine(lib().ds_engine_now(self.h, ctypes.byref(out)))
        return out.value

    def wait(self, rec: int, timeout_ms: int = 120000):
        check_engine(lib().ds_engine_wait(self.h, rec, timeout_ms))

    def record(self, rec: int) -> _abi.RecordInfo:
        out = _abi.RecordInfo()
        check_engine(lib().ds_engine_record(self.h, rec, ctypes.byref(out)))
        return out

    def snapshot(self):
        """ds_snapshot: the PolicyView a hook would see now."""
        v = _abi.View()
        check_engine(lib().ds_engine_snapshot(self.h, ctypes.byref(v)))
        return view_from_c(v)

    def ledger(self) -> dict:
        """OverheadLedger of this engine's run (device-measured, ns)."""
        l = _abi.Ledger()
        check_engine(lib().ds_engine_ledger(self.h, ctypes.byref(l)))
        return ledger_dict(l)

    def job_fingerprint(self, job: int) -> int:
        out = ctypes.c_uint64()
        check_engine(lib().ds_engine_job_fingerprint(self.h, job, ctypes.byref(out)))
        return out.value

    def counters(self) -> dict:
        c = _abi.EngineCounters()
        check_engine(lib().ds_engine_counters_get(self.h, ctypes.byref(c)))
        return {n: getattr(c, n) for n, _ in _abi.EngineCounters._fields_}

    def event_log(self) -> List[dict]:
        """The JSONL event log (reference schema, engine.cpp:316-329), parsed."""
        import json
        n = ctypes.c_int64()
        check_engine(lib().ds_engine_event_log(self.h, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value + 1)
        check_engine(lib().ds_engine_event_log(self.h, buf, n.value + 1, ctypes.byref(n)))
        return [json.loads(x) for x in buf.value.decode().splitlines() if x]

    def quarantines(self) -> List[Tuple[int, int]]:
        n = ctypes.c_int()
        check_engine(lib().ds_engine_quarantines(self.h, None, None, 0, ctypes.byref(n)))
        jobs = (ctypes.c_int32 * max(1, n.value))()
        ts = (ctypes.c_int64 * max(1, n.value))()
        check_engine(lib().ds_engine_quarantines(self.h, jobs, ts, n.value, ctypes.byref(n)))
        return [(jobs[i], ts[i]) for i in range(n.value)]

    def fault_local(self, pctx: int):
        """FaultSpec{LocalException, pctx} now (engine.cpp:1049-1083)."""
        check_engine(lib().ds_engine_fault_local(self.h, pctx))

    def job_status(self, job: int) -> int:
        out = ctypes.c_int()
        check_engine(lib().ds_engine_job_status(self.h, job, ctypes.byref(out)))
        return out.value

    def transcript(self, job: int) -> List[int]:
        n = ctypes.c_int()
        check_engine(lib().ds_engine_transcript(self.h, job, None, 0, ctypes.byref(n)))
        arr = (ctypes.c_uint64 * max(1, n.value))()
        check_engine(lib().ds_engine_transcript(self.h, job, arr, n.value, ctypes.byref(n)))
        return list(arr)[:n.value]
