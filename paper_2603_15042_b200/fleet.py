"""Fleet: cross-device moves over per-GPU domains (csrc/fleet.cpp, §8f rows 3-4).

Global exceptions with emergency migration to a standby device
(apply_global_exception / emergency_migrate, reference engine.cpp:1095-1166)
and working-set tracking with eager / lazy copies and demand faults for
planned cross-device migrations (begin_migration / advance_lazy /
service_demand_faults, engine.cpp:563-672).  Thin ctypes layer over the
``ds_fleet_*`` C ABI; the logic is native."""
from __future__ import annotations

import ctypes
from fractions import Fraction
from typing import List, Optional, Sequence, Tuple

from . import _abi
from ._abi import DsError
from .runtime import make_desc

STATUS = {0: "active", 1: "failed", 2: "stranded"}


class Reloc(ctypes.Structure):
    _fields_ = [("args_offset", ctypes.c_uint32), ("region", ctypes.c_int32), ("region_offset", ctypes.c_uint64)]


class PlacePctx(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("pctx", ctypes.c_int32), ("tier_num", ctypes.c_int64),
                ("tier_den", ctypes.c_int64), ("bound", ctypes.c_int32), ("pad", ctypes.c_int32)]


class Progress(ctypes.Structure):
    _fields_ = [("head", ctypes.c_uint64), ("tail", ctypes.c_uint64), ("enqueued", ctypes.c_uint64),
                ("claim_seq", ctypes.c_uint64), ("claim_open", ctypes.c_uint32), ("claim_block", ctypes.c_uint32),
                ("claim_grid", ctypes.c_uint32), ("claim_retired", ctypes.c_uint32), ("drained", ctypes.c_uint32),
                ("failed", ctypes.c_uint32)]


class JobInfo(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("tenant", ctypes.c_int32), ("pctx", ctypes.c_int32),
                ("status", ctypes.c_int32), ("launches", ctypes.c_uint64), ("migrations", ctypes.c_int32),
                ("lazy_pending", ctypes.c_int32)]


class MigrationInfo(ctypes.Structure):
    _fields_ = [("job", ctypes.c_int32), ("src_device", ctypes.c_int32), ("src_pctx", ctypes.c_int32),
                ("dst_device", ctypes.c_int32), ("dst_pctx", ctypes.c_int32), ("emergency", ctypes.c_int32),
                ("demand_faults", ctypes.c_int32), ("pad", ctypes.c_int32), ("eager_bytes", ctypes.c_uint64),
                ("lazy_bytes", ctypes.c_uint64), ("start_ns", ctypes.c_int64), ("end_ns", ctypes.c_int64),
                ("resumed_launch", ctypes.c_uint64), ("resumed_block", ctypes.c_uint32), ("pad2", ctypes.c_uint32)]


class Ledger(ctypes.Structure):
    _fields_ = [("migrations", ctypes.c_uint64), ("emergency_migrations", ctypes.c_uint64),
                ("stranded", ctypes.c_uint64), ("migration_total_ns", ctypes.c_int64),
                ("demand_faults", ctypes.c_uint64), ("demand_fault_total_ns", ctypes.c_int64),
                ("eager_bytes", ctypes.c_uint64), ("lazy_bytes", ctypes.c_uint64)]


_setup = False


def lib():
    global _setup
    L = _abi.lib()
    if not _setup:
        vp, i32p, u64p = ctypes.c_void_p, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_uint64)
        ip = ctypes.POINTER(ctypes.c_int)
        L.ds_fleet_last_error.restype = ctypes.c_char_p
        L.ds_launch_from.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint32, u64p]
        L.ds_tenant_progress.argtypes = [vp, ctypes.c_int, ctypes.POINTER(Progress)]
        L.ds_emergency_target.argtypes = [i32p, i32p, ctypes.c_int, ctypes.POINTER(PlacePctx), ctypes.c_int,
                                          ctypes.c_int64, ctypes.c_int64, ip]
        L.ds_fleet_create.argtypes = [ctypes.POINTER(vp)]
        L.ds_fleet_destroy.argtypes = [vp]
        L.ds_fleet_add_device.argtypes = [vp, vp, ctypes.c_int, ctypes.c_int, ip]
        L.ds_fleet_add_job.argtypes = [vp, ctypes.c_int, ctypes.POINTER(_abi.TenantDesc), ip]
        L.ds_fleet_add_region.argtypes = [vp, ctypes.c_int, vp, ctypes.c_uint64, ip]
        L.ds_fleet_add_kernel.argtypes = [vp, ctypes.c_int, ctypes.POINTER(_abi.KernelDesc), ctypes.POINTER(Reloc),
                                          ctypes.c_int, i32p, ctypes.c_int, ip]
        L.ds_fleet_kernel_id.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ip]
        L.ds_fleet_bind.argtypes = [vp, ctypes.c_int, ctypes.c_int]
        L.ds_fleet_launch.argtypes = [vp, ctypes.c_int, ctypes.c_int, u64p]
        L.ds_fleet_wait.argtypes = [vp, ctypes.c_int, ctypes.c_uint64, ctypes.c_int]
        L.ds_fleet_migrate.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.ds_fleet_global_exception.argtypes = [vp, ctypes.c_int, ctypes.c_int]
        L.ds_fleet_job_get.argtypes = [vp, ctypes.c_int, ctypes.POINTER(JobInfo)]
        L.ds_fleet_region.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp), ip, ip]
        L.ds_fleet_read_region.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp, ctypes.c_uint64]
        L.ds_fleet_migrations.argtypes = [vp, ctypes.POINTER(MigrationInfo), ctypes.c_int, ip]
        L.ds_fleet_ledger_get.argtypes = [vp, ctypes.POINTER(Ledger)]
        _setup = True
    return L


def check(rc: int):
    if rc != 0:
        L = lib()
        raise DsError(rc, f"{L.ds_fleet_last_error().decode()} / {L.ds_last_error().decode()}")


def emergency_target(failed: Sequence[bool], standby: Sequence[bool],
                     pools: Sequence[Tuple[int, int, Fraction, bool]], current: Fraction) -> int:
    """emergency_migrate's target rule; pools = (device, pctx, tier, bound).
    Returns an index into pools, or -1 (stranded)."""
    n = len(failed)
    fa = (ctypes.c_int32 * max(1, n))(*[int(x) for x in failed])
    sb = (ctypes.c_int32 * max(1, n))(*[int(x) for x in standby])
    arr = (PlacePctx * max(1, len(pools)))()
    for i, (d, p, t, b) in enumerate(pools):
        t = Fraction(t)
        arr[i] = PlacePctx(d, p, t.numerator, t.denominator, int(b), 0)
    out = ctypes.c_int(-2)
    current = Fraction(current)
    check(lib().ds_emergency_target(fa, sb, n, arr, len(pools), current.numerator, current.denominator,
                                    ctypes.byref(out)))
    return out.value


def tenant_progress(dom, tenant: int) -> Progress:
    p = Progress()
    check(lib().ds_tenant_progress(dom.h, tenant, ctypes.byref(p)))
    return p


def launch_from(dom, tenant: int, kernel: int, first_block: int, tag: int = 0) -> int:
    s = ctypes.c_uint64()
    check(lib().ds_launch_from(dom.h, tenant, kernel, tag, first_block, ctypes.byref(s)))
    return s.value


class Fleet:
    """Devices (one Domain per GPU, some standby), jobs with working-set
    regions, kernels with pointer relocations; see csrc/fleet.cpp."""

    def __init__(self):
        h = ctypes.c_void_p()
        check(lib().ds_fleet_create(ctypes.byref(h)))
        self.h = h
        self._keep = []

    def close(self):
        if self.h:
            lib().ds_fleet_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def add_device(self, dom, standby: bool = False) -> int:
        out = ctypes.c_int()
        check(lib().ds_fleet_add_device(self.h, dom.h, dom.device, int(standby), ctypes.byref(out)))
        return out.value

    def add_job(self, dev: int, name: str, priority: int = _abi.BEST_EFFORT) -> int:
        name_b = name.encode()
        self._keep.append(name_b)
        td = _abi.TenantDesc(name_b, priority)
        out = ctypes.c_int()
        check(lib().ds_fleet_add_job(self.h, dev, ctypes.byref(td), ctypes.byref(out)))
        return out.value

    def add_region(self, job: int, ptr: int, nbytes: int) -> int:
        out = ctypes.c_int()
        check(lib().ds_fleet_add_region(self.h, job, ctypes.c_void_p(ptr), nbytes, ctypes.byref(out)))
        return out.value

    def add_kernel(self, job: int, semantic_id: str, body: int, grid, args, relocs: Sequence[Tuple[str, int, int]] = (),
                   touched: Sequence[int] = ()) -> int:
        """relocs: (args field name, region, byte offset in the region)."""
        desc = make_desc(semantic_id, body, grid, args)
        self._keep.append((desc, args))
        rl = (Reloc * max(1, len(relocs)))()
        for i, (field, region, off) in enumerate(relocs):
            rl[i] = Reloc(getattr(type(args), field).offset, region, off)
        tt = (ctypes.c_int32 * max(1, len(touched)))(*touched)
        out = ctypes.c_int()
        check(lib().ds_fleet_add_kernel(self.h, job, ctypes.byref(desc), rl, len(relocs), tt, len(touched),
                                        ctypes.byref(out)))
        return out.value

    def kernel_id(self, job: int, kernel: int, dev: int) -> int:
        out = ctypes.c_int()
        check(lib().ds_fleet_kernel_id(self.h, job, kernel, dev, ctypes.byref(out)))
        return out.value

    def bind(self, job: int, pctx: int):
        check(lib().ds_fleet_bind(self.h, job, pctx))

    def launch(self, job: int, kernel: int) -> int:
        s = ctypes.c_uint64()
        check(lib().ds_fleet_launch(self.h, job, kernel, ctypes.byref(s)))
        return s.value

    def wait(self, job: int, launch: int, timeout_ms: int = 60000):
        check(lib().ds_fleet_wait(self.h, job, launch, timeout_ms))

    def migrate(self, job: int, dst_dev: int, dst_pctx: int, timeout_ms: int = 60000):
        check(lib().ds_fleet_migrate(self.h, job, dst_dev, dst_pctx, timeout_ms))

    def global_exception(self, dev: int, timeout_ms: int = 60000):
        check(lib().ds_fleet_global_exception(self.h, dev, timeout_ms))

    def job(self, job: int) -> JobInfo:
        j = JobInfo()
        check(lib().ds_fleet_job_get(self.h, job, ctypes.byref(j)))
        return j

    def region(self, job: int, region: int, dev: int = -1) -> Tuple[int, bool, bool]:
        p, res, dirty = ctypes.c_void_p(), ctypes.c_int(), ctypes.c_int()
        check(lib().ds_fleet_region(self.h, job, region, dev, ctypes.byref(p), ctypes.byref(res), ctypes.byref(dirty)))
        return p.value or 0, bool(res.value), bool(dirty.value)

    def read_region(self, job: int, region: int, out) -> None:
        """Copy the region's up-to-date bytes into `out` (a writable host
        buffer: numpy array, bytearray or ctypes array)."""
        import numpy as np
        a = np.asarray(out) if not isinstance(out, (bytearray, ctypes.Array)) else out
        if isinstance(a, np.ndarray):
            ptr, nbytes = a.ctypes.data, a.nbytes
        else:
            ptr, nbytes = ctypes.addressof((ctypes.c_char * len(a)).from_buffer(a)), len(a)
        check(lib().ds_fleet_read_region(self.h, job, region, ctypes.c_void_p(ptr), nbytes))

    def migrations(self) -> List[MigrationInfo]:
        n = ctypes.c_int()
        check(lib().ds_fleet_migrations(self.h, None, 0, ctypes.byref(n)))
        arr = (MigrationInfo * max(1, n.value))()
        check(lib().ds_fleet_migrations(self.h, arr, n.value, ctypes.byref(n)))
        return list(arr[:n.value])

    def ledger(self) -> dict:
        l = Ledger()
        check(lib().ds_fleet_ledger_get(self.h, ctypes.byref(l)))
        return {k: getattr(l, k) for k, _ in Ledger._fields_}
