"""Working-set migration across places over the native
library: the reference's compute_migration_set / full_eager_set
(proj/src/runtime/migration.cpp:21-58) and the peer-to-peer eager copy."""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Dict, List, Sequence, Set, Tuple

from . import _abi
from ._abi import check, lib


@dataclass
class Region:
    id: int
    bytes: int
    dirty: bool = False
    resident_on: Set[int] = field(default_factory=set)  # places (pctx or GPU ids < 64)


def _arr(ws: Sequence[Region]):
    a = (_abi.Region * max(1, len(ws)))()
    for i, r in enumerate(ws):
        mask = 0
        for p in r.resident_on:
            mask |= 1 << p
        a[i] = _abi.Region(r.id, int(r.dirty), r.bytes, mask)
    return a


def compute_migration_set(ws: Sequence[Region], touched: Sequence[int], dst: int):
    """-> (eager ids, eager bytes, lazy ids, lazy bytes); DsError(TraceViolation)
    if a touched region is outside the working set."""
    n = len(ws)
    t = (ctypes.c_int32 * max(1, len(touched)))(*touched)
    e, l = (ctypes.c_int32 * max(1, n))(), (ctypes.c_int32 * max(1, n))()
    ne, nl = ctypes.c_int(), ctypes.c_int()
    eb, lb = ctypes.c_uint64(), ctypes.c_uint64()
    rc = lib().ds_compute_migration_set(_arr(ws), n, t, len(touched), dst, e, ctypes.byref(ne), ctypes.byref(eb), l,
                                        ctypes.byref(nl), ctypes.byref(lb))
    if rc:
        raise _abi.DsError(rc, "compute_migration_set")
    return list(e[:ne.value]), eb.value, list(l[:nl.value]), lb.value


def full_eager_set(ws: Sequence[Region]):
    n = len(ws)
    e = (ctypes.c_int32 * max(1, n))()
    ne, eb = ctypes.c_int(), ctypes.c_uint64()
    check(lib().ds_full_eager_set(_arr(ws), n, e, ctypes.byref(ne), ctypes.byref(eb)))
    return list(e[:ne.value]), eb.value


def migrate_regions(src_device: int, dst_device: int, pairs: Sequence[Tuple[int, int, int]], stream: int = 0):
    """Copy (src_ptr, dst_ptr, bytes) regions peer to peer on the copy engines."""
    n = len(pairs)
    src = (ctypes.c_void_p * max(1, n))(*[p[0] for p in pairs])
    dst = (ctypes.c_void_p * max(1, n))(*[p[1] for p in pairs])
    nb = (ctypes.c_uint64 * max(1, n))(*[p[2] for p in pairs])
    check(lib().ds_migrate_regions(src_device, dst_device, src, dst, nb, n, ctypes.c_void_p(stream)))
