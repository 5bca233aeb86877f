"""Data-parallel training tenant: gradient all-reduce over NVLink peer memory
as an executor body (csrc/bodies/collective.cuh: reduce-scatter + all-gather
in one launch, rank-ordered fp32 sums), so the collective runs under the SM
arbiter on the tenant's own quota.

One process per GPU: each rank allocates its gradient / output / flag
buffers with ``ds_ipc_alloc``, the 64-byte IPC handles travel over the host
process group (``torch.distributed``: plumbing), and every rank opens its
peers' buffers.  ``peer_table`` is the rank-ordered pointer table the body
reads; ``virtual_group`` builds the same tables for W virtual ranks on one
GPU (W tenants of one domain), which is how the body is tested on a
single B200.
"""
from __future__ import annotations

import ctypes
from typing import Callable, List, Sequence

from . import _abi
from ._abi import check, lib

FLAG_BYTES = (2 * _abi.DP_SLOTS + 8 + _abi.DP_MAX_CHUNKS) * 8  # ready, done, abort (+pad), chunk epochs


def _alloc(device: int, nbytes: int) -> int:
    p = ctypes.c_void_p()
    check(lib().ds_ipc_alloc(device, nbytes, ctypes.byref(p)))
    return p.value


def ipc_handle(ptr: int) -> bytes:
    buf = ctypes.create_string_buffer(64)
    check(lib().ds_ipc_handle(ctypes.c_void_p(ptr), buf))
    return buf.raw


def ipc_open(device: int, handle: bytes) -> int:
    p = ctypes.c_void_p()
    check(lib().ds_ipc_open(device, handle, ctypes.byref(p)))
    return p.value


def peer_table(own: int, rank: int, handles: Sequence[bytes], open_fn: Callable[[bytes], int]) -> List[int]:
    """Rank-ordered pointers: own buffer at `rank`, opened peers elsewhere."""
    return [own if r == rank else open_fn(h) for r, h in enumerate(handles)]


def make_args(grads: Sequence[int], flags: Sequence[int], outs: Sequence[int], n: int, rank: int,
              chunk: int = 1 << 16) -> _abi.AllreduceArgs:
    """Rank `rank`'s arguments: every rank's gradient, flag and output
    buffers in rank order (own entries local, peers' opened over IPC)."""
    world = len(grads)
    if world > _abi.MAX_DP_RANKS or n % 8 or chunk % 8 or len(outs) != world or len(flags) != world:
        raise _abi.DsError(10, "DP all-reduce: <= 8 ranks, n and chunk multiples of 8, one buffer per rank")
    if (n + chunk - 1) // chunk > _abi.DP_MAX_CHUNKS:
        raise _abi.DsError(10, f"DP all-reduce: more than {_abi.DP_MAX_CHUNKS} chunks")
    a = _abi.AllreduceArgs()
    for r in range(world):
        a.grad[r] = grads[r]
        a.flags[r] = flags[r]
        a.outs[r] = outs[r]
    a.out, a.n, a.world, a.rank, a.chunk = outs[rank], n, world, rank, chunk
    return a


def shard_bounds(rank: int, G: int, world: int) -> tuple:
    """Chunks [lo, hi) rank `rank` reduces (collective.cuh: lo(r) = r G / W)."""
    return rank * G // world, (rank + 1) * G // world


def block_chunk(rank: int, j: int, G: int, world: int) -> int:
    """Chunk that logical block j of rank `rank` handles: its own shard
    first in claim order, then the others' (collective.cuh)."""
    return (shard_bounds(rank, G, world)[0] + j) % G


def grid_for(n: int, chunk: int = 1 << 16):
    return ((n + chunk - 1) // chunk, 1, 1)


class DpGroup:
    """This rank's share of a DP tenant's all-reduce (multi-process)."""

    def __init__(self, device: int, n: int, rank: int, world: int, gather_fn, chunk: int = 1 << 16):
        self.device, self.n, self.rank, self.world, self.chunk = device, n, rank, world, chunk
        self.grad = _alloc(device, 2 * n)
        self.out = _alloc(device, 2 * n)
        self.flags = _alloc(device, FLAG_BYTES)
        hs = gather_fn((ipc_handle(self.grad), ipc_handle(self.flags), ipc_handle(self.out)))
        opener = lambda h: ipc_open(device, h)  # noqa: E731
        self.grads = peer_table(self.grad, rank, [h[0] for h in hs], opener)
        self.flag_ptrs = peer_table(self.flags, rank, [h[1] for h in hs], opener)
        self.outs = peer_table(self.out, rank, [h[2] for h in hs], opener)
        self.args = make_args(self.grads, self.flag_ptrs, self.outs, n, rank, chunk)

    def abort(self):
        """Release this rank's blocks still waiting for a peer (shutdown)."""
        check(lib().ds_dp_abort(self.device, ctypes.c_void_p(self.flags)))

    def register(self, dom, semantic_id="train/dp_allreduce") -> int:
        return dom.kernel(semantic_id, _abi.BODY_ALLREDUCE_P2P, grid_for(self.n, self.chunk), self.args,
                          phase=_abi.TRAINING)


def virtual_group(device: int, n: int, world: int, chunk: int = 1 << 16):
    """W virtual ranks on one GPU: per rank (grad, out, flags) buffers and its
    AllreduceArgs over local pointers."""
    grads = [_alloc(device, 2 * n) for _ in range(world)]
    outs = [_alloc(device, 2 * n) for _ in range(world)]
    flags = [_alloc(device, FLAG_BYTES) for _ in range(world)]
    args = [make_args(grads, flags, outs, n, r, chunk) for r in range(world)]
    return grads, outs, flags, args
