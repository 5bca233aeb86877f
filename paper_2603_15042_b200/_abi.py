"""ctypes binding of the C ABI in include/detshare/ds.h (libdetshare.so).

This is the reference-side binding a Python maintainer would add (see
INTEGRATION.md); the product path is the native library.  There is no CPU
fallback: if the library or a GPU is missing, calls raise.
"""
from __future__ import annotations

import ctypes
import os

from . import build as _build

# DS_LIB: an experiment build of the same library (e.g. one lane per SM)
LIB_PATH = os.environ.get("DS_LIB", _build.LIB)

DS_MAX_TENANTS = 64
DS_MAX_SMS = 256

# ds_body_id
BODY_REDUCE_CHUNKS = 1
BODY_REDUCE_COMBINE = 2
BODY_SGEMM = 3
BODY_SPIN = 4
BODY_GEMV_BF16 = 5
BODY_ATTN_DECODE = 6
BODY_GEMM_BF16 = 7
BODY_RMSNORM = 8
BODY_EMBED = 9
BODY_ARGMAX = 10
BODY_SPLITK_REDUCE = 11
BODY_ALLREDUCE_P2P = 12
BODY_CHECKSUM = 13
MAX_DP_RANKS = 8
DP_SLOTS = 64
DP_MAX_CHUNKS = 4096  # collective.cuh kDpMaxChunks

LATENCY_CRITICAL, BEST_EFFORT = 0, 1
PREFILL, DECODE, TRAINING, OTHER = 0, 1, 2, 3

STATUS = {
    0: "Ok", 1: "InvalidTier", 2: "BindConflict", 3: "DoubleBind", 4: "CausalityViolation",
    5: "EventBudgetExceeded", 6: "TraceViolation", 7: "PlanMismatch", 8: "InvalidSplit",
    9: "ParseError", 10: "ConfigError", 100: "CudaError", 101: "NoDevice", 102: "NotRunning",
    103: "Timeout", 104: "RingFull", 105: "InvalidArgument", 106: "AlreadyRunning", 107: "TenantFailed",
    108: "RecordMutated",
}
RECORD_MUTATED = 108
TENANT_FAILED = 107
FAULT_BAD_INPUT, FAULT_INJECTED = 1, 2
ACTIVE, FAILED, STRANDED = 0, 1, 2  # VctxStatus (types.hpp:77)


class DsError(RuntimeError):
    """Mirror of corosim::SimError (errors.hpp:21-30): carries the status code."""

    def __init__(self, code: int, what: str):
        super().__init__(f"{STATUS.get(code, 'UnknownError')}: {what}")
        self.code = code


class DomainConfig(ctypes.Structure):
    _fields_ = [
        ("device", ctypes.c_int),
        ("n_tiers", ctypes.c_int),
        ("tier_num", ctypes.c_int64 * 16),
        ("tier_den", ctypes.c_int64 * 16),
        ("ring_capacity", ctypes.c_int),
        ("block_log_capacity", ctypes.c_int),
        ("lend_idle_sms", ctypes.c_int),
        ("executor_smem", ctypes.c_int),
    ]


class TenantDesc(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("priority", ctypes.c_int)]


class KernelDesc(ctypes.Structure):
    _fields_ = [
        ("semantic_id", ctypes.c_char_p),
        ("body", ctypes.c_int),
        ("grid_x", ctypes.c_uint32),
        ("grid_y", ctypes.c_uint32),
        ("grid_z", ctypes.c_uint32),
        ("block_threads", ctypes.c_uint32),
        ("args", ctypes.c_void_p),
        ("args_size", ctypes.c_uint32),
        ("phase", ctypes.c_int),
        ("request", ctypes.c_int64),
        ("decode_index", ctypes.c_int),
    ]


class Completion(ctypes.Structure):
    _fields_ = [
        ("tenant", ctypes.c_int32),
        ("kernel", ctypes.c_int32),
        ("seq", ctypes.c_uint64),
        ("launch_tag", ctypes.c_uint64),
        ("grid", ctypes.c_uint32),
        ("sms_used", ctypes.c_uint32),
        ("t_first_claim", ctypes.c_uint64),
        ("t_end", ctypes.c_uint64),
    ]


class BlockRecord(ctypes.Structure):
    _fields_ = [
        ("tenant", ctypes.c_int32),
        ("seq", ctypes.c_uint32),
        ("block", ctypes.c_uint32),
        ("smid", ctypes.c_uint16),
        ("flags", ctypes.c_uint16),
        ("t_start", ctypes.c_uint64),
        ("t_end", ctypes.c_uint64),
    ]


class SwitchRecord(ctypes.Structure):
    _fields_ = [
        ("smid", ctypes.c_uint16),
        ("from_tenant", ctypes.c_int16),
        ("to_tenant", ctypes.c_int16),
        ("pad", ctypes.c_uint16),
        ("ctl_gen", ctypes.c_uint32),
        ("t", ctypes.c_uint64),
    ]


class CtlRecord(ctypes.Structure):
    _fields_ = [("ctl_gen", ctypes.c_uint32), ("source", ctypes.c_uint32), ("t", ctypes.c_uint64)]


class Stats(ctypes.Structure):
    _fields_ = [
        ("launches_enqueued", ctypes.c_uint64),
        ("launches_completed", ctypes.c_uint64),
        ("blocks_executed", ctypes.c_uint64),
        ("ctl_changes", ctypes.c_uint64),
        ("switches", ctypes.c_uint64),
        ("block_log_entries", ctypes.c_uint64),
        ("block_log_dropped", ctypes.c_uint64),
        ("num_sms", ctypes.c_uint32),
        ("running", ctypes.c_uint32),
    ]


# ---- body argument structs (POD, mirrors csrc/bodies/*.cuh) ----
class ReduceArgs(ctypes.Structure):
    _fields_ = [("inp", ctypes.c_uint64), ("partials", ctypes.c_uint64), ("out", ctypes.c_uint64),
                ("ticket", ctypes.c_uint64), ("n", ctypes.c_int64), ("fmt", ctypes.c_int32),
                ("combine", ctypes.c_int32)]


class ChecksumArgs(ctypes.Structure):
    """Position-weighted checksum of a buffer per launch (bodies/reduce.cuh)."""
    _fields_ = [("src", ctypes.c_uint64), ("partials", ctypes.c_uint64), ("n_words", ctypes.c_int64),
                ("cap", ctypes.c_int32), ("pad", ctypes.c_int32)]


class SgemmArgs(ctypes.Structure):
    _fields_ = [("A", ctypes.c_uint64), ("B", ctypes.c_uint64), ("C", ctypes.c_uint64),
                ("M", ctypes.c_int32), ("N", ctypes.c_int32), ("K", ctypes.c_int32), ("pad", ctypes.c_int32)]


class TmaDesc(ctypes.Structure):
    _fields_ = [("w", ctypes.c_uint64 * 16)]


class GemmArgs(ctypes.Structure):
    """C[M,N] bf16 = A[M,K] . B[N,K]^T (csrc/bodies/gemm_tc.cuh)."""
    _fields_ = [("tmA", TmaDesc), ("tmB", TmaDesc), ("C", ctypes.c_uint64), ("M", ctypes.c_int32),
                ("N", ctypes.c_int32), ("K", ctypes.c_int32), ("group_m", ctypes.c_int32), ("bn", ctypes.c_int32),
                ("splits", ctypes.c_int32), ("ws", ctypes.c_uint64), ("bk", ctypes.c_int32),
                ("tma_store", ctypes.c_int32), ("abandon", ctypes.c_int32), ("l2_hint", ctypes.c_int32),
                ("tiles", ctypes.c_int32), ("fuse_fold", ctypes.c_int32),
                ("tmC", TmaDesc)]  # tmC: alignas(64)


class SplitkReduceArgs(ctypes.Structure):
    _fields_ = [("ws", ctypes.c_uint64), ("C", ctypes.c_uint64), ("M", ctypes.c_int32), ("N", ctypes.c_int32),
                ("K", ctypes.c_int32), ("group_m", ctypes.c_int32), ("bn", ctypes.c_int32), ("splits", ctypes.c_int32),
                ("rows", ctypes.c_int32), ("pad", ctypes.c_int32)]


def tensor_map_bf16(ptr: int, rows: int, cols: int, box_rows: int, box_cols: int = 64, pitch: int = 0) -> TmaDesc:
    """rows x cols bf16 (row pitch `pitch` elements, default cols): TMA boxes
    past the valid extent load zeros without reading memory; stores clip."""
    d = TmaDesc()
    if pitch and pitch != cols:
        L = lib()
        L.ds_tensor_map_bf16_2d_pitched.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                                    ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32]
        check(L.ds_tensor_map_bf16_2d_pitched(ctypes.byref(d), ctypes.c_void_p(ptr), rows, cols, pitch, box_rows,
                                              box_cols))
    else:
        check(lib().ds_tensor_map_bf16_2d(ctypes.byref(d), ctypes.c_void_p(ptr), rows, cols, box_rows, box_cols))
    return d


def measure_ffma_peak(device: int) -> float:
    """Measured fp32 FFMA TFLOP/s (no executor may be resident)."""
    v = ctypes.c_double()
    lib().ds_measure_ffma_peak.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
    check(lib().ds_measure_ffma_peak(device, ctypes.byref(v)))
    return v.value


def attn_chunk() -> int:
    """KV positions per attention pipeline stage (bodies/decode.cuh kAttnChunk) of the loaded build."""
    return int(lib().ds_attn_chunk())


def tensor_map_kv(ptr: int, rows: int, box_rows: int = 0) -> TmaDesc:
    box_rows = box_rows or attn_chunk()
    d = TmaDesc()
    check(lib().ds_tensor_map_bf16_kv(ctypes.byref(d), ctypes.c_void_p(ptr), rows, box_rows))
    return d


GEMM_BM, GEMM_BN = 128, 256


def gemm_args(A: int, B: int, C: int, M: int, N: int, K: int, group_m: int = 16, bn: int = GEMM_BN,
              splits: int = 1, ws: int = 0, bk: int = 64, tma_store: bool = True,
              abandon: bool = False, l2_hint: int = 0, tiles: int = 1, valid=None,
              fuse_fold: bool = False) -> "GemmArgs":
    """C[M,N] = A[M,K] . B[N,K]^T over tile-padded arrays.  valid = (m, n, k):
    the true extents inside them (<= M, N, K): the operand loads stop there
    (TMA zero fill, padding never read) and the TMA stores clip at (m, n
    rounded up to 8: the store unit is 16 bytes; those columns get zeros);
    None = the padded arrays are the operands."""
    if bn not in (64, 128, 256):
        raise DsError(10, f"gemm tile width {bn} not in (64, 128, 256)")
    if M % GEMM_BM or N % bn or K % 64:
        raise DsError(10, f"gemm shape {M}x{N}x{K} must tile by 128x{bn}x64")
    if splits > 1 and (not ws or splits > K // 64):
        raise DsError(10, "split-K needs a workspace and <= K/64 splits")
    if bk not in (64, 32) or (bk == 32 and bn != 256):
        raise DsError(10, "bk 32 (SWIZZLE_64B, 4 stages) is built for 128x256 tiles only")
    if tiles > 1 and (bn not in (64, 128) or splits > 1 or bk != 64 or not tma_store or abandon):
        raise DsError(10, "multi-tile GEMM blocks need bn 64/128, no split-K, bk 64, TMA stores, no abandon")
    m, n, k = valid if valid is not None else (M, N, K)
    if not (0 < m <= M and 0 < n <= N and 0 < k <= K):
        raise DsError(10, f"valid extents {valid} outside the {M}x{N}x{K} arrays")
    if valid is not None and splits <= 1 and not tma_store:
        raise DsError(10, "valid extents need TMA stores (or split-K) to keep C's padding unwritten")
    # TMA stores clip at 16-byte granularity: columns up to the next multiple
    # of 8 past n are written (zeros: B's rows >= n load as zeros)
    tmC = tensor_map_bf16(C, m, min(N, -(-n // 8) * 8), GEMM_BM, 64, pitch=N) if tma_store else TmaDesc()
    a = GemmArgs(tensor_map_bf16(A, m, k, GEMM_BM, bk, pitch=K), tensor_map_bf16(B, n, k, bn, bk, pitch=K), C, M, N,
                 K, group_m, bn, max(1, splits), ws, bk, int(tma_store))
    a.tmC = tmC
    a.abandon = int(abandon)  # False/0 off, True/1 restart, 2 spill + resume
    # L2 policy of the operand loads: bits [1:0] A, [3:2] B; 0 default (A evict_last, B none),
    # 1 evict_first, 2 evict_last, 3 evict_normal
    a.l2_hint = int(l2_hint)
    a.tiles = max(1, int(tiles))  # T consecutive raster tiles per logical block (gemm_multi)
    if fuse_fold and (splits <= 1 or abandon):
        raise DsError(10, "fuse_fold needs split-K (splits > 1) and no abandon")
    # split-K with the fold inside: the last split of each tile folds it; the
    # workspace needs splitk_ws_elems + fold_tickets (zeroed) elements
    a.fuse_fold = int(bool(fuse_fold))
    return a


def gemm_grid(M: int, N: int, bn: int = GEMM_BN, splits: int = 1, tiles: int = 1):
    n = (M // GEMM_BM) * (N // bn)
    if tiles > 1:
        return ((n + tiles - 1) // tiles, 1, 1)
    return (n * max(1, splits), 1, 1)


def fold_tickets(M: int, N: int, bn: int) -> int:
    """Workspace elements (after splitk_ws_elems) holding a fused-fold GEMM's
    per-tile tickets; zero them once, the last arriver resets its own."""
    return (M // GEMM_BM) * (N // bn)


def splitk_ws_elems(M: int, N: int, bn: int, splits: int) -> int:
    """fp32 workspace elements for a split-K GEMM: [tiles][S][128][bn]."""
    return (M // GEMM_BM) * (N // bn) * splits * GEMM_BM * bn


def splitk_reduce(ws: int, C: int, M: int, N: int, K: int, group_m: int, bn: int, splits: int, rows: int = 16):
    """(args, grid) of the split-K fold launch that follows a split GEMM:
    one block per (tile, group of `rows` rows), rows in (16, 32, 64, 128)."""
    if rows not in (16, 32, 64, 128):
        raise DsError(10, f"split-K fold rows per block {rows} not in (16, 32, 64, 128)")
    return (SplitkReduceArgs(ws, C, M, N, K, group_m, bn, splits, rows),
            ((M // GEMM_BM) * (N // bn) * (GEMM_BM // rows), 1, 1))


def fold_rows(M: int, N: int, bn: int, workers: int) -> int:
    """Widest row group (fewest, largest fold blocks) that still gives every
    worker lane a block: per-block overhead dominates 16-row groups."""
    tiles = (M // GEMM_BM) * (N // bn)
    for rows in (128, 64, 32):
        if tiles * (GEMM_BM // rows) >= workers:
            return rows
    return 16


class GemvArgs(ctypes.Structure):
    """Decode projection on tcgen05 (csrc/bodies/decode.cuh)."""
    _fields_ = [("tmW", TmaDesc), ("tmX", TmaDesc), ("out", ctypes.c_uint64), ("resid", ctypes.c_uint64),
                ("ws", ctypes.c_uint64), ("counters", ctypes.c_uint64), ("stats_in", ctypes.c_uint64),
                ("stats_out", ctypes.c_uint64), ("kcache", ctypes.c_uint64), ("vcache", ctypes.c_uint64),
                ("N", ctypes.c_int32), ("K", ctypes.c_int32), ("S", ctypes.c_int32), ("mode", ctypes.c_int32),
                ("P_in", ctypes.c_int32), ("eps", ctypes.c_float), ("pos", ctypes.c_int32), ("Lmax", ctypes.c_int32),
                ("q_dim", ctypes.c_int32), ("kv_dim", ctypes.c_int32), ("dbg", ctypes.c_uint64),
                ("w_packed", ctypes.c_uint64), ("bm", ctypes.c_int32), ("l2_pf_kb", ctypes.c_int32),
                ("sk", ctypes.c_int32), ("pair", ctypes.c_int32), ("pf_ahead", ctypes.c_int32),
                ("pad_pf", ctypes.c_int32)]


GEMV_STORE, GEMV_RESID, GEMV_SILU_MUL, GEMV_QKV = 0, 1, 2, 3


class RmsArgs(ctypes.Structure):
    _fields_ = [("x", ctypes.c_uint64), ("stats", ctypes.c_uint64), ("K", ctypes.c_int32), ("pad", ctypes.c_int32)]




class AttnArgs(ctypes.Structure):
    _fields_ = [("tmK", TmaDesc), ("tmV", TmaDesc), ("q", ctypes.c_uint64), ("out", ctypes.c_uint64),
                ("ws", ctypes.c_uint64), ("counters", ctypes.c_uint64), ("L", ctypes.c_int32),
                ("Lmax", ctypes.c_int32), ("S", ctypes.c_int32), ("scale", ctypes.c_float), ("dbg", ctypes.c_uint64),
                ("kbase", ctypes.c_uint64), ("vbase", ctypes.c_uint64), ("l2_pf_kb", ctypes.c_int32),
                ("tc", ctypes.c_int32)]


class EmbedArgs(ctypes.Structure):
    _fields_ = [("table", ctypes.c_uint64), ("tokens", ctypes.c_uint64), ("h", ctypes.c_uint64),
                ("d", ctypes.c_int32), ("vocab", ctypes.c_int32), ("stats", ctypes.c_uint64)]


class ArgmaxArgs(ctypes.Structure):
    _fields_ = [("logits", ctypes.c_uint64), ("tokens", ctypes.c_uint64), ("ws", ctypes.c_uint64),
                ("counters", ctypes.c_uint64), ("vocab", ctypes.c_int32), ("chunks", ctypes.c_int32)]


class SpinArgs(ctypes.Structure):
    _fields_ = [("out", ctypes.c_uint64), ("ns", ctypes.c_uint64)]


class EngineConfig(ctypes.Structure):
    _fields_ = [("policy", ctypes.c_char_p), ("quantum_ns", ctypes.c_int64), ("alpha", ctypes.c_double),
                ("cold_start_ns", ctypes.c_int64), ("release_on_idle", ctypes.c_int), ("fair_handover", ctypes.c_int),
                ("lend_tenant", ctypes.c_int), ("n_assignments", ctypes.c_int), ("assign_vctx", ctypes.c_int32 * 64),
                ("assign_pctx", ctypes.c_int32 * 64), ("hang_detection", ctypes.c_int), ("hang_threshold", ctypes.c_double),
                ("capture_log", ctypes.c_int), ("reset_delay_ns", ctypes.c_int64)]


class RecordDesc(ctypes.Structure):
    _fields_ = [("semantic_id", ctypes.c_char_p), ("grid_size", ctypes.c_int64),
                ("kernels", ctypes.POINTER(ctypes.c_int32)), ("n_kernels", ctypes.c_int), ("phase", ctypes.c_int),
                ("request", ctypes.c_int64), ("decode_index", ctypes.c_int), ("arrival_ns", ctypes.c_int64),
                ("request_arrival_ns", ctypes.c_int64), ("ttft_ns", ctypes.c_int64), ("tpot_ns", ctypes.c_int64),
                ("base_hint_ns", ctypes.c_int64), ("sat_num", ctypes.c_int64), ("sat_den", ctypes.c_int64)]


class RecordInfo(ctypes.Structure):
    _fields_ = [("id", ctypes.c_uint64), ("job", ctypes.c_int32), ("state", ctypes.c_int32),
                ("pctx", ctypes.c_int32), ("preempted", ctypes.c_int32), ("phase", ctypes.c_int32),
                ("decode_index", ctypes.c_int32), ("request", ctypes.c_int64), ("arrival_host_ns", ctypes.c_int64),
                ("dispatch_host_ns", ctypes.c_int64), ("finish_host_ns", ctypes.c_int64),
                ("t_first_claim", ctypes.c_uint64), ("t_end", ctypes.c_uint64), ("first_seq", ctypes.c_uint64),
                ("last_seq", ctypes.c_uint64)]


class EngineCounters(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in ("decisions", "dispatches", "completed", "preemptions", "migrations",
                                               "unbinds", "policy_errors", "failed_jobs")]


class FaultInfo(ctypes.Structure):
    _fields_ = [("code", ctypes.c_uint32), ("block", ctypes.c_uint32), ("seq", ctypes.c_uint64),
                ("first_failed", ctypes.c_uint64), ("t_ns", ctypes.c_uint64)]


class RequestOutcome(ctypes.Structure):
    _fields_ = [("inference", ctypes.c_int32), ("completed", ctypes.c_int32), ("output_tokens", ctypes.c_int32),
                ("has_slo", ctypes.c_int32), ("arrival_ns", ctypes.c_int64), ("first_decode_finish_ns", ctypes.c_int64),
                ("last_finish_ns", ctypes.c_int64), ("ttft_slo_ns", ctypes.c_int64), ("tpot_slo_ns", ctypes.c_int64),
                ("kernels_done", ctypes.c_int64)]


class Dist(ctypes.Structure):
    _fields_ = [("count", ctypes.c_int64), ("mean", ctypes.c_double)] + [
        (f"{p}_{x}", ctypes.c_int64) for p in ("p50", "p90", "p99") for x in ("num", "den")]


class Metrics(ctypes.Structure):
    _fields_ = [("makespan_ns", ctypes.c_int64), ("kernels_completed", ctypes.c_int64),
                ("inference_completed", ctypes.c_int64), ("training_kernels_completed", ctypes.c_int64),
                ("inference_throughput", ctypes.c_double), ("training_throughput", ctypes.c_double),
                ("ttft", Dist), ("tpot", Dist), ("tpot_excluded", ctypes.c_int64), ("slo_requests", ctypes.c_int64),
                ("ttft_violations", ctypes.c_int64), ("tpot_violations", ctypes.c_int64),
                ("ttft_violation_rate", ctypes.c_double), ("tpot_violation_rate", ctypes.c_double)]


class RequestTemplate(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("prompt_tokens", ctypes.c_int), ("prompt_tokens_max", ctypes.c_int),
                ("output_tokens", ctypes.c_int), ("output_tokens_max", ctypes.c_int), ("iterations", ctypes.c_int),
                ("streams", ctypes.c_int)]


class Request(ctypes.Structure):
    _fields_ = [("arrival_q", ctypes.c_int64), ("stream", ctypes.c_int32), ("kind", ctypes.c_int32),
                ("prompt_tokens", ctypes.c_int32), ("output_tokens", ctypes.c_int32), ("iterations", ctypes.c_int32),
                ("pad", ctypes.c_int32)]


class ExpandParams(ctypes.Structure):
    _fields_ = [("tokens_per_grid_unit", ctypes.c_int64), ("decode_grid", ctypes.c_int64),
                ("train_grid", ctypes.c_int64), ("default_iterations", ctypes.c_int32), ("pad", ctypes.c_int32)]


class KernelPlan(ctypes.Structure):
    _fields_ = [("request", ctypes.c_int64), ("job", ctypes.c_int32), ("phase", ctypes.c_int32),
                ("decode_index", ctypes.c_int32), ("pad", ctypes.c_int32), ("grid_size", ctypes.c_int64),
                ("arrival_q", ctypes.c_int64), ("lab_seed", ctypes.c_uint64)]


REQ_INFERENCE, REQ_TRAINING = 0, 1


class AllreduceArgs(ctypes.Structure):
    """csrc/bodies/collective.cuh"""
    _fields_ = [("grad", ctypes.c_uint64 * 8), ("flags", ctypes.c_uint64 * 8), ("out", ctypes.c_uint64),
                ("outs", ctypes.c_uint64 * 8),
                ("n", ctypes.c_int64), ("world", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("chunk", ctypes.c_int32), ("pad", ctypes.c_int32)]


class Region(ctypes.Structure):
    _fields_ = [("id", ctypes.c_int32), ("dirty", ctypes.c_int32), ("bytes", ctypes.c_uint64),
                ("resident_mask", ctypes.c_uint64)]


class TenantDemand(ctypes.Structure):
    _fields_ = [("priority", ctypes.c_int32), ("phase", ctypes.c_int32), ("hbm_frac", ctypes.c_double),
                ("tensor_frac", ctypes.c_double), ("mem_gb", ctypes.c_double)]

# ---- user policies over the C ABI (ds_policy_vtable) ----
VIEW_MAX_PCTX = VIEW_MAX_VCTX = 64
VIEW_MAX_DEVICES = 8
DISPATCH_DIRECT, DISPATCH_REMAP, DISPATCH_DEFER, PREEMPT, NO_ACTION = 0, 1, 2, 3, 4


class ViewPctx(ctypes.Structure):
    _fields_ = [("id", ctypes.c_int32), ("device", ctypes.c_int32), ("tier_num", ctypes.c_int64),
                ("tier_den", ctypes.c_int64), ("standby", ctypes.c_int32), ("available", ctypes.c_int32),
                ("bound", ctypes.c_int32), ("has_running", ctypes.c_int32), ("running_kernel", ctypes.c_uint64),
                ("running_semantic_id", ctypes.c_char_p), ("running_grid", ctypes.c_int64),
                ("running_remaining_ns", ctypes.c_int64), ("running_phase", ctypes.c_int32),
                ("running_priority", ctypes.c_int32)]


class ViewVctx(ctypes.Structure):
    _fields_ = [("id", ctypes.c_int32), ("priority", ctypes.c_int32), ("quarantined", ctypes.c_int32),
                ("bound", ctypes.c_int32), ("pending", ctypes.c_int64), ("head_phase", ctypes.c_int32),
                ("decoding", ctypes.c_int32)]


class View(ctypes.Structure):
    _fields_ = [("now_ns", ctypes.c_int64), ("n_pctx", ctypes.c_int32), ("n_vctx", ctypes.c_int32),
                ("pctx", ViewPctx * VIEW_MAX_PCTX), ("vctx", ViewVctx * VIEW_MAX_VCTX),
                ("n_devices", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("bound_tier_sum_num", ctypes.c_int64 * VIEW_MAX_DEVICES),
                ("bound_tier_sum_den", ctypes.c_int64 * VIEW_MAX_DEVICES),
                ("min_tier_num", ctypes.c_int64 * VIEW_MAX_DEVICES), ("min_tier_den", ctypes.c_int64 * VIEW_MAX_DEVICES),
                ("active_vctx_count", ctypes.c_int64), ("predictor", ctypes.c_void_p)]


class LaunchCtx(ctypes.Structure):
    _fields_ = [("vctx", ctypes.c_int32), ("has_kernel", ctypes.c_int32), ("kernel_id", ctypes.c_uint64),
                ("semantic_id", ctypes.c_char_p), ("grid_size", ctypes.c_int64), ("base_hint_ns", ctypes.c_int64),
                ("sat_num", ctypes.c_int64), ("sat_den", ctypes.c_int64), ("phase", ctypes.c_int32),
                ("decode_index", ctypes.c_int32), ("request", ctypes.c_int64), ("arrival_ns", ctypes.c_int64),
                ("request_arrival_ns", ctypes.c_int64), ("has_slo", ctypes.c_int32), ("pool_exhausted", ctypes.c_int32),
                ("ttft_ns", ctypes.c_int64), ("tpot_ns", ctypes.c_int64)]


class Decision(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("target", ctypes.c_int32)]


HOOK = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.POINTER(View), ctypes.POINTER(LaunchCtx), ctypes.POINTER(Decision))
ORDER_KEY = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(LaunchCtx))
REVIEW = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(View), ctypes.POINTER(ctypes.c_int64))
DESTROY = ctypes.CFUNCTYPE(None, ctypes.c_void_p)


class PolicyVtable(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("on_launch", HOOK), ("on_completion", HOOK), ("on_congestion", HOOK),
                ("launch_order_key", ORDER_KEY), ("next_review_time", REVIEW), ("destroy", DESTROY)]


class Ledger(ctypes.Structure):
    """OverheadLedger measured on the device (ds_ledger)."""
    _fields_ = [("ctx_switches", ctypes.c_uint64), ("ctx_switch_total_ns", ctypes.c_uint64),
                ("preemptions", ctypes.c_uint64), ("preempt_total_ns", ctypes.c_uint64),
                ("migrations", ctypes.c_uint64), ("migration_total_ns", ctypes.c_uint64),
                ("demand_faults", ctypes.c_uint64), ("demand_fault_total_ns", ctypes.c_uint64)]


class KernelInfo(ctypes.Structure):
    _fields_ = [("fingerprint", ctypes.c_uint64), ("args_device", ctypes.c_uint64), ("args_size", ctypes.c_uint32),
                ("grid", ctypes.c_uint32), ("body", ctypes.c_int32), ("phase", ctypes.c_int32)]


class JobSpan(ctypes.Structure):
    _fields_ = [("first_arrival_ns", ctypes.c_int64), ("last_finish_ns", ctypes.c_int64), ("valid", ctypes.c_int32),
                ("pad", ctypes.c_int32)]


# exported symbols the header declares (checked by the CPU test suite)
EXPORTS = [
    "ds_status_name", "ds_last_error", "ds_abi_version", "ds_domain_create", "ds_domain_destroy",
    "ds_num_sms", "ds_smids", "ds_pctx_count", "ds_pctx_info", "ds_tenant_register", "ds_kernel_register",
    "ds_start", "ds_stop", "ds_launch", "ds_launch_atomized", "ds_wait_tenant", "ds_poll", "ds_bind",
    "ds_unbind", "ds_migrate", "ds_preempt", "ds_bound_pctx", "ds_quota_set", "ds_quota_get",
    "ds_set_lend", "ds_quota_at_claim", "ds_quota_periodic", "ds_stats_get", "ds_transcript",
    "ds_logical_progress", "ds_block_log", "ds_switch_log", "ds_ctl_log", "ds_clear_logs",
    "ds_globaltimer", "ds_debug_dump", "ds_ctl_roundtrip", "ds_measure_ffma_peak", "ds_solo_launch", "ds_solo_launch_registered", "ds_solo_trace", "ds_body_smem",
    "ds_tensor_map_bf16_2d", "ds_tensor_map_bf16_2d_pitched", "ds_tensor_map_bf16_kv", "ds_attn_chunk", "ds_engine_last_error", "ds_engine_create", "ds_engine_destroy",
    "ds_engine_add_job", "ds_engine_submit", "ds_engine_start", "ds_engine_stop", "ds_engine_now", "ds_engine_wait",
    "ds_engine_record", "ds_engine_counters_get", "ds_engine_transcript", "ds_engine_predict", "ds_policy_names",
    "ds_gen_poisson", "ds_gen_burst", "ds_expand_workload", "ds_place_tenants",
    "ds_ipc_alloc", "ds_ipc_free", "ds_ipc_handle", "ds_ipc_open", "ds_ipc_close", "ds_dp_abort",
    "ds_engine_event_log", "ds_engine_quarantines", "ds_quota_triggers_reset",
    "ds_compute_migration_set", "ds_full_eager_set", "ds_migrate_regions",
    "ds_fault_inject", "ds_tenant_fault", "ds_engine_fault_local", "ds_engine_job_status",
    "ds_compute_metrics", "ds_set_lane_split", "ds_tenant_abandonable", "ds_set_drain_exit",
    "ds_engine_create_with_policy", "ds_engine_snapshot", "ds_predictor_predict", "ds_predict_hol_blocking",
    "ds_builtin_decide", "ds_add_normalization", "ds_seeded_values", "ds_round_to", "ds_ledger_get",
    "ds_kernel_info_get", "ds_verify_kernels", "ds_engine_ledger", "ds_engine_job_fingerprint",
    "ds_launch_from", "ds_tenant_progress", "ds_emergency_target", "ds_fleet_create", "ds_fleet_destroy",
    "ds_fleet_add_device", "ds_fleet_add_job", "ds_fleet_add_region", "ds_fleet_add_kernel", "ds_fleet_kernel_id",
    "ds_fleet_bind", "ds_fleet_launch", "ds_fleet_wait", "ds_fleet_migrate", "ds_fleet_global_exception",
    "ds_fleet_job_get", "ds_fleet_region", "ds_fleet_read_region", "ds_fleet_migrations", "ds_fleet_ledger_get", "ds_fleet_last_error",
]

_lib = None


def lib():
    """Load libdetshare.so (building it in-tree if absent).  Raises if it
    cannot be loaded — there is no fallback path."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            _build.build()
        L = ctypes.CDLL(LIB_PATH)
        vp = ctypes.c_void_p
        i32p = ctypes.POINTER(ctypes.c_int32)
        L.ds_status_name.restype = ctypes.c_char_p
        L.ds_status_name.argtypes = [ctypes.c_int]
        L.ds_last_error.restype = ctypes.c_char_p
        L.ds_domain_create.argtypes = [ctypes.POINTER(DomainConfig), ctypes.POINTER(vp)]
        L.ds_domain_destroy.argtypes = [vp]
        L.ds_num_sms.argtypes = [vp, ctypes.POINTER(ctypes.c_int)]
        L.ds_smids.argtypes = [vp, ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        L.ds_pctx_count.argtypes = [vp, ctypes.POINTER(ctypes.c_int)]
        L.ds_pctx_info.argtypes = [vp, ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                                   ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
        L.ds_tenant_register.argtypes = [vp, ctypes.POINTER(TenantDesc), ctypes.POINTER(ctypes.c_int)]
        L.ds_kernel_register.argtypes = [vp, ctypes.POINTER(KernelDesc), ctypes.POINTER(ctypes.c_int)]
        L.ds_start.argtypes = [vp]
        L.ds_stop.argtypes = [vp]
        L.ds_launch.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64)]
        L.ds_launch_atomized.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_int64,
                                         ctypes.c_int64, ctypes.POINTER(ctypes.c_uint64)]
        L.ds_wait_tenant.argtypes = [vp, ctypes.c_int, ctypes.c_uint64, ctypes.c_int]
        L.ds_poll.argtypes = [vp, ctypes.POINTER(Completion), ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        L.ds_bind.argtypes = [vp, ctypes.c_int, ctypes.c_int]
        L.ds_unbind.argtypes = [vp, ctypes.c_int]
        L.ds_migrate.argtypes = [vp, ctypes.c_int, ctypes.c_int]
        L.ds_preempt.argtypes = [vp, ctypes.c_int]
        L.ds_bound_pctx.argtypes = [vp, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        L.ds_quota_set.argtypes = [vp, i32p, i32p, ctypes.c_int]
        L.ds_quota_get.argtypes = [vp, i32p, i32p, ctypes.c_int]
        L.ds_set_lend.argtypes = [vp, ctypes.c_int]
        L.ds_quota_at_claim.argtypes = [vp, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint32, i32p, i32p, ctypes.c_int]
        L.ds_quota_periodic.argtypes = [vp, ctypes.c_uint64, i32p, i32p, i32p, i32p, ctypes.c_int]
        L.ds_stats_get.argtypes = [vp, ctypes.POINTER(Stats)]
        L.ds_transcript.argtypes = [vp, ctypes.c_int, i32p, ctypes.POINTER(ctypes.c_uint32), ctypes.c_int,
                                    ctypes.POINTER(ctypes.c_int)]
        L.ds_logical_progress.argtypes = [vp, ctypes.c_int, ctypes.POINTER(ctypes.c_int64)]
        L.ds_block_log.argtypes = [vp, ctypes.POINTER(BlockRecord), ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]
        L.ds_switch_log.argtypes = [vp, ctypes.POINTER(SwitchRecord), ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]
        L.ds_ctl_log.argtypes = [vp, ctypes.POINTER(CtlRecord), ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]
        L.ds_clear_logs.argtypes = [vp]
        L.ds_globaltimer.argtypes = [vp, ctypes.POINTER(ctypes.c_uint64)]
        L.ds_debug_dump.argtypes = [vp, ctypes.c_char_p, ctypes.c_int64]
        L.ds_ctl_roundtrip.argtypes = [vp, ctypes.c_int, ctypes.POINTER(ctypes.c_uint64)]
        L.ds_solo_launch.argtypes = [ctypes.c_int, ctypes.POINTER(KernelDesc), vp]
        L.ds_solo_launch_registered.argtypes = [vp, ctypes.c_int, vp]
        L.ds_body_smem.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_uint32)]
        L.ds_tensor_map_bf16_2d.argtypes = [vp, vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32]
        L.ds_tensor_map_bf16_kv.argtypes = [vp, vp, ctypes.c_uint64, ctypes.c_uint32]
        L.ds_engine_last_error.restype = ctypes.c_char_p
        L.ds_engine_create.argtypes = [vp, ctypes.POINTER(EngineConfig), ctypes.POINTER(vp)]
        L.ds_engine_destroy.argtypes = [vp]
        L.ds_engine_add_job.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        L.ds_engine_submit.argtypes = [vp, ctypes.c_int, ctypes.POINTER(RecordDesc), ctypes.POINTER(ctypes.c_uint64)]
        L.ds_engine_start.argtypes = [vp]
        L.ds_engine_stop.argtypes = [vp]
        L.ds_engine_now.argtypes = [vp, ctypes.POINTER(ctypes.c_int64)]
        L.ds_engine_wait.argtypes = [vp, ctypes.c_uint64, ctypes.c_int]
        L.ds_engine_record.argtypes = [vp, ctypes.c_uint64, ctypes.POINTER(RecordInfo)]
        L.ds_engine_counters_get.argtypes = [vp, ctypes.POINTER(EngineCounters)]
        L.ds_engine_transcript.argtypes = [vp, ctypes.c_int, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int,
                                           ctypes.POINTER(ctypes.c_int)]
        L.ds_engine_predict.argtypes = [vp, ctypes.c_char_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]
        L.ds_policy_names.argtypes = [ctypes.c_char_p, ctypes.c_int]
        L.ds_gen_poisson.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.POINTER(RequestTemplate),
                                     ctypes.c_uint64, ctypes.POINTER(Request), ctypes.c_int64,
                                     ctypes.POINTER(ctypes.c_int64)]
        L.ds_gen_burst.argtypes = [ctypes.c_double] * 5 + [ctypes.POINTER(RequestTemplate), ctypes.c_uint64,
                                                           ctypes.POINTER(Request), ctypes.c_int64,
                                                           ctypes.POINTER(ctypes.c_int64)]
        L.ds_ipc_alloc.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.POINTER(vp)]
        L.ds_ipc_free.argtypes = [ctypes.c_int, vp]
        L.ds_ipc_handle.argtypes = [vp, ctypes.c_char_p]
        L.ds_ipc_open.argtypes = [ctypes.c_int, ctypes.c_char_p, ctypes.POINTER(vp)]
        L.ds_ipc_close.argtypes = [ctypes.c_int, vp]
        L.ds_quota_triggers_reset.argtypes = [vp]
        i32p_, u64p_, ip_ = ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_int)
        L.ds_compute_migration_set.argtypes = [ctypes.POINTER(Region), ctypes.c_int, i32p_, ctypes.c_int, ctypes.c_int,
                                               i32p_, ip_, u64p_, i32p_, ip_, u64p_]
        L.ds_full_eager_set.argtypes = [ctypes.POINTER(Region), ctypes.c_int, i32p_, ip_, u64p_]
        L.ds_migrate_regions.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp), ctypes.POINTER(vp), u64p_,
                                         ctypes.c_int, vp]
        L.ds_engine_event_log.argtypes = [vp, ctypes.c_char_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]
        L.ds_engine_quarantines.argtypes = [vp, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64),
                                            ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        L.ds_dp_abort.argtypes = [ctypes.c_int, vp]
        L.ds_fault_inject.argtypes = [vp, ctypes.c_int, ctypes.c_uint32]
        L.ds_tenant_fault.argtypes = [vp, ctypes.c_int, ctypes.POINTER(FaultInfo)]
        L.ds_engine_fault_local.argtypes = [vp, ctypes.c_int]
        L.ds_set_lane_split.argtypes = [vp, ctypes.c_int]
        L.ds_tenant_abandonable.argtypes = [vp, ctypes.c_int, ctypes.c_int]
        L.ds_set_drain_exit.argtypes = [vp, ctypes.c_int, ctypes.c_uint64]
        L.ds_engine_create_with_policy.argtypes = [vp, ctypes.POINTER(EngineConfig), ctypes.POINTER(PolicyVtable), vp,
                                                   ctypes.POINTER(vp)]
        L.ds_engine_snapshot.argtypes = [vp, ctypes.POINTER(View)]
        L.ds_predictor_predict.argtypes = [vp, ctypes.c_char_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int64,
                                           ctypes.POINTER(ctypes.c_int64)]
        L.ds_predict_hol_blocking.argtypes = [ctypes.POINTER(View), ctypes.c_int, ctypes.POINTER(ctypes.c_int64)]
        L.ds_builtin_decide.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(View), ctypes.POINTER(LaunchCtx),
                                        ctypes.c_int64, ctypes.POINTER(Decision)]
        L.ds_add_normalization.argtypes = [ctypes.POINTER(JobSpan), ctypes.POINTER(JobSpan), ctypes.c_int,
                                           ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                                           ctypes.POINTER(ctypes.c_double)]
        L.ds_seeded_values.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, ctypes.POINTER(ctypes.c_uint32)]
        L.ds_round_to.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.POINTER(ctypes.c_uint32)]
        L.ds_ledger_get.argtypes = [vp, ctypes.POINTER(Ledger)]
        L.ds_kernel_info_get.argtypes = [vp, ctypes.c_int, ctypes.POINTER(KernelInfo)]
        L.ds_verify_kernels.argtypes = [vp, ctypes.POINTER(ctypes.c_int)]
        L.ds_engine_ledger.argtypes = [vp, ctypes.POINTER(Ledger)]
        L.ds_engine_job_fingerprint.argtypes = [vp, ctypes.c_int, ctypes.POINTER(ctypes.c_uint64)]
        L.ds_compute_metrics.argtypes = [ctypes.POINTER(RequestOutcome), ctypes.c_int64, ctypes.c_int64,
                                         ctypes.c_int64, ctypes.POINTER(Metrics)]
        L.ds_engine_job_status.argtypes = [vp, ctypes.c_int, ip_]
        L.ds_place_tenants.argtypes = [ctypes.POINTER(TenantDemand), ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                       ctypes.POINTER(ctypes.c_int32)]
        L.ds_expand_workload.argtypes = [ctypes.POINTER(Request), ctypes.c_int64, ctypes.POINTER(ExpandParams),
                                         ctypes.POINTER(KernelPlan), ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        raise DsError(rc, (lib().ds_last_error() or b"").decode())


def check_engine(rc: int) -> None:
    if rc != 0:
        raise DsError(rc, (lib().ds_engine_last_error() or b"").decode())
