/*
 * detshare B200 GPU-coroutine runtime — C ABI (the drop-in boundary).
 *
 * Plain C types only: no torch, no C++ types, no exceptions across the ABI.
 * Every entry point returns a ds_status (0 = ok).  Status codes 1..10 follow
 * the reference's Errc order (proj/include/corosim/errors.hpp:8-19); codes
 * >= 100 are runtime/CUDA conditions the CPU reference never had.
 *
 * Reference interfaces each group replaces (file:line under /root/reference/proj):
 *   domain/pool     create_pool, Device, QuotaTier     include/corosim/core/types.hpp:19-21,102-109,133-137
 *   tenants         JobSpec -> VirtualContext          include/corosim/engine/engine.hpp:43-48; core/types.hpp:80-88
 *   kernels         immutable Kernel record            include/corosim/core/types.hpp:29-68
 *   launch          kernel arrival -> pending queue    src/engine/engine.cpp:810-819 (on_arrival)
 *   bind/unbind     BindingTable, bind, unbind         include/corosim/core/types.hpp:112-131; src/core/types.cpp:62-85
 *   preempt         signal_preempt / rck_flag          src/engine/engine.cpp:756-806; core/types.hpp:97
 *   migrate         begin_migration (remap)            src/engine/engine.cpp:620-672
 *   transcript      SimulationReport.vctx_transcripts  include/corosim/engine/engine.hpp:124-129
 *   solo baseline   exclusive_baseline                 src/engine/engine.cpp:1400-1417
 *   policy engine   SimEngine + Policy hooks           include/corosim/engine/engine.hpp:152-170; policy/policy.hpp:97-126
 */
#ifndef DETSHARE_DS_H
#define DETSHARE_DS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DS_ABI_VERSION 1
#define DS_MAX_TENANTS 64
#define DS_MAX_SMS 256
#define DS_MASK_WORDS 8 /* 8 x 32 bits = 256 SM slots */

typedef enum ds_status {
    DS_OK = 0,
    /* Errc (errors.hpp:8-19), same order */
    DS_INVALID_TIER = 1,
    DS_BIND_CONFLICT = 2,
    DS_DOUBLE_BIND = 3,
    DS_CAUSALITY_VIOLATION = 4,
    DS_EVENT_BUDGET_EXCEEDED = 5,
    DS_TRACE_VIOLATION = 6,
    DS_PLAN_MISMATCH = 7,
    DS_INVALID_SPLIT = 8,
    DS_PARSE_ERROR = 9,
    DS_CONFIG_ERROR = 10,
    /* runtime conditions */
    DS_CUDA_ERROR = 100,
    DS_NO_DEVICE = 101,
    DS_NOT_RUNNING = 102,
    DS_TIMEOUT = 103,
    DS_RING_FULL = 104,
    DS_INVALID_ARGUMENT = 105,
    DS_ALREADY_RUNNING = 106,
    DS_TENANT_FAILED = 107,     /* the tenant raised a local exception (ds_tenant_fault) */
    DS_RECORD_MUTATED = 108     /* an immutable kernel record changed during the run (engine.cpp:1379-1383) */
} ds_status;

/* Local-exception codes a tenant body raises (any nonzero code may be injected). */
#define DS_FAULT_BAD_INPUT 1u   /* e.g. a token id outside the embedding table */
#define DS_FAULT_INJECTED 2u    /* ds_engine_fault_local */

/* Tenant bodies compiled into the executor ("unmodified kernels": each is a
 * device function of the logical block index, also launchable solo as a
 * plain __global__ grid). */
typedef enum ds_body_id {
    DS_BODY_NONE = 0,
    DS_BODY_REDUCE_CHUNKS = 1,  /* block c folds chunk c (reduction.cpp:22-34) */
    DS_BODY_REDUCE_COMBINE = 2, /* grid 1: fold partials left-to-right (reduction.cpp:67-70) */
    DS_BODY_SGEMM = 3,          /* fp32 C = A.B, 64x64 tiles, k-ascending fma */
    DS_BODY_SPIN = 4,           /* test body: busy-wait ns per block, writes (smid, t) */
    DS_BODY_GEMV_BF16 = 5,      /* decode projection: y[32,N] = x[32,K] W^T (+fused epilogue) */
    DS_BODY_ATTN_DECODE = 6,    /* GQA decode attention over a KV cache */
    DS_BODY_GEMM_BF16 = 7,      /* training GEMM on tcgen05/TMEM */
    DS_BODY_RMSNORM = 8,        /* row RMS statistics for the decode tenant */
    DS_BODY_EMBED = 9,          /* token embedding gather (decode step input) */
    DS_BODY_ARGMAX = 10,        /* greedy sampling (decode step result) */
    DS_BODY_SPLITK_REDUCE = 11, /* fold a split-K GEMM's fp32 partials in fixed split order */
    DS_BODY_ALLREDUCE_P2P = 12, /* DP gradient all-reduce over NVLink peer memory, rank-ordered sum */
    DS_BODY_CHECKSUM = 13,      /* position-weighted integer checksum of a buffer, one slot per launch */
    DS_BODY_COUNT = 14
} ds_body_id;

typedef enum ds_priority { DS_LATENCY_CRITICAL = 0, DS_BEST_EFFORT = 1 } ds_priority; /* types.hpp:24 */
typedef enum ds_phase { DS_PREFILL = 0, DS_DECODE = 1, DS_TRAINING = 2, DS_OTHER = 3 } ds_phase; /* types.hpp:23 */

typedef struct ds_domain ds_domain;

typedef struct ds_domain_config {
    int device;                /* CUDA ordinal */
    int n_tiers;               /* pool: one pctx per tier (create_pool, types.cpp:87-106) */
    int64_t tier_num[16];      /* tier fraction = num/den in (0, 1] */
    int64_t tier_den[16];
    int ring_capacity;         /* launches in flight per tenant (power of two, <= 4096) */
    int block_log_capacity;    /* logical-block claim log entries (0 = off) */
    int lend_idle_sms;         /* 1: unbound SMs run best-effort tenants' blocks until reclaimed */
    int executor_smem;         /* dynamic smem per worker CTA (bytes); 0 = default */
} ds_domain_config;

typedef struct ds_tenant_desc {
    const char* name;
    int priority; /* ds_priority */
} ds_tenant_desc;

typedef struct ds_kernel_desc {
    const char* semantic_id; /* KernelSignature.semantic_id (types.hpp:29-34) */
    int body;                /* ds_body_id */
    uint32_t grid_x, grid_y, grid_z; /* logical grid; grid_size = product */
    uint32_t block_threads;  /* <= 256 */
    const void* args;        /* host pointer to the body's POD argument struct (copied) */
    uint32_t args_size;      /* <= 512 */
    int phase;               /* ds_phase */
    int64_t request;         /* request id for metrics, -1 if none */
    int decode_index;        /* 0-based decode step within a request, -1 otherwise */
} ds_kernel_desc;

typedef struct ds_completion {
    int32_t tenant;
    int32_t kernel;          /* registered kernel id */
    uint64_t seq;            /* per-tenant launch sequence number (program order) */
    uint64_t launch_tag;     /* caller tag passed to ds_launch */
    uint32_t grid;           /* executed grid size */
    uint32_t sms_used;       /* distinct SMs that ran >= 1 block */
    uint64_t t_first_claim;  /* %globaltimer ns */
    uint64_t t_end;          /* %globaltimer ns (last block retired) */
} ds_completion;

typedef struct ds_block_record {
    int32_t tenant;
    uint32_t seq;
    uint32_t block;
    uint16_t smid;
    uint16_t flags;
    uint64_t t_start;
    uint64_t t_end;
} ds_block_record;

typedef struct ds_switch_record { /* an SM changing tenant at a block boundary */
    uint16_t smid;
    int16_t from_tenant;      /* -1 = idle */
    int16_t to_tenant;        /* -1 = idle */
    uint16_t pad;
    uint32_t ctl_gen;         /* control generation in force */
    uint64_t t;               /* %globaltimer ns */
} ds_switch_record;

typedef struct ds_ctl_record { /* control-word change observed on the device */
    uint32_t ctl_gen;
    uint32_t source;          /* 0 host mailbox, 1 claim trigger, 2 time trigger */
    uint64_t t;
} ds_ctl_record;

typedef struct ds_stats {
    uint64_t launches_enqueued;
    uint64_t launches_completed;
    uint64_t blocks_executed;
    uint64_t ctl_changes;
    uint64_t switches;
    uint64_t block_log_entries;
    uint64_t block_log_dropped;
    uint32_t num_sms;
    uint32_t running;
} ds_stats;

/* ---- errors ---- */
const char* ds_status_name(int status);
const char* ds_last_error(void); /* thread-local detail for the last failing call */
int ds_abi_version(void);

/* ---- domain / pool ---- */
int ds_domain_create(const ds_domain_config* cfg, ds_domain** out);
int ds_domain_destroy(ds_domain* dom);
int ds_num_sms(ds_domain* dom, int* out);
int ds_smids(ds_domain* dom, int* out, int cap, int* n); /* physical %smid of each worker slot */
int ds_pctx_count(ds_domain* dom, int* out);
int ds_pctx_info(ds_domain* dom, int pctx, int64_t* tier_num, int64_t* tier_den, int* n_sms, int* bound_tenant);

/* ---- registration (immutable records) ---- */
int ds_tenant_register(ds_domain* dom, const ds_tenant_desc* desc, int* tenant_id);
int ds_kernel_register(ds_domain* dom, const ds_kernel_desc* desc, int* kernel_id);

/* ---- executor lifecycle ---- */
int ds_start(ds_domain* dom);
int ds_stop(ds_domain* dom);
/* Run-to-drain mode (set before ds_start): the executor exits on its own once
 * every launch enqueued so far has completed (launches, control words and
 * claim triggers may all be issued before ds_start), and in any case after
 * deadline_ms (0 = no deadline).  For hosts that cannot talk to a resident
 * kernel, e.g. under a profiler that serialises kernel launches. */
int ds_set_drain_exit(ds_domain* dom, int enable, uint64_t deadline_ms);

/* ---- launches (program order per tenant; "kernel resumes, never restarts") ---- */
int ds_launch(ds_domain* dom, int tenant, int kernel_id, uint64_t tag, uint64_t* seq);
/* negative-control mutant (engine.hpp:68-71): executed grid = max(1, floor(grid * tier)) */
int ds_launch_atomized(ds_domain* dom, int tenant, int kernel_id, uint64_t tag, int64_t tier_num,
                       int64_t tier_den, uint64_t* seq);
/* A launch whose logical blocks [0, first_block) already ran elsewhere (on the
 * device a tenant migrated from, into memory copied here with its working
 * set): the executor hands out blocks first_block .. grid-1 only, in the same
 * order, so the launch completes exactly as one uninterrupted run would
 * (begin_migration / on_migration_done, engine.cpp:620-672,986-1009:
 * "kernel resumes, never restarts").  first_block < grid. */
int ds_launch_from(ds_domain* dom, int tenant, int kernel_id, uint64_t tag, uint32_t first_block, uint64_t* seq);
/* Where a tenant stands on the device (read from HBM while the executor runs). */
typedef struct ds_progress {
    uint64_t head;          /* launches completed */
    uint64_t tail;          /* launches the device has seen */
    uint64_t enqueued;      /* launches enqueued by the host */
    uint64_t claim_seq;     /* launch the claim word is on */
    uint32_t claim_open;    /* 1: claim_seq is open for claims */
    uint32_t claim_block;   /* next logical block it hands out (open only) */
    uint32_t claim_grid;
    uint32_t claim_retired; /* blocks of claim_seq retired (those before its first block included) */
    uint32_t drained;       /* no block of the tenant is running: head == claim_seq and every
                               claimed block of it retired */
    uint32_t failed;
} ds_progress;
int ds_tenant_progress(ds_domain* dom, int tenant, ds_progress* out);
int ds_wait_tenant(ds_domain* dom, int tenant, uint64_t seq, int timeout_ms); /* until seq completed;
                                                                               DS_TENANT_FAILED once the tenant failed */
/* Local exception (FaultSpec::LocalException, apply_local_exception engine.cpp:1049-1083):
 * the tenant fails alone — no SM claims another of its blocks, blocks already
 * running finish, its pending launches never complete, later ds_launch calls
 * return DS_TENANT_FAILED.  Other tenants are unaffected (bit-exact).
 * code must be nonzero; the first fault of a tenant wins. */
int ds_fault_inject(ds_domain* dom, int tenant, uint32_t code);
typedef struct ds_fault_info {
    uint32_t code;          /* 0 = healthy */
    uint32_t block;         /* logical block that raised it (0xffffffff: injected) */
    uint64_t seq;           /* launch that raised it (injected: the launch open for claims) */
    uint64_t first_failed;  /* launches >= this never count as completed (the tenant's head
                               when it faulted: earlier launches had finished intact) */
    uint64_t t_ns;          /* %globaltimer */
} ds_fault_info;
int ds_tenant_fault(ds_domain* dom, int tenant, ds_fault_info* out);
int ds_poll(ds_domain* dom, ds_completion* out, int cap, int* n);

/* ---- arbiter: pctx binding and raw SM quota ---- */
int ds_bind(ds_domain* dom, int tenant, int pctx);
int ds_unbind(ds_domain* dom, int tenant);
int ds_migrate(ds_domain* dom, int tenant, int dst_pctx);
int ds_preempt(ds_domain* dom, int pctx); /* revoke at the next logical-block boundary */
int ds_bound_pctx(ds_domain* dom, int tenant, int* pctx);
/* raw control word: SM slot i (0..num_sms-1) runs owner[i] first, then lender[i]
 * when the owner has no claimable block; -1 = none */
int ds_quota_set(ds_domain* dom, const int32_t* owner, const int32_t* lender, int n);
int ds_quota_get(ds_domain* dom, int32_t* owner, int32_t* lender, int n);
/* Sub-block yields: blocks of an abandonable body launched by this tenant
 * (DS_BODY_GEMM_BF16 with GemmArgs.abandon != 0) give their logical block up
 * within ~2 k-blocks when the SM is revoked.  abandon = 1: the next claimer
 * re-runs the tile from scratch; abandon = 2: the fp32 accumulators are
 * spilled and the next claimer resumes at the same k-block.  Either way the
 * MMA sequence is unchanged, so results are bit-identical; only a completed
 * run retires the block.  Call before ds_start. */
int ds_tenant_abandonable(ds_domain* dom, int tenant, int enable);
/* Lane split: every SM owned by a tenant also runs the lend tenant on its
 * second worker lane (mode 1: lane 0 runs the owner, then the lend tenant when
 * the owner has nothing; mode 2: lane 0 runs the owner only).  A memory-bound
 * owner (decode) and a compute-bound lender (training GEMM) then share each SM
 * instead of splitting the SM set.  Modes 3, 4: as 1, 2 on every other owned
 * SM only (the rest keep both lanes for the owner).  0 = off (default). */
int ds_set_lane_split(ds_domain* dom, int mode);
int ds_set_lend(ds_domain* dom, int lend_tenant); /* tenant allowed on idle SMs (-1 none) */
/* device-side control program: when tenant's launch `seq` has claimed `block`
 * blocks, install owner/lender (n entries).  Used for exact mid-kernel
 * quota changes (config 1) and the migration sweep (config 3). */
int ds_quota_at_claim(ds_domain* dom, int tenant, uint64_t seq, uint32_t block, const int32_t* owner,
                      const int32_t* lender, int n);
/* empty the claim-trigger table (triggers fire in install order) */
int ds_quota_triggers_reset(ds_domain* dom);
/* periodic device-timer flips between two control words (period ns, 0 = off) */
int ds_quota_periodic(ds_domain* dom, uint64_t period_ns, const int32_t* owner_a, const int32_t* lender_a,
                      const int32_t* owner_b, const int32_t* lender_b, int n);

/* ---- observation ---- */
int ds_stats_get(ds_domain* dom, ds_stats* out);
int ds_transcript(ds_domain* dom, int tenant, int32_t* kernel_ids, uint32_t* grids, int cap, int* n);
int ds_logical_progress(ds_domain* dom, int tenant, int64_t* out);
int ds_block_log(ds_domain* dom, ds_block_record* out, int64_t cap, int64_t* n);
int ds_switch_log(ds_domain* dom, ds_switch_record* out, int64_t cap, int64_t* n);
int ds_ctl_log(ds_domain* dom, ds_ctl_record* out, int64_t cap, int64_t* n);
int ds_clear_logs(ds_domain* dom);
int ds_globaltimer(ds_domain* dom, uint64_t* ns); /* device %globaltimer now (probe kernel) */
int ds_debug_dump(ds_domain* dom, char* out, int64_t cap); /* text snapshot of device control state */
/* host write of the control word -> device install acknowledged in host memory, n samples (ns) */
int ds_ctl_roundtrip(ds_domain* dom, int n, uint64_t* out_ns);
/* Measured fp32 FFMA throughput of the device (TFLOP/s; a plain kernel, so
 * call it while no executor is resident): config 1's roofline denominator */
int ds_measure_ffma_peak(int device, double* tflops);

/* Overhead ledger (OverheadLedger, engine.hpp:94-107) measured from device
 * %globaltimer stamps, summed over worker lanes (ns):
 *   ctx_switch: a lane's gap between its last block of one tenant and its first of another
 *   preempt:    a lane leaving a tenant its SM was revoked from: control install -> retire of
 *               the block it was running (the boundary wait; count = lane yields)
 *   migration:  a lane's first block of a tenant after a control change, from the install
 *   demand_fault: always 0 (one address space per GPU; cross-GPU copies: ds_migrate_regions) */
typedef struct ds_ledger {
    uint64_t ctx_switches, ctx_switch_total_ns;
    uint64_t preemptions, preempt_total_ns;
    uint64_t migrations, migration_total_ns;
    uint64_t demand_faults, demand_fault_total_ns;
} ds_ledger;
int ds_ledger_get(ds_domain* dom, ds_ledger* out);

/* Kernel-record immutability (Kernel::fingerprint types.cpp:39-48; checked at
 * finalize, engine.cpp:1379-1383): every registered kernel's fingerprint over
 * its immutable record — semantic id, logical grid, body and argument block —
 * recomputed from the device copy of the argument block the executor reads. */
typedef struct ds_kernel_info {
    uint64_t fingerprint;
    uint64_t args_device;     /* device address of the immutable argument block */
    uint32_t args_size, grid;
    int32_t body, phase;
} ds_kernel_info;
int ds_kernel_info_get(ds_domain* dom, int kernel_id, ds_kernel_info* out);
/* DS_OK if no record changed; DS_RECORD_MUTATED with the first mutated
 * kernel id in *first_bad otherwise (-1 if none) */
int ds_verify_kernels(ds_domain* dom, int* first_bad);

/* ---- solo baseline: the same body as a plain __global__ grid (exclusive_baseline) ---- */
int ds_solo_launch(int device, const ds_kernel_desc* desc, void* stream);
int ds_solo_launch_registered(ds_domain* dom, int kernel_id, void* stream);
/* diagnostics: per-CTA globaltimer stamps of later solo launches on `device`
 * into dev_buf (uint64 [grid][4]: entry, TMEM allocated, body returned,
 * exit); NULL turns them off */
int ds_solo_trace(int device, void* dev_buf);
int ds_body_smem(int body, uint32_t* bytes);

/* ---- body argument helpers ---- */
/* encode a TMA descriptor (CUtensorMap, 128 B) for a row-major bf16 [rows][cols]
 * matrix, SWIZZLE_128B boxes of box_rows x box_cols (box_cols*2 must be 128) */
int ds_tensor_map_bf16_2d(void* out128, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                          uint32_t box_cols);
/* the same over a pitched array: rows x cols valid elements, rows `pitch`
 * elements apart (cols <= pitch); loads past the valid extent read zeros
 * without touching memory, stores past it are dropped */
int ds_tensor_map_bf16_2d_pitched(void* out128, const void* base, uint64_t rows, uint64_t cols, uint64_t pitch,
                                  uint32_t box_rows, uint32_t box_cols);
/* KV-cache rows of 128 bf16 as a 3-D {64 dims, rows, 2 halves} view: one box
 * = box_rows rows as two SWIZZLE_128B half-tiles (dims 0-63, then 64-127).
 * box_rows must equal ds_attn_chunk(). */
int ds_tensor_map_bf16_kv(void* out128, const void* base, uint64_t rows, uint32_t box_rows);
/* KV positions per attention pipeline stage of this build (DS_BODY_ATTN_DECODE) */
int ds_attn_chunk(void);

/* ---- policy engine: the SimEngine dispatch loop over the executor ----
 * (engine.hpp:152-170; Policy hooks policy.hpp:97-126; built-ins
 * policies.hpp:12-75).  Records are the reference's Kernel launch records;
 * each runs as >= 1 registered device kernels in program order. */
typedef struct ds_engine ds_engine;

typedef struct ds_engine_config {
    const char* policy;        /* "slo-aware" | "tpot-first" | "temporal" | "static" */
    int64_t quantum_ns;        /* temporal slice (PolicyConfig.quantum) */
    double alpha;              /* predictor EWMA (PolicyConfig.predictor_alpha) */
    int64_t cold_start_ns;     /* PolicyConfig.cold_start_prediction */
    int release_on_idle;       /* EngineConfig.release_on_idle */
    int fair_handover;         /* temporal: preempt the previous owner at each quantum */
    int lend_tenant;           /* tenant run on unbound SMs (-1: strict, idle SMs stay idle) */
    int n_assignments;         /* static partition map */
    int32_t assign_vctx[64];
    int32_t assign_pctx[64];
    int hang_detection;        /* EngineConfig.hang_detection (engine.hpp:63) */
    double hang_threshold;     /* EngineConfig.hang_threshold (default 3) */
    int capture_log;           /* EngineConfig.capture_log: JSONL event log */
    int64_t reset_delay_ns;    /* EngineConfig.reset_delay: pctx downtime after a local exception (0: 200 us) */
} ds_engine_config;

typedef struct ds_record_desc {
    const char* semantic_id;
    int64_t grid_size;         /* signature grid (predictor key) */
    const int32_t* kernels;    /* registered kernel ids, program order */
    int n_kernels;
    int phase;                 /* ds_phase */
    int64_t request;
    int decode_index;
    int64_t arrival_ns;        /* engine clock; 0 = now */
    int64_t request_arrival_ns;
    int64_t ttft_ns, tpot_ns;  /* SLO (0 = none) */
    int64_t base_hint_ns;      /* predictor cold-start hint */
    int64_t sat_num, sat_den;  /* compute saturation in (0, 1] */
} ds_record_desc;

typedef struct ds_record_info {
    uint64_t id;
    int32_t job, state;        /* state: 0 queued, 1 dispatched, 2 done, 3 failed (job hit a local exception) */
    int32_t pctx, preempted;
    int32_t phase, decode_index;
    int64_t request;
    int64_t arrival_host_ns, dispatch_host_ns, finish_host_ns;
    uint64_t t_first_claim, t_end; /* device %globaltimer */
    uint64_t first_seq, last_seq;  /* the tenant launch sequence numbers of its first / last kernel (dispatched) */
} ds_record_info;

typedef struct ds_engine_counters {
    uint64_t decisions, dispatches, completed, preemptions, migrations, unbinds, policy_errors;
    uint64_t failed_jobs;      /* local exceptions (VctxStatus::Failed) */
} ds_engine_counters;

const char* ds_engine_last_error(void);
int ds_engine_create(ds_domain* dom, const ds_engine_config* cfg, ds_engine** out);
int ds_engine_destroy(ds_engine* eng);
int ds_engine_add_job(ds_engine* eng, int tenant, int priority, int* job);
int ds_engine_submit(ds_engine* eng, int job, const ds_record_desc* rec, uint64_t* rec_id);
int ds_engine_start(ds_engine* eng);
int ds_engine_stop(ds_engine* eng);
int ds_engine_now(ds_engine* eng, int64_t* ns);
int ds_engine_wait(ds_engine* eng, uint64_t rec_id, int timeout_ms);
int ds_engine_record(ds_engine* eng, uint64_t rec_id, ds_record_info* out);
int ds_engine_counters_get(ds_engine* eng, ds_engine_counters* out);
int ds_engine_transcript(ds_engine* eng, int job, uint64_t* rec_ids, int cap, int* n);
int ds_engine_predict(ds_engine* eng, const char* semantic_id, int64_t grid, int64_t* ns);
int ds_policy_names(char* out, int cap);
/* JSONL event log {"t","seq","kind",...} (engine.cpp:316-329); *len = full length */
int ds_engine_event_log(ds_engine* eng, char* out, int64_t cap, int64_t* len);
/* quarantined vctxs (SimulationReport.quarantines, engine.hpp:136) */
int ds_engine_quarantines(ds_engine* eng, int32_t* jobs, int64_t* t_ns, int cap, int* n);
/* FaultSpec{LocalException, pctx} at engine time now: the job bound to pctx
 * fails (status Failed, pending records dropped, unbound), the pctx is held
 * unavailable for reset_delay; no effect on an unbound pctx (logged).
 * Device-raised faults (ds_tenant_fault) take the same path automatically. */
int ds_engine_fault_local(ds_engine* eng, int pctx);
/* SimulationReport.vctx_status: 0 Active, 1 Failed, 2 Stranded (types.hpp:77) */
int ds_engine_job_status(ds_engine* eng, int job, int* status);
/* OverheadLedger of the run: the domain's device-measured ledger since ds_engine_start */
int ds_engine_ledger(ds_engine* eng, ds_ledger* out);
/* SimulationReport.kernel_fingerprints: xor of the job's launch-record
 * fingerprints at submit; ds_engine_stop re-checks them and every device
 * kernel record (ds_verify_kernels) and returns DS_RECORD_MUTATED on change */
int ds_engine_job_fingerprint(ds_engine* eng, int job, uint64_t* fp);


/* ---- user policies over the C ABI (Policy, policy.hpp:97-126) ----
 * A policy is a POD vtable of pure, synchronous hooks over a read-only
 * snapshot (PolicyView, policy.hpp:24-69).  The engine validates every
 * returned decision exactly as the reference's apply_decision
 * (engine.cpp:688-754): an illegal one becomes Defer and policy_errors++. */
#define DS_VIEW_MAX_PCTX 64
#define DS_VIEW_MAX_VCTX 64
#define DS_VIEW_MAX_DEVICES 8

typedef struct ds_view_pctx {          /* PolicyView::PctxEntry */
    int32_t id, device;
    int64_t tier_num, tier_den;
    int32_t standby, available;
    int32_t bound;                     /* vctx id, -1 = unbound */
    int32_t has_running;
    uint64_t running_kernel;           /* record id */
    const char* running_semantic_id;   /* valid during the callback */
    int64_t running_grid;
    int64_t running_remaining_ns;      /* predicted remaining wall time */
    int32_t running_phase, running_priority;
} ds_view_pctx;

typedef struct ds_view_vctx {          /* PolicyView::VctxEntry */
    int32_t id, priority, quarantined, bound;
    int64_t pending;
    int32_t head_phase, decoding;
} ds_view_vctx;

typedef struct ds_view {               /* PolicyView */
    int64_t now_ns;
    int32_t n_pctx, n_vctx;
    ds_view_pctx pctx[DS_VIEW_MAX_PCTX];   /* pool order across devices */
    ds_view_vctx vctx[DS_VIEW_MAX_VCTX];
    int32_t n_devices, pad;
    int64_t bound_tier_sum_num[DS_VIEW_MAX_DEVICES], bound_tier_sum_den[DS_VIEW_MAX_DEVICES];
    int64_t min_tier_num[DS_VIEW_MAX_DEVICES], min_tier_den[DS_VIEW_MAX_DEVICES];
    int64_t active_vctx_count;
    const void* predictor;             /* for ds_predictor_predict; valid during the callback */
} ds_view;

typedef struct ds_launch_ctx {         /* LaunchContext (policy.hpp:71-78) + its Kernel record */
    int32_t vctx;
    int32_t has_kernel;
    uint64_t kernel_id;                /* record id */
    const char* semantic_id;           /* valid during the callback */
    int64_t grid_size, base_hint_ns;
    int64_t sat_num, sat_den;
    int32_t phase, decode_index;
    int64_t request, arrival_ns, request_arrival_ns;
    int32_t has_slo, pool_exhausted;
    int64_t ttft_ns, tpot_ns;
} ds_launch_ctx;

typedef enum ds_decision_kind {        /* PolicyDecision::Kind */
    DS_DISPATCH_DIRECT = 0, DS_DISPATCH_REMAP = 1, DS_DISPATCH_DEFER = 2, DS_PREEMPT = 3, DS_NO_ACTION = 4
} ds_decision_kind;
typedef struct ds_decision { int32_t kind; int32_t target; } ds_decision;

/* Hooks write their decision to *out (plain C calling convention: no
 * struct returns, so any FFI can implement them); *out arrives as the
 * hook's default (defer / no action).  An out-of-range kind is an illegal
 * decision (Defer + policy_errors). */
typedef struct ds_policy_vtable {
    const char* name;
    void (*on_launch)(void* user, const ds_view* view, const ds_launch_ctx* launch, ds_decision* out);  /* required */
    void (*on_completion)(void* user, const ds_view* view, const ds_launch_ctx* next, ds_decision* out); /* NULL: no action */
    void (*on_congestion)(void* user, const ds_view* view, const ds_launch_ctx* launch, ds_decision* out); /* NULL: defer */
    int (*launch_order_key)(void* user, const ds_launch_ctx* launch);                              /* NULL: 0 */
    int (*next_review_time)(void* user, const ds_view* view, int64_t* t_ns);                       /* NULL or 0: none */
    void (*destroy)(void* user);                                                                   /* NULL: none */
} ds_policy_vtable;

/* SimEngine(Scenario, std::unique_ptr<Policy>) (engine.hpp:155): the engine
 * owns `user` and calls vt->destroy(user) from ds_engine_destroy. */
int ds_engine_create_with_policy(ds_domain* dom, const ds_engine_config* cfg, const ds_policy_vtable* vt, void* user,
                                 ds_engine** out);
/* the PolicyView the engine would hand a hook right now (ds_snapshot) */
int ds_engine_snapshot(ds_engine* eng, ds_view* out);
/* DurationPredictor::predict (predictor.cpp:20-38) of the view's predictor:
 * EWMA of measured device durations, else the hint (has_hint), else the
 * largest seen for the semantic id, else the cold-start value. */
int ds_predictor_predict(const void* predictor, const char* semantic_id, int64_t grid, int has_hint, int64_t hint_ns,
                         int64_t* out_ns);
/* predict_hol_blocking (policy.hpp:92-95) of pctx in a view */
int ds_predict_hol_blocking(const ds_view* view, int pctx, int64_t* out_ns);
/* the built-in policies' hooks over a C view (make_policy(name)): lets a C
 * user policy delegate, and tests pin the C path to the C++ one */
int ds_builtin_decide(const char* policy, int hook /* 0 launch, 1 completion, 2 congestion, 3 launch_order_key
                                                     (the key in out->target) */, const ds_view* view,
                      const ds_launch_ctx* launch, int64_t quantum_ns, ds_decision* out);

/* ---- request streams and workload expansion ----
 * gen_poisson / gen_burst       proj/src/io/trace.cpp:189-232 (RequestTemplate trace.hpp:41-53)
 * expand_workload               proj/src/io/workload.cpp:51-174
 * Arrival times: arrival_q = round(t * 1e9), t in the trace's time unit
 * (the reference's quantize(), trace.cpp:159-162, as an exact integer). */
typedef enum ds_request_kind { DS_REQ_INFERENCE = 0, DS_REQ_TRAINING = 1 } ds_request_kind;

typedef struct ds_request_template {
    int kind;                              /* ds_request_kind */
    int prompt_tokens, prompt_tokens_max;  /* drawn uniformly in [v, v_max] when v_max > v */
    int output_tokens, output_tokens_max;
    int iterations;                        /* training */
    int streams;                           /* requests round-robin over `streams` job ids */
} ds_request_template;

typedef struct ds_request {
    int64_t arrival_q;  /* round(arrival * 1e9) */
    int32_t stream;     /* job id "<prefix>-<stream>" */
    int32_t kind;
    int32_t prompt_tokens, output_tokens, iterations;
    int32_t pad;
} ds_request;

typedef struct ds_expand_params {
    int64_t tokens_per_grid_unit; /* InferenceProfile (workload.hpp:24): prefill grid = ceil(prompt / this) */
    int64_t decode_grid;          /* InferenceProfile.decode_grid */
    int64_t train_grid;           /* TrainingProfile.grid */
    int32_t default_iterations;   /* TrainingProfile.iterations */
    int32_t pad;
} ds_expand_params;

typedef struct ds_kernel_plan { /* one expanded Kernel record */
    int64_t request;            /* index into the request array */
    int32_t job;                /* vctx index: first appearance of the stream */
    int32_t phase;              /* ds_phase */
    int32_t decode_index;       /* -1 unless decode */
    int32_t pad;
    int64_t grid_size;
    int64_t arrival_q;          /* arrival_floor */
    uint64_t lab_seed;          /* mix_seed(job, position in job) (workload.cpp:10-16) */
} ds_kernel_plan;

/* out may be NULL / cap 0 to size the result: *n is always the full count */
int ds_gen_poisson(double rate, double duration, const ds_request_template* tmpl, uint64_t seed, ds_request* out,
                   int64_t cap, int64_t* n);
int ds_gen_burst(double base_rate, double burst_rate, double burst_duration, double period, double duration,
                 const ds_request_template* tmpl, uint64_t seed, ds_request* out, int64_t cap, int64_t* n);
int ds_expand_workload(const ds_request* reqs, int64_t n_reqs, const ds_expand_params* params, ds_kernel_plan* out,
                       int64_t cap, int64_t* n);

/* ---- peer memory for the data-parallel training tenant's all-reduce body ----
 * (one process per GPU; handles travel over the host process group).
 * Buffers are zero-filled.  handle = 64 opaque bytes (cudaIpcMemHandle_t). */
int ds_ipc_alloc(int device, uint64_t bytes, void** ptr);
int ds_ipc_free(int device, void* ptr);
int ds_ipc_handle(void* ptr, void* handle64);
int ds_ipc_open(int device, const void* handle64, void** ptr);
int ds_ipc_close(int device, void* ptr);
/* release this rank's all-reduce blocks still waiting on peers (shutdown) */
int ds_dp_abort(int device, void* flags);

/* ---- workload-aware placement across GPUs (config 5) ----
 * Replaces first-fit pick_bind_target across devices (policies.cpp:74-94) for
 * whole tenants: balances per-device HBM and tensor load, spreads
 * latency-critical tenants, respects a resident-memory cap.  Deterministic. */
typedef struct ds_tenant_demand {
    int32_t priority;    /* ds_priority */
    int32_t phase;       /* ds_phase of its kernels */
    double hbm_frac;     /* solo HBM bytes/s / device peak */
    double tensor_frac;  /* solo tensor flop/s / device peak */
    double mem_gb;       /* resident footprint */
} ds_tenant_demand;

int ds_place_tenants(const ds_tenant_demand* tenants, int n, int n_devices, double mem_cap_gb, int32_t* device_out);

/* ---- working-set migration across places ----
 * compute_migration_set / full_eager_set (proj/src/runtime/migration.cpp:21-58):
 * eager = touched regions that are dirty or not resident on dst (sorted,
 * unique); lazy = the remaining dirty regions (ascending id).  A touched
 * region outside the working set -> DS_TRACE_VIOLATION.  Output arrays hold
 * up to n_ws ids.  ds_migrate_regions copies regions peer to peer (copy
 * engines over NVLink; no SMs taken from the resident executors). */
/* ---- metrics over measured request outcomes (compute_metrics, metrics.cpp:9-85) ---- */
typedef struct ds_request_outcome {  /* RequestOutcome engine.hpp:117-125 + RequestMeta :50-57; ns */
    int32_t inference, completed;
    int32_t output_tokens, has_slo;
    int64_t arrival_ns, first_decode_finish_ns, last_finish_ns;
    int64_t ttft_slo_ns, tpot_slo_ns;
    int64_t kernels_done;
} ds_request_outcome;

typedef struct ds_dist {  /* DistSummary metrics.hpp:14-20; percentiles exact (TPOT is a ratio) */
    int64_t count;
    double mean;
    int64_t p50_num, p50_den, p90_num, p90_den, p99_num, p99_den;
} ds_dist;

typedef struct ds_metrics {  /* MetricsReport metrics.hpp:22-46 (throughputs per ns) */
    int64_t makespan_ns, kernels_completed, inference_completed, training_kernels_completed;
    double inference_throughput, training_throughput;
    ds_dist ttft, tpot;
    int64_t tpot_excluded, slo_requests, ttft_violations, tpot_violations;
    double ttft_violation_rate, tpot_violation_rate;
} ds_metrics;

/* TTFT = first decode finish - arrival (metrics.cpp:46), TPOT = (last - first
 * decode finish) / (tokens - 1) for >= 2 tokens, nearest-rank percentiles
 * (k = ceil(pct n / 100), metrics.cpp:9-16), SLO violations strictly above the
 * deadline; incomplete or non-inference requests count only toward training. */
int ds_compute_metrics(const ds_request_outcome* reqs, int64_t n, int64_t makespan_ns, int64_t kernels_completed,
                       ds_metrics* out);

/* add_normalization (metrics.cpp:81-102): normalized throughput of job i =
 * exclusive span / shared span of its kernels (first arrival -> last finish;
 * 0 if a span is missing or the shared span is empty), exact num/den, and the
 * aggregate sum.  The exclusive spans come from each job run alone
 * (exclusive_baseline) on the same inputs. */
typedef struct ds_job_span {
    int64_t first_arrival_ns, last_finish_ns;
    int32_t valid, pad;
} ds_job_span;
int ds_add_normalization(const ds_job_span* shared, const ds_job_span* solo, int n, int64_t* num, int64_t* den,
                         double* aggregate);

/* ---- determinism-lab inputs (the reduction tenant's input stream) ----
 * seeded_values (equivalence.cpp:7-17): Rng(seed).uniform(-1, 1) rounded to
 * the format (fmt 0 fp16, 1 bf16, 2 fp32; round_to float_format.cpp:43-67:
 * RNE, subnormals, overflow -> inf, no signed zero); raw bit patterns. */
int ds_seeded_values(uint64_t seed, int64_t n, int fmt, uint32_t* bits);
int ds_round_to(int fmt, double x, uint32_t* bits);

typedef struct ds_region {
    int32_t id;
    int32_t dirty;
    uint64_t bytes;
    uint64_t resident_mask; /* bit p: resident on place p (pctx or GPU, p < 64) */
} ds_region;

int ds_compute_migration_set(const ds_region* ws, int n_ws, const int32_t* touched, int n_touched, int dst,
                             int32_t* eager, int* n_eager, uint64_t* eager_bytes, int32_t* lazy, int* n_lazy,
                             uint64_t* lazy_bytes);
int ds_full_eager_set(const ds_region* ws, int n_ws, int32_t* eager, int* n_eager, uint64_t* eager_bytes);
int ds_migrate_regions(int src_device, int dst_device, const void* const* src_ptrs, void* const* dst_ptrs,
                       const uint64_t* bytes, int n, void* stream);

/* ---- fleet: cross-device moves over per-GPU domains (§8f rows 3-4) ----
 * Global exceptions with emergency migration to a standby device
 * (apply_global_exception / emergency_migrate, engine.cpp:1095-1166), and
 * working-set tracking with eager / lazy copies and demand faults for
 * planned cross-device migrations (begin_migration, advance_lazy,
 * service_demand_faults, engine.cpp:563-672).  A job is one tenant per device
 * it has lived on; its regions are device buffers copied peer to peer on the
 * copy engines; its kernels are re-registered on the destination with their
 * pointer arguments relocated. */
typedef struct ds_fleet ds_fleet;
typedef struct ds_reloc {     /* an 8-byte device pointer inside a kernel's args */
    uint32_t args_offset;
    int32_t region;           /* working-set region it points into */
    uint64_t region_offset;   /* pointer = region base on the running device + region_offset */
} ds_reloc;
typedef struct ds_place_pctx { /* a pctx of a device, as emergency_migrate sees the pools */
    int32_t device, pctx;
    int64_t tier_num, tier_den;
    int32_t bound, pad;
} ds_place_pctx;
typedef struct ds_fleet_job_info {
    int32_t device, tenant, pctx;
    int32_t status;           /* VctxStatus: 0 Active, 1 Failed, 2 Stranded (types.hpp:77) */
    uint64_t launches;
    int32_t migrations;
    int32_t lazy_pending;     /* background region copies still in flight */
} ds_fleet_job_info;
typedef struct ds_migration_info { /* MigrationRecord (migration.hpp:34-45) */
    int32_t job, src_device, src_pctx, dst_device, dst_pctx;
    int32_t emergency, demand_faults, pad;
    uint64_t eager_bytes, lazy_bytes;
    int64_t start_ns, end_ns;  /* host steady clock: start -> the job resumed on dst */
    uint64_t resumed_launch;   /* job launch index it resumed at */
    uint32_t resumed_block, pad2;  /* ... and that launch's first block on dst */
} ds_migration_info;
typedef struct ds_fleet_ledger { /* OverheadLedger migration / fault fields (engine.hpp:94-107), measured */
    uint64_t migrations, emergency_migrations, stranded;
    int64_t migration_total_ns;
    uint64_t demand_faults;
    int64_t demand_fault_total_ns;
    uint64_t eager_bytes, lazy_bytes;
} ds_fleet_ledger;
const char* ds_fleet_last_error(void);
/* emergency_migrate's target rule (engine.cpp:1128-1154) over POD pools: sets
 * *target to an index into pctxs, or -1 (the vctx is stranded) */
int ds_emergency_target(const int32_t* dev_failed, const int32_t* dev_standby, int n_devices,
                        const ds_place_pctx* pctxs, int n_pctxs, int64_t cur_tier_num, int64_t cur_tier_den,
                        int* target);
int ds_fleet_create(ds_fleet** out);
int ds_fleet_destroy(ds_fleet* f);   /* frees the region copies it allocated (stop the domains first) */
int ds_fleet_add_device(ds_fleet* f, ds_domain* dom, int cuda_device, int standby, int* dev);
int ds_fleet_add_job(ds_fleet* f, int dev, const ds_tenant_desc* desc, int* job);
int ds_fleet_add_region(ds_fleet* f, int job, void* ptr, uint64_t bytes, int* region);
int ds_fleet_add_kernel(ds_fleet* f, int job, const ds_kernel_desc* desc, const ds_reloc* relocs, int n_relocs,
                        const int32_t* touched, int n_touched, int* kernel);
int ds_fleet_kernel_id(ds_fleet* f, int job, int kernel, int dev, int* domain_kernel_id); /* -1: not there */
int ds_fleet_bind(ds_fleet* f, int job, int pctx);
int ds_fleet_launch(ds_fleet* f, int job, int kernel, uint64_t* launch); /* program order; demand faults first */
int ds_fleet_wait(ds_fleet* f, int job, uint64_t launch, int timeout_ms);
int ds_fleet_migrate(ds_fleet* f, int job, int dst_dev, int dst_pctx, int timeout_ms);
int ds_fleet_global_exception(ds_fleet* f, int dev, int timeout_ms);
int ds_fleet_job_get(ds_fleet* f, int job, ds_fleet_job_info* out);
int ds_fleet_region(ds_fleet* f, int job, int region, int dev /* -1: the job's */, void** ptr, int* resident,
                    int* dirty);
/* copy the region's up-to-date contents (wherever they live) into host memory */
int ds_fleet_read_region(ds_fleet* f, int job, int region, void* host, uint64_t bytes);
int ds_fleet_migrations(ds_fleet* f, ds_migration_info* out, int cap, int* n);
int ds_fleet_ledger_get(ds_fleet* f, ds_fleet_ledger* out);

#ifdef __cplusplus
}
#endif
#endif /* DETSHARE_DS_H */
