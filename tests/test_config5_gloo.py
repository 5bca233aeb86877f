"""Config 5's multi-GPU host path at N = 8 on CPU (gloo, one process per
rank, 127.0.0.1): every rank computes the same workload-aware placement of
the 16-tenant mix and its own share, the DP tenant's IPC handles (gradient,
flags, output) cross the process group into rank-ordered peer tables, the
all-reduce body's chunk plan gives every chunk exactly one reducing rank
with each rank's own shard first in claim order, and rank 0 forms the
whole-job config-5 and bench lines from the eight per-rank results."""
import os
import socket

import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 8


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_2603_15042_b200 import dp
    from paper_2603_15042_b200.placement import config5_mix, place

    def gather(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    mix = config5_mix()
    where = place(mix, world, mem_cap_gb=150.0)
    mine = [t.name for t, d in zip(mix, where) if d == rank]
    # the DP tenant's handle exchange, as dp.DpGroup does it (fake handles:
    # the opener decodes the owning rank)
    hs = gather((bytes([rank, 0]) * 32, bytes([rank, 1]) * 32, bytes([rank, 2]) * 32))
    opener = lambda h: 1000 * (h[1] + 1) + h[0]  # noqa: E731
    grads = dp.peer_table(1000 + rank, rank, [h[0] for h in hs], opener)
    flags = dp.peer_table(2000 + rank, rank, [h[1] for h in hs], opener)
    outs = dp.peer_table(3000 + rank, rank, [h[2] for h in hs], opener)
    n, chunk = 4096 * 4096, 1 << 16
    a = dp.make_args(grads, flags, outs, n, rank, chunk)
    G = dp.grid_for(n, chunk)[0]
    chunks = [dp.block_chunk(rank, j, G, world) for j in range(G)]
    part = {"rank": rank, "tenants": mine, "decode_tokens_per_s": 100.0 * (rank + 1), "train_tflops": 10.0 * rank,
            "tpot_ms": [5.0 + rank, 6.0], "requests": 3, "train_iters": 4 + rank, "dp_iters": 40,
            "engine_counters": {"incomplete_records": 0}}
    line = {"value": 7.0 + 0.1 * rank, "train_tflops": 600.0 + rank, "e2e": {"value": 7.5 + 0.1 * rank, "unit": "ms"},
            "ms_per_step": 80.0 + rank, "timeslice": {"p99_tpot_ms": 9.0 + 0.1 * rank, "train_tflops": 500.0},
            "bit_exact_vs_solo": True, "gpu_launches": 1000, "n_gpus": 1}
    res = gather({"where": where, "mine": mine, "grads": list(a.grad[:world]), "flags": list(a.flags[:world]),
                  "outs": list(a.outs[:world]), "out": a.out, "chunks": chunks, "G": G,
                  "shard": dp.shard_bounds(rank, G, world), "part": part})
    whole = bench.gather_ranks(line, world)
    if rank == 0:
        q.put((res, bench.aggregate_config5([r["part"] for r in res]), whole))
    dist.barrier()
    dist.destroy_process_group()


def test_config5_host_path_eight_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res, c5, whole = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # one placement, agreed by every rank; the shares partition the mix
    assert all(r["where"] == res[0]["where"] for r in res)
    names = sorted(n for r in res for n in r["mine"])
    assert len(names) == 16 and len(set(names)) == 16
    assert set(res[0]["where"]) <= set(range(WORLD))
    # peer tables: rank-ordered, own buffer local, every peer opened
    for rank, r in enumerate(res):
        assert r["grads"] == [1000 + rank if p == rank else 1000 + p for p in range(WORLD)]
        assert r["flags"] == [2000 + rank if p == rank else 2000 + p for p in range(WORLD)]
        assert r["outs"] == [3000 + rank if p == rank else 3000 + p for p in range(WORLD)]
        assert r["out"] == 3000 + rank
    # chunk plan: each rank visits every chunk once, its own shard first; the
    # shards partition the chunks (exactly one reducing rank per chunk)
    G = res[0]["G"]
    owner = [None] * G
    for rank, r in enumerate(res):
        assert sorted(r["chunks"]) == list(range(G))
        lo, hi = r["shard"]
        assert r["chunks"][: hi - lo] == list(range(lo, hi))
        for c in range(lo, hi):
            assert owner[c] is None
            owner[c] = rank
    assert None not in owner
    # whole-job lines
    assert c5["n_gpus"] == WORLD and c5["dp_iters_submitted"] == [40] * WORLD
    assert c5["decode_tokens_per_s"] == sum(100.0 * (r + 1) for r in range(WORLD))
    assert c5["p99_tpot_ms"] == 5.0 + WORLD - 1
    assert whole["n_gpus"] == WORLD and whole["value"] == 7.0 + 0.1 * (WORLD - 1)
    assert whole["train_tflops"] == sum(600.0 + r for r in range(WORLD))
    assert whole["gpu_launches"] == 1000 * WORLD
