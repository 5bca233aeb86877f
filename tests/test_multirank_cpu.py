"""N>1 host path on CPU: two gloo ranks gather their per-GPU bench lines and
rank 0 forms the whole-job line (independent sharing domains, weak scaling)."""
import os
import socket

import torch.distributed as dist
import torch.multiprocessing as mp


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
    line = {"value": 10.0 + rank, "train_tflops": 500.0 + rank, "e2e": {"value": 11.0 + rank, "unit": "ms"},
            "ms_per_step": 90.0 + rank, "timeslice": {"p99_tpot_ms": 20.0 - rank, "train_tflops": 600.0},
            "bit_exact_vs_solo": True, "gpu_launches": 100, "n_gpus": 1}
    out = bench.gather_ranks(line, world)
    if rank == 0:
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_aggregation():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out["n_gpus"] == 2
    assert out["value"] == 11.0            # worst P99 over ranks
    assert out["train_tflops"] == 1001.0   # throughput sums
    assert out["e2e"]["value"] == 12.0
    assert out["ms_per_step"] == 91.0      # max over ranks
    assert out["timeslice"]["p99_tpot_ms"] == 20.0
    assert out["gpu_launches"] == 200
