import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_15042_b200 import _abi, dp
from paper_2603_15042_b200.runtime import Domain
world, n, chunk = int(os.environ.get("W", "2")), int(os.environ.get("N", "8192")), int(os.environ.get("C", "4096"))
flags = [torch.zeros(dp.FLAG_BYTES, dtype=torch.uint8, device="cuda") for _ in range(world)]
outs = [torch.zeros(n, dtype=torch.bfloat16, device="cuda") for _ in range(world)]
grads = [torch.ones(n, device="cuda", dtype=torch.bfloat16) * (r + 1) for r in range(world)]
dom = Domain(0, block_log_capacity=1 << 12)
dom.start()
ts = [dom.tenant(f"rank{r}", _abi.BEST_EFFORT) for r in range(world)]
per = dom.num_sms // world
dom.quota_set([ts[min(i // per, world - 1)] for i in range(dom.num_sms)])
kids = []
for r in range(world):
    a = dp.make_args([x.data_ptr() for x in grads], [f.data_ptr() for f in flags], outs[r].data_ptr(), n, r, chunk)
    kids.append(dom.kernel("dp", _abi.BODY_ALLREDUCE_P2P, dp.grid_for(n, chunk), a, phase=_abi.TRAINING))
seqs = [dom.launch(ts[r], kids[r]) for r in range(world)]
print("launched", seqs, flush=True)
for r in range(world):
    try:
        dom.wait(ts[r], seqs[r], 5000)
        print("rank", r, "done", flush=True)
    except Exception as e:
        print("rank", r, "timeout", e, flush=True)
print(dom.debug()[:3000], flush=True)
print([b.tenant for b in dom.block_log()], flush=True)
for r in range(world):
    print("outs", outs[r][:4].cpu() if False else "skip")
os._exit(0)
