"""One ResNet stream GEMM (default conv1/fwd) as plain-grid solo launches x3,
for ncu (-k regex:ds_solo_kernel -s 2 -c 1).  DS_RESNET_TILES selects the
multi-tile (T <= 4) or one-tile (1) record."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from fractions import Fraction
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import ResNetStream

name = sys.argv[1] if len(sys.argv) > 1 else "resnet/conv1/fwd"
rs = ResNetStream()
dom = Domain(0, tiers=[Fraction(1)], block_log_capacity=0)
kids = rs.register(dom)
k = kids[[r[0] for r in rs.records].index(name)]
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    dom.solo(k, s)
torch.cuda.synchronize()
dom.close()
print("done", name, rs.records[[r[0] for r in rs.records].index(name)][2])
