import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2603_15042_b200.tenants import DecodeModel, DecodeConfig
m = DecodeModel(DecodeConfig(layers=2, vocab=2048, L=96, attn_splits=2), seed=5)
for _ in range(int(os.environ.get("REP", "1"))):
    m.solo_step()
torch.cuda.synchronize()
m.solo_step()
torch.cuda.synchronize()
print("ok")
