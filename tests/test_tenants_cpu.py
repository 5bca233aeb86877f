"""Host-side planning of the decode tenant (no GPU needed)."""
from paper_2603_15042_b200.tenants import pick_split


def test_pick_split_wave_efficiency():
    assert pick_split(48, 64) == 3       # QKV 6144 rows: 144 blocks on 148 SMs
    assert pick_split(1002, 64) == 1     # LM head: 1002 slabs, 97% wave efficiency already
    assert pick_split(32, 224) >= 4      # down proj: 32 slabs need K-split
    for nb, kb in ((48, 64), (32, 64), (224, 64), (32, 224), (1002, 64)):
        s = pick_split(nb, kb)
        assert kb // s >= 4
