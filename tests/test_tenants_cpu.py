"""Host-side planning of the decode tenant (no GPU needed)."""
from paper_2603_15042_b200.tenants import pick_split


def test_pick_split_wave_efficiency():
    assert pick_split(48, 64, sms=148) == 3   # QKV 6144 rows: 144 blocks on 148 workers
    assert pick_split(1002, 64, sms=148) == 1  # LM head: 1002 slabs, 97% wave efficiency already
    assert pick_split(48, 64) == 6            # 288 blocks on 296 worker lanes
    assert pick_split(32, 224) >= 4      # down proj: 32 slabs need K-split
    for nb, kb in ((48, 64), (32, 64), (224, 64), (32, 224), (1002, 64)):
        s = pick_split(nb, kb)
        assert kb // s >= 4


def test_pack_sw128_is_the_tma_swizzle_image():
    """Weights are pre-packed as the SWIZZLE_128B smem image of [128 x 64]
    tiles: 16-B chunk c of row r sits at chunk c ^ (r % 8)."""
    import torch
    from paper_2603_15042_b200.tenants import pack_sw128
    W = torch.arange(256 * 192, dtype=torch.float32).view(256, 192).to(torch.bfloat16)
    P = pack_sw128(W)
    assert P.shape == (2, 3, 128, 8, 8)
    for slab in range(2):
        for kb in range(3):
            t = P[slab, kb].reshape(128, 64)
            for r in (0, 5, 8, 77, 127):
                for c in range(8):
                    p = c ^ (r % 8)
                    assert torch.equal(t[r, p * 8:(p + 1) * 8], W[slab * 128 + r, kb * 64 + c * 8:kb * 64 + (c + 1) * 8])


def test_resnet_stream_plan_covers_resnet50():
    """Config 4 layer table: 53 convs, 161 GEMMs per iteration (fwd + dgrad +
    wgrad, no input-image dgrad), 4.09 GMAC/image forward at 224^2."""
    from paper_2603_15042_b200.tenants import plan_gemm, resnet50_convs, resnet50_gemms
    assert len(resnet50_convs()) == 53
    g = resnet50_gemms()
    assert len(g) == 161
    fwd = sum(M * N * K for n, M, N, K in g if n.endswith("/fwd"))
    assert abs(fwd / 128 / 1e9 - 4.09) < 0.02
    for _, M, N, K in g:
        Mp, Np, Kp, bn, s = plan_gemm(M, N, K)
        assert Mp % 128 == 0 and Np % bn == 0 and Kp % 64 == 0 and Mp >= M and Np >= N and Kp >= K
        assert 1 <= s <= Kp // 64


def test_resnet_multi_tile_plan():
    """plan_tiles: only un-split, short-K (<= 1152) GEMMs with >= 2 waves of
    tiles get multi-tile blocks (tile narrowed to <= 128 columns, >= 2 blocks
    per worker lane, <= 8 tiles per block)."""
    from paper_2603_15042_b200.tenants import plan_gemm, plan_tiles, resnet50_gemms, WORKERS
    n_multi = 0
    for name, M, N, K in resnet50_gemms():
        Mp, Np, Kp, bn, s = plan_gemm(M, N, K)
        bn2, T = plan_tiles(Mp, Np, Kp, bn, s)
        if T == 1:
            assert bn2 == bn
            continue
        n_multi += 1
        assert s == 1 and Kp <= 1152 and bn2 in (64, 128) and Np % bn2 == 0 and 2 <= T <= 8
        assert -(-(Mp // 128) * (Np // bn2) // T) >= 2 * WORKERS
    assert n_multi > 0
    assert plan_tiles(8192, 8192, 8192, 256, 1) == (256, 1)   # long K: one tile per block
    assert plan_tiles(401408, 64, 64, 64, 1, max_tiles=1) == (64, 1)


def test_resnet_tuned_plan_table_is_valid():
    """resnet_plan.json (scripts/autotune_resnet.py): measured (tile width,
    split-K, tiles per block) per GEMM of the stream; every entry names a GEMM
    of the stream, its tile divides the padded N, every split keeps >= 8
    k-blocks, and multi-tile blocks only where gemm_multi supports them."""
    import json, os
    from paper_2603_15042_b200.tenants import plan_gemm, resnet50_gemms
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "paper_2603_15042_b200", "resnet_plan.json")
    table = json.load(open(path))
    shapes = {}
    for name, M, N, K in resnet50_gemms():
        pad = lambda m, n: ((m + 127) // 128 * 128) * ((n + 63) // 64 * 64)  # noqa: E731
        shapes[name] = (N, M, K) if pad(N, M) < pad(M, N) else (M, N, K)  # ResNetStream's orientation
    assert table
    for name, t in table.items():
        Mp, Np, Kp, bn, s = plan_gemm(*shapes[name])
        assert t["bn"] in (64, 128, 256) and Np % t["bn"] == 0, name
        assert t["splits"] == 1 or (Kp // 64) // t["splits"] >= 8, name
        T = t.get("tiles", 1)
        assert T == 1 or (t["splits"] == 1 and t["bn"] <= 128 and Kp <= 1152), name
