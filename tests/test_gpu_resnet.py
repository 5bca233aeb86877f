"""Config 4's ResNet-50 stream with its measured plan (resnet_plan.json):
multi-tile GEMM blocks, tuned tile widths and split-K + fold records give the
same bits as a coroutine under mid-launch quota changes as they do as
plain-grid solo launches, and the stream's GEMMs match an fp32 reference."""
import pytest
import torch

from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain, solo_launch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def stream():
    from paper_2603_15042_b200.tenants import ResNetStream
    return ResNetStream()


def _pick(rs):
    """GEMM records (with their fold) covering each plan kind: multi-tile,
    tuned split-K (+ fold), one-tile unsplit, and one with padded extents
    (conv1: K = 147 of 192)."""
    recs = rs.records
    out, kinds = [], set()
    for i, (sid, body, grid, args, _) in enumerate(recs):
        if body != _abi.BODY_GEMM_BF16:
            continue
        kind = "multi" if args.tiles > 1 else ("split" if args.splits > 1 else "one")
        if sid.startswith("resnet/conv1/") and "conv1" not in kinds:
            kind = "conv1"
        if kind in kinds:
            continue
        kinds.add(kind)
        group = [recs[i]]
        if args.splits > 1 and not args.fuse_fold:
            group.append(recs[i + 1])
            assert recs[i + 1][1] == _abi.BODY_SPLITK_REDUCE
        out.append((kind, group))
    assert {"multi", "split", "one", "conv1"} <= kinds
    return out


def test_resnet_records_coroutine_bit_exact_vs_solo(stream):
    rs = stream
    for kind, group in _pick(rs):
        args0 = group[0][3]
        M, N = args0.M, args0.N
        C = rs.C[: M * N]
        rs.C.zero_()
        for sid, body, grid, args, _ in group:
            solo_launch(0, sid, body, grid, args)
        torch.cuda.synchronize()
        want = C.clone()
        rs.C.zero_()
        with Domain(0, block_log_capacity=0) as dom:
            dom.start()
            t = dom.tenant("train", _abi.BEST_EFFORT)
            dom.quota_set(dom.mask(t, 0, dom.num_sms))
            ks = [dom.kernel(sid, body, grid, args, phase=_abi.TRAINING) for sid, body, grid, args, _ in group]
            g0 = group[0][2][0]
            dom.quota_at_claim(t, 0, g0 // 3, dom.mask(t, 8, 40))
            dom.quota_at_claim(t, 0, 2 * g0 // 3, dom.mask(t, 0, dom.num_sms))
            seqs = [dom.launch(t, k) for k in ks]
            dom.wait(t, seqs[-1])
        torch.cuda.synchronize()
        assert torch.equal(C.view(torch.int16), want.view(torch.int16)), kind
        # fp32 reference on a sample of rows over the true extents (the
        # arenas are [M][K] / [N][K] with K padded; the loads stop at the
        # valid m, n, k and the stores clip at (m, n))
        K = args0.K
        m, n, k = next((gm, gn, gk) for name, gm, gn, gk in rs.gemms if group[0][0] == f"resnet/{name}")
        A = rs.A[: M * K].view(M, K)[:m, :k]
        B = rs.B[: N * K].view(N, K)[:n, :k]
        rows = torch.arange(0, m, max(1, m // 64), device="cuda")
        ref = A[rows].float() @ B.float().t()
        got = want.view(M, N)[rows, :n].float()
        assert bool(((got - ref).abs() <= ref.abs() * 2 ** -7 + 2 ** -4).all()), kind
