"""Host-side decode plans (CPU): the stream-K GEMV plan mirrors the body's
block -> (slab, k-block) units exactly, and the gate/up row interleave keeps
every SiLU pair in adjacent rows of one slab."""
import pytest
import torch

from paper_2603_15042_b200.tenants import sk_contributors


def body_pieces(t, nb, kb, G):
    """bodies/decode.cuh gemv_body, a.sk = 1: block t's pieces (slab, ka, kb, contributor, n_contributors)."""
    U = nb * kb
    block_of = lambda u: ((u + 1) * G - 1) // U  # noqa: E731
    u0, u1 = t * U // G, (t + 1) * U // G
    out, u = [], u0
    while u < u1:
        n, ka = divmod(u, kb)
        kend = min(kb, ka + (u1 - u))
        first, last = block_of(n * kb), block_of(n * kb + kb - 1)
        out.append((n, ka, kend, t - first, last - first + 1))
        u += kend - ka
    return out


@pytest.mark.parametrize("nb,kb,G", [(48, 64, 296), (32, 64, 148), (224, 64, 296), (32, 224, 296), (96, 64, 444)])
def test_stream_k_plan_covers_every_unit_once_in_k_order(nb, kb, G):
    cmax = sk_contributors(nb, kb, G)
    seen = {}
    for t in range(G):
        ps = body_pieces(t, nb, kb, G)
        assert 1 <= len(ps) <= 2  # the body handles at most two slabs per block
        for n, ka, kend, c, nc in ps:
            assert nc <= cmax and 0 <= c < nc
            seen.setdefault(n, []).append((ka, kend, c, t))
    for n in range(nb):
        runs = sorted(seen[n])
        assert runs[0][0] == 0 and runs[-1][1] == kb
        for (a0, a1, c0, t0), (b0, b1, c1, t1) in zip(runs, runs[1:]):
            assert a1 == b0 and c1 == c0 + 1 and t1 == t0 + 1  # contiguous, contributor = ascending k
        assert runs[-1][2] == len(runs) - 1  # the owner (last contributor) holds the slab's last k-block


def test_stream_k_plan_rejects_runs_longer_than_a_slab():
    with pytest.raises(ValueError):
        sk_contributors(224, 64, 148)


def test_gate_up_interleave_pairs_rows():
    """tenants._gemv (mode SiLU): slabs [64 gate | 64 up] -> rows 2i gate, 2i+1 up of feature i."""
    N, K, bm = 256, 8, 128
    W = torch.arange(N * K, dtype=torch.float32).view(N, K)
    Wil = W.view(N // bm, 2, 64, K).transpose(1, 2).reshape(N, K)
    for slab in range(N // bm):
        for i in range(64):
            assert torch.equal(Wil[slab * bm + 2 * i], W[slab * bm + i])            # gate feature i
            assert torch.equal(Wil[slab * bm + 2 * i + 1], W[slab * bm + 64 + i])   # its up partner
