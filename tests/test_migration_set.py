"""Working-set migration sets (native csrc/migration.cpp) against the
REFERENCE library (oracle/_ref: compute_migration_set / full_eager_set,
proj/src/runtime/migration.cpp:21-58) on random working sets, plus the
SPEC example (A eager, B lazy, C excluded)."""
import random

import pytest

from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200 import migration_set as ms


def native(regions, touched, dst):
    ws = [ms.Region(i, b, d, set(p)) for i, b, d, p in regions]
    try:
        e, eb, l, lb = ms.compute_migration_set(ws, touched, dst)
    except _abi.DsError as ex:
        assert ex.code == _abi.DsError(6, "").code
        return "error: TraceViolation"
    return " ".join(map(str, e)) + (" " if e else "") + f"| {eb} | " + " ".join(map(str, l)) + (" " if l else "") + f"| {lb}"


def test_spec_example():
    # A touched & dirty -> eager; B untouched & dirty -> lazy; C clean & resident on dst -> excluded
    regions = [(0, 100, True, [0]), (1, 200, True, [0, 1]), (2, 300, False, [1])]
    e, eb, l, lb = ms.compute_migration_set([ms.Region(i, b, d, set(p)) for i, b, d, p in regions], [0, 2], 1)
    assert (e, eb, l, lb) == ([0], 100, [1], 200)


def test_matches_reference_random(ref):
    from oracle import loader
    rnd = random.Random(8)
    for _ in range(300):
        n = rnd.randint(0, 12)
        ids = rnd.sample(range(40), n)
        regions = [(i, rnd.randint(1, 1 << 30), rnd.random() < 0.5, rnd.sample(range(4), rnd.randint(0, 3)))
                   for i in ids]
        touched = [rnd.choice(ids) for _ in range(rnd.randint(0, 6))] if ids else []
        if rnd.random() < 0.1:
            touched.append(99)  # outside the working set
        dst = rnd.randrange(4)
        assert native(regions, touched, dst) == loader.ref_migration_set(regions, touched, dst), (regions, touched, dst)


def test_full_eager_matches_reference(ref):
    from oracle import loader
    rnd = random.Random(9)
    for _ in range(50):
        ids = rnd.sample(range(40), rnd.randint(0, 10))
        regions = [(i, rnd.randint(1, 1 << 20), rnd.random() < 0.5, []) for i in ids]
        e, eb = ms.full_eager_set([ms.Region(i, b, d, set(p)) for i, b, d, p in regions])
        want = loader.ref_migration_set(regions, [], 0, full=True)
        assert " ".join(map(str, e)) + (" " if e else "") + f"| {eb} | | 0" == want


@pytest.mark.gpu
def test_migrate_regions_copies_on_copy_engines():
    import torch
    src = torch.arange(1 << 20, dtype=torch.int32, device="cuda")
    dst = torch.zeros_like(src)
    ms.migrate_regions(0, 0, [(src.data_ptr(), dst.data_ptr(), src.numel() * 4)],
                       torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(src, dst)
