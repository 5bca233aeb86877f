"""Emergency migration target rule (fleet, csrc/fleet.cpp) vs the reference.

The reference engine (oracle/_ref, compiled from /root/reference) runs random
scenarios with a global exception on device 0 (static placement of training
jobs on its pctxs, standby devices with random pools): every vctx on the
failed device is moved by emergency_migrate (engine.cpp:1124-1166) to a
standby pctx, or stranded.  Replaying the reference's own sequence of
emergency decisions through ds_emergency_target over the same pools must pick
the same pctx (or strand) every time."""
import json
import random
from fractions import Fraction

import pytest

from paper_2603_15042_b200 import fleet

TIERS = ["0.25", "0.5", "0.75", "1"]


def _scenario(rng):
    n_dev = rng.randint(2, 4)
    devices = []
    for d in range(n_dev):
        pool = [rng.choice(TIERS) for _ in range(rng.randint(1, 4))]
        devices.append({"tiers": pool, "standby": d > 0 and rng.random() < 0.8})
    # feasible static placement of jobs on device 0's pctxs
    assign, total = {}, Fraction(0)
    for p, t in enumerate(devices[0]["tiers"]):
        if total + Fraction(t) <= 1 and rng.random() < 0.9:
            assign[len(assign)] = p
            total += Fraction(t)
    if not assign:
        assign[0] = 0
        devices[0]["tiers"][0] = "0.25"
    profiles, records = {}, []
    for j in assign:
        # distinct iteration costs: the jobs reach their preemption boundaries at distinct times
        profiles[f"p{j}"] = {"iteration_cost": str(3 + 2 * j) + ".0" + str(rng.randint(1, 9)),
                             "weights_bytes": rng.randint(1, 1 << 20), "optimizer_bytes": rng.randint(0, 1 << 16),
                             "activation_bytes": rng.randint(0, 1 << 12)}
        records.append({"arrival_time": "0", "job_id": f"j{j}", "kind": "training", "iterations": 50,
                        "profile": f"p{j}"})
    sc = {"devices": devices, "policy": "static", "policy_params": {"assignments": {str(k): v for k, v in assign.items()}},
          "capture_log": True, "profiles": {"training": profiles}, "workload": {"records": records},
          "faults": [{"kind": "global", "device": 0, "time": str(rng.randint(2, 9))}]}
    return sc, assign


def _replay(sc, assign, rep):
    devices = sc["devices"]
    gid, pools = 0, []  # (device, pctx_local, tier, global id)
    for d, dev in enumerate(devices):
        for p, t in enumerate(dev["tiers"]):
            pools.append([d, p, Fraction(t), gid])
            gid += 1
    # the reference's emergency decisions in call order: emergency migration
    # records (start) and stranded log lines (t)
    events = [(Fraction(m["start"]), m["vctx"], m["dst"]) for m in rep["migrations"] if m["emergency"]]
    for line in rep["event_log"]:
        e = json.loads(line)
        if e["kind"] == "MigrationDone" and e.get("stranded"):
            events.append((Fraction(e["t"]), e["vctx"], -1))
    events.sort(key=lambda x: x[0])
    times = [t for t, _, _ in events]
    if len(set(times)) != len(times):
        return None  # simultaneous boundaries: the call order is not observable from the report
    failed = [d == 0 for d in range(len(devices))]
    standby = [bool(dev.get("standby")) for dev in devices]
    bound = {g: False for *_, g in pools}
    checked = 0
    for _, vctx, dst in events:
        cur = Fraction(devices[0]["tiers"][assign[vctx]])
        idx = fleet.emergency_target(failed, standby, [(d, p, t, bound[g]) for d, p, t, g in pools], cur)
        got = pools[idx][3] if idx >= 0 else -1
        assert got == dst, (vctx, got, dst, sc)
        if dst >= 0:
            bound[dst] = True
            standby[pools[idx][0]] = False  # hosts live work from now on
        checked += 1
    return checked


def test_emergency_target_matches_reference(ref):
    from oracle import loader
    rng = random.Random(7)
    n_events = n_stranded = n_moved = 0
    for _ in range(60):
        sc, assign = _scenario(rng)
        rep = json.loads(loader.ref_simulate(json.dumps(sc)))
        k = _replay(sc, assign, rep)
        if k is None:
            continue
        n_events += k
        n_stranded += sum(1 for v in rep["vctx_status"].values() if v == 2)
        n_moved += sum(1 for m in rep["migrations"] if m["emergency"])
        # full eager set: every region of the job's working set is copied
        for m in rep["migrations"]:
            if m["emergency"]:
                p = sc["profiles"]["training"][f"p{m['vctx']}"]
                assert m["eager_bytes"] == p["weights_bytes"] + p["optimizer_bytes"] + p["activation_bytes"]
                assert m["lazy_bytes"] == 0
    assert n_events >= 60 and n_stranded >= 5 and n_moved >= 20, (n_events, n_stranded, n_moved)


def test_emergency_target_rule_cases():
    F = Fraction
    # smallest adequate tier on the first healthy standby device
    pools = [(0, 0, F(1, 2), True), (1, 0, F(1, 4), False), (1, 1, F(3, 4), False), (1, 2, F(1, 2), False)]
    assert fleet.emergency_target([True, False], [False, True], pools, F(1, 2)) == 3
    # none adequate: the largest smaller one
    pools = [(1, 0, F(1, 4), False), (1, 1, F(1, 2), False)]
    assert fleet.emergency_target([True, False], [False, True], pools, F(3, 4)) == 1
    # feasibility: bound 3/4 leaves room for 1/4 only
    pools = [(1, 0, F(3, 4), True), (1, 1, F(1, 2), False), (1, 2, F(1, 4), False)]
    assert fleet.emergency_target([True, False], [False, True], pools, F(1, 2)) == 2
    # a non-standby or failed device is never a target: stranded
    assert fleet.emergency_target([True, False], [False, False], pools, F(1, 4)) == -1
    assert fleet.emergency_target([True, True], [False, True], pools, F(1, 4)) == -1
    # device order first: device 1 full, device 2 takes it
    pools = [(1, 0, F(1), True), (2, 0, F(1), False)]
    assert fleet.emergency_target([True, False, False], [False, True, True], pools, F(1, 4)) == 1
