"""Product planner (C++ via the C-ABI, Python value types) vs the reference outputs and
the pinned oracle.  Bit-exact: placements, shard maps, routes, and every float64
latency/estimate the decisions compare."""

import json

import numpy as np
import pytest

import paper_2502_02581_b200 as F
from oracle import planner_oracle as O
from tests._golden import entries, goldens


def topo(tj):
    return F.ClusterTopology(*tj)


def place(E, D, pairs):
    return F.ChunkPlacement.from_pairs(E, D, pairs)


# ---------------------------------------------------------------- reference-generated corpora
def test_materialization_corpus():
    for c in goldens()["materialization"]:
        t = topo(c["topo"])
        base = place(c["E"], t.num_devices, c["base"])
        plan = F.sparse_materialization(base, np.array(c["loads"]), c["t"], c["m"], t)
        assert plan.target.entries == entries(c["target"])
        assert list(plan.added_per_device) == c["added"]


def test_calibrate_corpus():
    for c in goldens()["calibrate"]:
        t = topo(c["topo"])
        D = t.num_devices
        src, tgt = place(c["E"], D, c["source"]), place(c["E"], D, c["target"])
        plan = F.MaterializationPlan(src, tgt, tuple(np.array(tgt.counts_per_device()) -
                                                     np.array(src.counts_per_device())))
        o = F.calibrate(plan, np.array(c["actual"]), c["rem_m"], c["t_rem"], t, c["cb"], c["tb"],
                        c["ptt"])
        assert o.accepted == c["accepted"]
        assert o.plan.target.entries == entries(c["out_target"])
        assert list(o.plan.added_per_device) == c["added"]
        assert (o.extra_seconds, o.estimate_before, o.estimate_after) == (
            c["extra"], c["before"], c["after"])


def test_sharding_corpus():
    for c in goldens()["sharding"]:
        plan = F.heterogeneous_sharding(F.GlobalLoadProfile(np.array(c["profile"])), c["t"],
                                        topo(c["topo"]))
        assert plan.owners().tolist() == c["owners"]
        assert plan.slots_per_device == c["slots"]


def test_dispatch_corpus():
    for c in goldens()["dispatch"]:
        t = topo(c["topo"])
        p = place(c["E"], t.num_devices, c["placement"])
        assert F.build_dispatch(np.array(c["counts"]), p, t).route.tolist() == c["route"]


def test_traffic_corpus():
    for c in goldens()["traffic"]:
        t = topo(c["topo"])
        D = t.num_devices
        pre, post = place(c["E"], D, c["pre"]), place(c["E"], D, c["post"])
        for kind, fn, a, b in (("spag", F.spag_traffic, pre, post),
                               ("sprs", F.sprs_traffic, post, pre)):
            exp = c[kind]
            if "error" in exp:
                with pytest.raises(F.InvalidPairError) as ei:
                    fn(a, b, c["bytes"])
                assert str(ei.value) == exp["error"]
            else:
                tr, rep = fn(a, b, c["bytes"])
                assert tr.data.tolist() == exp["matrix"]
                assert [rep.sparsity, rep.total_interdevice_bytes, rep.bottleneck_device,
                        rep.bottleneck_bytes] == exp["report"]
                assert F.collective_latency(tr, t) == exp["latency"]


def test_estimate_corpus():
    for c in goldens()["estimate"]:
        got = F.estimate_loads([np.array(h) for h in c["history"]], c["window"])
        assert got.tolist() == c["mean"]


def test_moe_latency_corpus():
    for c in goldens()["moe_latency"]:
        t = topo(c["topo"])
        p = place(c["E"], t.num_devices, c["placement"])
        assert F.estimate_moe_latency(p, np.array(c["tokens"]), t, c["tb"], c["ptt"]) == c["latency"]


def test_shard_score_corpus_numpy_pairwise_order():
    for c in goldens()["shard_score"]:
        t = topo(c["topo"])
        prof = np.array(c["profile"])
        L, E = prof.shape
        cfg = F.ModelConfig(L, E, 1000, 8, 1e-3, 1e-6)
        pl = F.FssdpPlanner(cfg, t, F.Policy(F.PolicyKind.FSSDP))
        plan = F.ShardPlan.from_owners(np.array(c["owners"]), t.num_devices)
        assert list(pl._shard_score(plan, F.GlobalLoadProfile(prof))) == c["score"]


def test_fssdp_replays_match_reference_engine():
    """FssdpPlanner reproduces FssdpState.run_iteration (engine.py:457-557) iteration by
    iteration: re-shards, materialized targets and build_dispatch routes."""
    for rp in goldens()["replays"]:
        (L, E, nodes, dpn, tok, skew, drift, t, m, calib, remat, rint, iters, attn, ptt) = rp["spec"]
        tp = F.ClusterTopology(nodes, dpn, 150e9, 25e9 if nodes > 1 else 150e9)
        cfg = F.ModelConfig(L, E, 16 * 2 ** 20, 2048, attn, ptt)
        pol = F.Policy(F.PolicyKind.FSSDP, calibration=calib, rematerialize=remat,
                       reshard_interval=rint, overlap_override=t, capacity_override=m)
        pl = F.FssdpPlanner(cfg, tp, pol)
        assert (pl.t, pl.m) == (rp["state_t"], rp["state_m"])
        for it in rp["iterations"]:
            decisions = pl.run_iteration([np.array(cn) for cn in it["counts"]])
            assert pl.shards.owners().tolist() == it["owners"]
            for l, lay in enumerate(it["layers"]):
                assert decisions[l].target.entries == entries(lay["target"])
                assert decisions[l].route.tolist() == lay["route"]


# ---------------------------------------------------------------- product vs oracle, wider sweeps
def _rand_topo(rng):
    nodes, dpn = [(1, 8), (1, 4), (2, 4), (1, 2), (4, 2), (1, 16), (1, 1)][int(rng.integers(0, 7))]
    bw = float(rng.choice([150e9, 770e9]))
    return (nodes, dpn, bw, float(rng.choice([25e9, bw])), 10e-6)


def test_plan_layer_vs_oracle_random():
    rng = np.random.default_rng(11)
    for _ in range(150):
        tj = _rand_topo(rng)
        t, ot = topo(tj), O.Topo(*tj)
        D = t.num_devices
        E = int(rng.choice([8, 16, 64]))
        owner = np.array(O.even_owner(E, D), dtype=np.int32)
        if rng.random() < 0.5:  # a heterogeneous (permuted) but slot-exact ownership
            owner = owner[rng.permutation(E)]
        zipf = 1.0 / np.arange(1, E + 1) ** rng.uniform(0.5, 1.5)
        zipf = zipf[rng.permutation(E)]
        actual = rng.multinomial(int(rng.integers(100, 5000)), zipf / zipf.sum(), size=D)
        est = None if rng.random() < 0.2 else actual * rng.uniform(0.5, 1.5, size=actual.shape)
        knobs = dict(t=int(rng.integers(0, E + 1)), m=int(rng.integers(0, 5)),
                     calibration=bool(rng.random() < 0.8), rematerialize=bool(rng.random() < 0.5),
                     expert_bytes=int(rng.choice([2 ** 20, 16 * 2 ** 20, 336 * 2 ** 20])),
                     token_bytes=int(rng.choice([512, 2048, 8192])),
                     attn_fwd_time=float(rng.choice([1e-4, 1e-3, 5e-3])),
                     ptt=float(rng.choice([12.2e-9, 255e-9, 1e-6])))
        exp = O.plan_layer(owner.tolist(), est, actual, ot, knobs)
        cfg = F.ModelConfig(1, E, knobs["expert_bytes"], knobs["token_bytes"],
                            knobs["attn_fwd_time"], knobs["ptt"])
        pol = F.Policy(F.PolicyKind.FSSDP, calibration=knobs["calibration"],
                       rematerialize=knobs["rematerialize"], overlap_override=knobs["t"],
                       capacity_override=knobs["m"])
        pl = F.FssdpPlanner(cfg, t, pol)
        pl.shards = F.ShardPlan.from_owners(owner[None, :], D)
        if est is not None:
            pl.history[0].append(est)  # window-1 mean of a float matrix == the matrix
        got = pl.plan_layer(0, actual)
        assert got.target.entries == exp["target"]
        assert list(got.added_per_device) == exp["added"]
        assert np.array_equal(got.route, exp["route"])
        assert (got.spag_latency, got.sprs_latency, got.remat_latency, got.calib_time) == (
            exp["spag"], exp["sprs"], exp["remat"], exp["calib"])


def test_large_dispatch_vs_oracle():
    rng = np.random.default_rng(5)
    for _ in range(20):
        tj = _rand_topo(rng)
        t, ot = topo(tj), O.Topo(*tj)
        D, E = t.num_devices, 64
        ent = {(e, int(d)) for e in range(E) for d in rng.choice(D, int(rng.integers(1, D + 1)), False)}
        counts = rng.integers(0, 20000, size=(D, E))
        got = F.build_dispatch(counts, place(E, D, ent), t).route
        assert np.array_equal(got, O.route_counts(counts, frozenset(ent), E, ot))


# ---------------------------------------------------------------- API behaviour (reference tests)
def test_placement_api_and_json_round_trip():  # test_placement.py:151-190
    p = place(4, 2, [(0, 0), (1, 0), (2, 1), (3, 1), (0, 1)])
    assert p.devices_of(0) == {0, 1} and p.chunks_on(1) == {0, 2, 3}
    assert p.replica_counts() == [2, 1, 1, 1] and p.counts_per_device() == [2, 3]
    assert not p.is_partition()
    with pytest.raises(F.InternalError):
        p.owner(0)
    obj = json.loads(json.dumps(p.to_json_obj()))
    assert F.ChunkPlacement.from_json_obj(obj) == p
    assert obj["entries"] == [[0, 0], [0, 1], [1, 0], [2, 1], [3, 1]]
    assert p.union([(0, 0)]) == p and p.issubset(p.union([(1, 1)]))
    with pytest.raises(F.DimensionError):
        place(2, 2, [(2, 0)])
    with pytest.raises(F.DimensionError):
        F.ChunkPlacement.from_json_obj({"num_chunks": 2})


def test_verdicts():  # test_placement.py:71-125
    pre = place(3, 3, [(0, 0), (1, 1), (2, 2)])
    assert F.validate_spag_pair(pre, pre.union([(0, 1)])).ok
    v = F.validate_spag_pair(place(3, 3, [(0, 0), (1, 1)]), pre)
    assert (v.reason, v.chunk, v.device) == ("missing_chunk", 2, None)
    v = F.validate_spag_pair(pre.union([(1, 0), (1, 2)]), pre.union([(1, 0), (1, 2)]))
    assert (v.reason, v.chunk, v.device) == ("duplicate_owner", 1, 1)
    v = F.validate_spag_pair(pre, place(3, 3, [(0, 0), (1, 1)]))
    assert (v.reason, v.chunk, v.device) == ("dropped_entry", 2, 2)
    assert v.describe() == "dropped_entry chunk=2 device=2"
    assert F.validate_sprs_pair(pre.union([(0, 1)]), pre).ok
    with pytest.raises(F.DimensionMismatchError):
        F.validate_spag_pair(pre, place(3, 2, []))


def test_shard_plan_even_and_checks():  # test_placement.py:192-226
    t = F.ClusterTopology(1, 3, 1e9, 1e9)
    plan = F.ShardPlan.even(3, 4, t)
    assert plan.owners().tolist() == O.shard_plan_even_owners(3, 4, 3)
    assert plan.slots_per_device == 4
    with pytest.raises(F.InternalError):
        F.ShardPlan((place(2, 2, [(0, 0), (1, 0)]),), 1)
    with pytest.raises(F.InternalError):
        F.ShardPlan((place(2, 2, [(0, 0), (0, 1), (1, 1)]),), 1)
    with pytest.raises(F.DimensionError):
        F.ShardPlan((), 0)


def test_dispatch_errors():  # test_dispatch.py:177-203
    t = F.ClusterTopology(2, 2, 100e9, 25e9)
    p = place(8, 4, [(e, e // 2) for e in range(8)])
    for bad in (np.zeros((4, 8, 2)), np.zeros((3, 8)), np.full((4, 8), -1), np.full((4, 8), 0.5)):
        with pytest.raises(F.DimensionError):
            F.build_dispatch(bad, p, t)
    c = np.zeros((4, 2), int)
    c[1, 1] = 3
    with pytest.raises(F.OrphanExpertError):
        F.build_dispatch(c, place(2, 4, [(0, 0)]), t)


def test_traffic_matrix_validation_and_latency_dims():  # test_costmodel.py:46-59, 222-228
    with pytest.raises(F.DimensionMismatchError):
        F.TrafficMatrix(np.zeros((2, 3)))
    with pytest.raises(F.DimensionMismatchError):
        F.TrafficMatrix(np.array([[0.0, -1.0], [0.0, 0.0]]))
    with pytest.raises(F.DimensionMismatchError):
        F.TrafficMatrix(np.eye(2))
    with pytest.raises(F.DimensionMismatchError):
        F.collective_latency(F.TrafficMatrix.zeros(3), F.ClusterTopology(2, 2, 1e9, 1e9))


def test_estimate_loads_errors():
    with pytest.raises(F.EmptyHistoryError):
        F.estimate_loads([])
    with pytest.raises(F.EmptyHistoryError):
        F.estimate_loads([np.zeros((2, 2))], window=0)


def test_memory_report_ratios():  # test_engine.py:288-309
    t = F.ClusterTopology(1, 2, 1e9, 1e9)
    cfg = F.ModelConfig(2, 4, 50_000_000, 8, 1e-3, 1e-6)
    plan = F.ShardPlan.even(2, 4, t)
    base = plan.per_layer[0]
    m1 = F.MaterializationPlan(base, base.union([(0, 1)]), (0, 1))
    m2 = F.MaterializationPlan(plan.per_layer[1], plan.per_layer[1].union([(2, 0), (3, 0)]), (2, 0))
    ret = F.memory_report(plan, [m1, m2], cfg, "retain")
    rem = F.memory_report(plan, [m1, m2], cfg, "rematerialize")
    assert ret.materialized_bytes.tolist() == [100e6, 50e6]
    assert rem.materialized_bytes.tolist() == [100e6, 50e6]
    assert ret.param_bytes.tolist() == [200e6, 200e6]
    assert ret.optimizer_total() == 6 * 400e6
    with pytest.raises(F.ConfigError):
        F.memory_report(plan, None, cfg, "bogus")
