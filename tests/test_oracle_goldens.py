"""Pin the CPU oracle (oracle/planner_oracle.py) before trusting it.

1. The reference's own hand-written golden tables and known answers (re-expressed
   from /root/reference/pkg/tests; cited per test).
2. Every case of tests/golden/planner_goldens.json.gz, which the real reference produced.
"""

import numpy as np
import pytest

from oracle import planner_oracle as O
from tests._golden import entries, goldens


def topo2x1():
    return O.Topo(2, 1, 100e9, 25e9)


def topo2x2():
    return O.Topo(2, 2, 100e9, 25e9)


BASE4 = [0, 0, 1, 1]  # test_planner.py:34-36 — d0 {0,1}, d1 {2,3}


# ---------------------------------------------------------------- reference golden tables
@pytest.mark.parametrize("t,m,loads,expected", [  # test_planner.py:65-80 (= test_acceptance.py:170-180)
    (0, 3, (5, 1, 3, 1), set()),
    (1, 1, (5, 1, 3, 1), {(0, 1)}),
    (2, 2, (5, 1, 3, 1), {(0, 1), (2, 0)}),
    (2, 1, (5, 1, 3, 1), {(0, 1), (2, 0)}),
    (4, 1, (5, 1, 3, 1), {(0, 1), (2, 0)}),
    (2, 2, (0, 0, 0, 0), {(0, 1), (1, 1)}),
    (3, 1, (1, 2, 3, 4), {(1, 1), (3, 0)}),
    (3, 2, (9, 1, 1, 1), {(0, 1), (1, 1), (2, 0)}),
])
def test_alg1_oracle_table(t, m, loads, expected):
    tgt, _ = O.materialize(BASE4, np.array(loads, float), t, m, topo2x1())
    assert set(tgt - O.owner_entries(BASE4)) == expected


def test_alg1_branch1_everywhere():  # test_planner.py:83-90
    base = O.even_owner(8, 4)
    tgt, _ = O.materialize(base, np.array([9, 1, 1, 1, 8, 1, 1, 2], float), 2, 4, topo2x2())
    h = O.holders_map(tgt, 8)
    assert h[0] == set(range(4)) and h[4] == set(range(4))
    for e in (1, 2, 3, 5, 6, 7):
        assert h[e] == {base[e]}


def test_alg1_proportional_shares():  # test_planner.py:93-101
    base = O.even_owner(8, 4)
    tgt, added = O.materialize(base, np.array([40, 20, 20, 20, 10, 10, 10, 10], float), 4, 2,
                               topo2x2())
    new = tgt - O.owner_entries(base)
    per = {e: sum(1 for c, _ in new if c == e) for e in range(4)}
    assert per == {0: 3, 1: 2, 2: 2, 3: 1} and len(new) == 8 and max(added) <= 2


def test_alg1_node_preference():  # test_planner.py:122-130
    base = O.even_owner(8, 4)
    tgt, _ = O.materialize(base, np.array([5.0, 4.0, 3.0, 0, 0, 0, 0, 0]), 3, 1, topo2x2())
    assert set(tgt - O.owner_entries(base)) == {(0, 1), (0, 2), (1, 3), (2, 0)}


def test_alg2_goldens():  # test_planner.py:214-229
    prof = np.array([[10.0, 10.0, 1.0, 1.0]])
    assert O.shard(prof, 0, topo2x2())[0] == [0, 2, 1, 3]
    assert O.shard(prof, 1, topo2x2())[0] == [1, 0, 2, 3]


def test_dispatch_remainder_golden():  # test_dispatch.py:78-88
    t = O.Topo(1, 3, 100e9, 100e9)
    ent = O.holders_map([], 2)
    p = frozenset([(0, 1), (0, 2), (1, 1), (1, 2)])
    r = O.route_counts(np.array([[5, 1], [0, 0], [0, 0]]), p, 2, t)
    assert r[0, 0, 1] == 3 and r[0, 0, 2] == 2 and r[0, 1, 2] == 1 and r[0, 1, 1] == 0
    del ent


def test_dispatch_routing_goldens():  # test_dispatch.py:34-70, 164-174
    topo = O.Topo(2, 2, 100e9, 25e9)
    base = frozenset((e, e // 2) for e in range(8))
    c = np.zeros((4, 8), int)
    c[1, 2] = 37
    r = O.route_counts(c, base, 8, topo)
    assert r[1, 2, 1] == 37 and r.sum() == 37 and O.a2a_matrix(r, 4096).sum() == 0
    c = np.zeros((4, 8), int)
    c[0, 5] = 10
    assert O.route_counts(c, base | {(5, 1)}, 8, topo)[0, 5, 1] == 10
    c[3, 5] = 4
    r = O.route_counts(c, base, 8, topo)
    m = O.a2a_matrix(r, 4096)
    assert m[0, 2] == 40960 and m[3, 2] == 16384 and r.sum(axis=(0, 1))[2] == 14
    c = np.zeros((4, 8), int)
    c[0, 0] = 10
    p = frozenset([(0, 2), (0, 3)] + [(e, e // 2) for e in range(1, 8)])
    r = O.route_counts(c, p, 8, topo)
    assert r[0, 0, 2] == 5 and r[0, 0, 3] == 5
    with pytest.raises(O.OracleError):
        c = np.zeros((4, 2), int)
        c[1, 1] = 3
        O.route_counts(c, frozenset([(0, 0)]), 2, topo)


MB = 1_000_000


def test_latency_knowns():  # test_costmodel.py:170-192
    t = O.Topo(1, 4, 300e9, 300e9)
    m = np.zeros((4, 4))
    m[1, 0] = m[2, 0] = m[3, 0] = MB
    assert O.latency(m, t) == pytest.approx(20e-6)
    t = O.Topo(2, 2, 300e9, 12.5e9)
    m = np.zeros((4, 4))
    m[2, 0] = m[3, 0] = 1.5 * MB
    assert O.latency(m, t) == pytest.approx(250e-6)
    assert O.latency(np.zeros((4, 4)), O.Topo(2, 2, 100e9, 25e9)) == 0.0
    t = O.Topo(1, 2, 100e9, 100e9, alpha=0.0)
    assert O.latency(np.array([[0.0, MB], [MB, 0.0]]), t) == pytest.approx(MB / 100e9)


def test_overlap_knowns():  # test_costmodel.py:232-247
    t = O.Topo(2, 2, 100e9, 12.5e9)
    assert O.overlap(10e-3, t, 25 * MB) == 5
    assert O.overlap(10e-3, t, 200 * MB) == 0
    assert O.overlap(0.0, t, 25 * MB) == 0
    assert O.overlap(1e-3, O.Topo(2, 2, 10e9, 50e9), MB) == 10
    t = O.Topo(1, 2, 10e9, 10e9)
    assert O.overlap(0.99 * MB / 10e9, t, MB) == 0
    assert O.overlap(1.01 * MB / 10e9, t, MB) == 1


def test_traffic_knowns():  # test_costmodel.py:62-121
    pre = frozenset((e, e // 2) for e in range(8))
    post = pre | {(0, 1), (0, 2), (0, 3)}
    mat, rep = O.spag_matrix(pre, post, 8, 4, 1000)
    assert mat[0, 1] == mat[0, 2] == mat[0, 3] == 1000 and rep[1] == 3000 and rep[0] == 1 / 8
    smat, _ = O.sprs_matrix(post, pre, 8, 4, 1000)
    assert np.array_equal(smat, mat.T)
    assert not O.spag_matrix(pre, pre, 8, 4, 1000)[0].any()
    with pytest.raises(O.OracleError):
        O.spag_matrix(post, post, 8, 4, 1000)


def test_estimate_knowns():  # test_planner.py:47-50
    hist = [np.full((2, 2), v, dtype=float) for v in (10, 20, 40)]
    assert np.array_equal(O.estimate(hist, 2), np.full((2, 2), 30.0))
    assert np.array_equal(O.estimate(hist, 5), np.full((2, 2), 70 / 3))


def test_calibration_knowns():  # test_planner.py:155-188
    t = topo2x2()
    base = O.owner_entries(O.even_owner(8, 4))
    actual = np.zeros((4, 8))
    actual[:, 0] = 100
    ok, tgt, extra, before, after = O.calibrate(base, base, actual, 8, 1.0, t, 8, 1000, 8, 1e-3)
    assert ok and extra > 0 and after + extra < before
    assert O.holders_map(tgt, 8)[0] == set(range(4))
    ok, tgt, extra, *_ = O.calibrate(base, base, np.full((4, 8), 10.0), 8, 1.0, t, 8, 10 ** 9, 8,
                                     1e-3)
    assert not ok and tgt == base and extra == 0.0
    for rm, tr in ((0, 1.0), (8, 0.0)):
        ok, _, _, b, a = O.calibrate(base, base, actual, rm, tr, t, 8, 1000, 8, 1e-3)
        assert not ok and a == b


# ---------------------------------------------------------------- reference-generated corpora
def _topo(tj):
    return O.Topo(*tj)


def test_oracle_materialization_corpus():
    for c in goldens()["materialization"]:
        owner = [d for _, d in sorted(entries(c["base"]))]
        tgt, added = O.materialize(owner, np.array(c["loads"]), c["t"], c["m"], _topo(c["topo"]))
        assert tgt == entries(c["target"]) and added == c["added"]


def test_oracle_calibrate_corpus():
    for c in goldens()["calibrate"]:
        ok, tgt, extra, before, after = O.calibrate(
            entries(c["source"]), entries(c["target"]), np.array(c["actual"]), c["rem_m"],
            c["t_rem"], _topo(c["topo"]), c["E"], c["cb"], c["tb"], c["ptt"])
        assert ok == c["accepted"] and tgt == entries(c["out_target"])
        assert (extra, before, after) == (c["extra"], c["before"], c["after"])  # bit-exact


def test_oracle_sharding_corpus():
    for c in goldens()["sharding"]:
        assert O.shard(np.array(c["profile"]), c["t"], _topo(c["topo"])) == c["owners"]


def test_oracle_dispatch_corpus():
    for c in goldens()["dispatch"]:
        r = O.route_counts(np.array(c["counts"]), entries(c["placement"]), c["E"], _topo(c["topo"]))
        assert r.tolist() == c["route"]


def test_oracle_traffic_corpus():
    for c in goldens()["traffic"]:
        topo = _topo(c["topo"])
        pre, post = entries(c["pre"]), entries(c["post"])
        for kind, fn, a, b in (("spag", O.spag_matrix, pre, post), ("sprs", O.sprs_matrix, post, pre)):
            exp = c[kind]
            if "error" in exp:
                with pytest.raises(O.OracleError) as ei:
                    fn(a, b, c["E"], topo.D, c["bytes"])
                assert str(ei.value).endswith(exp["error"])
            else:
                mat, rep = fn(a, b, c["E"], topo.D, c["bytes"])
                assert mat.tolist() == exp["matrix"] and list(rep) == exp["report"]
                assert O.latency(mat, topo) == exp["latency"]


def test_oracle_estimate_corpus():
    for c in goldens()["estimate"]:
        got = O.estimate([np.array(h) for h in c["history"]], c["window"])
        assert got.tolist() == c["mean"]


def test_oracle_moe_latency_corpus():
    for c in goldens()["moe_latency"]:
        got = O.moe_latency(entries(c["placement"]), np.array(c["tokens"]), c["E"], _topo(c["topo"]),
                            c["tb"], c["ptt"])
        assert got == c["latency"]


def test_oracle_shard_score_corpus():
    for c in goldens()["shard_score"]:
        got = O.shard_score(c["owners"], np.array(c["profile"]), _topo(c["topo"]))
        assert list(got) == c["score"]


def test_oracle_replays():
    for rp in goldens()["replays"]:
        (L, E, nodes, dpn, tok, skew, drift, t, m, calib, remat, rint, iters, attn, ptt) = rp["spec"]
        topo = O.Topo(nodes, dpn, 150e9, 25e9 if nodes > 1 else 150e9)
        knobs = dict(t=rp["state_t"], m=rp["state_m"], calibration=calib, rematerialize=remat,
                     expert_bytes=16 * 2 ** 20, token_bytes=2048, attn_fwd_time=attn, ptt=ptt)
        rep = O.FssdpReplay(L, E, topo, knobs, reshard_interval=rint)
        for it in rp["iterations"]:
            out, _ = rep.step([np.array(cn) for cn in it["counts"]])
            assert rep.owners == it["owners"]
            for l, lay in enumerate(it["layers"]):
                assert out[l]["target"] == entries(lay["target"])
                assert out[l]["route"].tolist() == lay["route"]
