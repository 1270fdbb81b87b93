"""SparseAllGather / SparseReduceScatter entry points and the make_policy_state shim on
the CPU (no kernel launches): the pair contracts raise the reference's InvalidPairError
before any device work, and the per-rank pull schedules the kernels execute move exactly
the reference's spag_traffic / sprs_traffic byte matrices (reference-generated traffic
corpus, tests/golden/make_goldens.py; costmodel.py:87-132)."""

import numpy as np
import pytest

import paper_2502_02581_b200 as F
from paper_2502_02581_b200.sparse import spag_copies, sprs_schedule

from _golden import goldens


def place(E, D, pairs):
    return F.ChunkPlacement.from_pairs(E, D, pairs)


def _schedule_matrix_spag(pre, post, S):
    D = pre.num_devices
    mat = np.zeros((D, D))
    for r in range(D):
        for src, _, _ in spag_copies(pre, post, r):
            mat[src, r] += S
    return mat


def _schedule_matrix_sprs(pre, post, S):
    D = pre.num_devices
    mat = np.zeros((D, D))
    for r in range(D):
        jobs, srcs = sprs_schedule(pre, post, r)
        for _, b, n in jobs:
            for h, _ in srcs[b:b + n]:
                if h != r:
                    mat[h, r] += S
    return mat


def test_schedules_reproduce_reference_traffic_corpus():
    n_valid = n_invalid = 0
    for c in goldens()["traffic"]:
        D = int(c["topo"][0]) * int(c["topo"][1])
        pre, post = place(c["E"], D, c["pre"]), place(c["E"], D, c["post"])
        S = c["bytes"]
        # SpAG(pre -> post); SpRS(post -> pre): the corpus' post is the materialized side
        for kind, a, b, fn, mk in (("spag", pre, post, F.sparse_all_gather, _schedule_matrix_spag),
                                   ("sprs", post, pre, F.sparse_reduce_scatter,
                                    _schedule_matrix_sprs)):
            exp = c[kind]
            if "error" in exp:
                # the contract is checked before the buffer is touched (None here)
                with pytest.raises(F.InvalidPairError) as ei:
                    fn(a, b, None)
                assert str(ei.value) == exp["error"]
                n_invalid += 1
            else:
                assert mk(a, b, S).tolist() == exp["matrix"], (kind, c)
                n_valid += 1
    assert n_valid > 100 and n_invalid > 50


def test_slot_convention_prefix():
    """Partition chunks first (ascending), then the extra chunks: SpAG's pre slots are a
    prefix of its post slots, SpRS's post (owned) slots a prefix of its pre slots."""
    topo = F.ClusterTopology.for_nvswitch(4)
    base = F.make_even_partition(10, topo)
    post = base.union([(0, 3), (9, 0), (4, 1), (5, 0)])
    for d in range(4):
        m = F.chunk_slots(base, post, d)
        own = sorted(base.chunks_on(d))
        assert [m[e] for e in own] == list(range(len(own)))
        extra = sorted(set(post.chunks_on(d)) - set(own))
        assert [m[e] for e in extra] == list(range(len(own), len(own) + len(extra)))
    # rank 0 receives chunks 5 and 9 from their owners' slot positions
    cp = spag_copies(base, post, 0)
    assert cp.tolist() == [[base.owner(5), F.chunk_slots(base, post, base.owner(5))[5], 3],
                           [base.owner(9), F.chunk_slots(base, post, base.owner(9))[9], 4]]
    jobs, srcs = sprs_schedule(post, base, 0)  # owner 0 reduces chunk 0 from ranks 0 and 3
    assert jobs.tolist() == [[0, 0, 2]] and srcs.tolist() == [[0, 0], [3, 2]]  # 3 owns 8, 9


def test_make_policy_state_is_the_fssdp_state():
    """make_policy_state(...).run_iteration(step) follows moesim's FssdpState decisions
    (engine.py:457-557; the replay goldens pin them iteration by iteration)."""
    rp = goldens()["replays"][0]
    (L, E, nodes, dpn, tok, skew, drift, t, m, calib, remat, rint, iters, attn, ptt) = rp["spec"]
    tp = F.ClusterTopology(nodes, dpn, 150e9, 25e9 if nodes > 1 else 150e9)
    cfg = F.ModelConfig(L, E, 16 * 2 ** 20, 2048, attn, ptt)
    pol = F.Policy(F.PolicyKind.FSSDP, calibration=calib, rematerialize=remat,
                   reshard_interval=rint, overlap_override=t, capacity_override=m)
    st = F.make_policy_state(cfg, tp, pol)
    assert (st.t, st.m) == (rp["state_t"], rp["state_m"])
    for it in rp["iterations"]:
        decisions = st.run_iteration([np.array(cn) for cn in it["counts"]])
        assert st.shards.owners().tolist() == it["owners"]
        for l, lay in enumerate(it["layers"]):
            assert decisions[l].target.entries == frozenset(map(tuple, lay["target"]))
            assert decisions[l].route.tolist() == lay["route"]
    mem = st.memory(decisions)
    assert mem.param_bytes.sum() == L * E * cfg.expert_bytes
    ep = F.make_policy_state(cfg, tp, F.Policy(F.PolicyKind.EP))
    dec = ep.run_iteration([np.array(cn) for cn in rp["iterations"][0]["counts"]])
    assert all(d.is_identity for d in dec)
    with pytest.raises(F.ConfigError):
        F.make_policy_state(cfg, tp, type("P", (), {"kind": "swap_balance"})())
