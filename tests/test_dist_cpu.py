"""The N > 1 host protocol over real processes (torch.distributed gloo, world_size 2 and
4, CPU): every rank computes its own gate counts, the counts are all-gathered, and every
rank then derives the SAME global plan (FssdpState's per-layer decisions, engine.py:457-557,
with re-sharding) and its own device tables — no plan is ever communicated.  The gathered
per-rank tables must agree with each other: identical decisions, SpAG copies naming the
owner's real slot, receive positions tiling every destination's segments, SpRS staging
indices matching between each holder's wgrad push and its owner's reduction."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2502_02581_b200 as F
        from paper_2502_02581_b200.plan_tables import NativeTables

        L, E, T, k, d, f = 2, 16, 512, 2, 256, 512
        topo = F.ClusterTopology.for_nvswitch(world)
        cfg = F.ModelConfig(L, E, 2 * 2 * d * f, 2 * d, 1e-3, 1e-6)
        pol = F.Policy(F.PolicyKind.FSSDP, overlap_override=6, capacity_override=2,
                       reshard_interval=3)
        planner = F.FssdpPlanner(cfg, topo, pol)
        rng = np.random.default_rng(100 + rank)  # this rank's own tokens
        p = 1.0 / np.arange(1, E + 1) ** 1.4
        p = p[np.random.default_rng(7).permutation(E)]
        records = []
        for it in range(8):
            rec = {"it": it}
            for layer in range(L):
                pre = planner.candidate(layer)  # before the gate: history only
                mine = rng.multinomial(T * k, np.roll(p, layer) / p.sum()).astype(np.int32)
                gathered = [torch.zeros(E, dtype=torch.int32) for _ in range(world)]
                dist.all_gather(gathered, torch.from_numpy(mine))
                counts = torch.stack(gathered).numpy()
                dec = planner.plan(layer, counts)
                owner = np.asarray(planner.shards.per_layer[layer].owners(), dtype=np.int32)
                tab = NativeTables(rank, owner, dec.target.mask, dec.route, d, f, pre_mask=pre)
                rec[layer] = dict(
                    owner=owner.tolist(), target=dec.target.mask.tolist(),
                    route=dec.route.tolist(), pre=None if pre is None else pre.tolist(),
                    slot_expert=tab.slot_expert.tolist(), seg_start=tab.seg_start.tolist(),
                    seg_rows=tab.seg_rows.tolist(), recv_base=tab.recv_base.tolist(),
                    spag=tab.spag_copies.tolist(), jobs=tab.sprs_jobs.tolist(),
                    srcs=tab.sprs_srcs.tolist(),
                    wgrad=[g.tolist() for g in tab.groups("wgrad1")[["c_dest", "c_off"]]],
                    n_stage=tab.n_stage)
            planner.finish()
            rec["moves"] = [list(m) for m in planner.last_reshard_moves]
            records.append(rec)
        allrec = [None] * world
        dist.all_gather_object(allrec, records)
        if rank == 0:
            out_q.put(allrec)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_ranks_derive_identical_plans_and_consistent_tables(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    allrec = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    d, f, n1 = 256, 512, 512
    moved = 0
    replicas = 0
    for it in range(len(allrec[0])):
        recs = [allrec[r][it] for r in range(world)]
        moved += len(recs[0]["moves"])
        for r in range(1, world):  # the global decision is identical on every rank
            assert recs[r]["moves"] == recs[0]["moves"]
        for layer in (0, 1):
            lr = [rec[layer] for rec in recs]
            for key in ("owner", "target", "route", "pre"):
                assert all(x[key] == lr[0][key] for x in lr), (it, layer, key)
            owner = np.array(lr[0]["owner"])
            target = np.array(lr[0]["target"], dtype=bool)
            route = np.array(lr[0]["route"])
            replicas += int(target.sum()) - len(owner)
            slot_of = [{e: s for s, e in enumerate(x["slot_expert"])} for x in lr]
            # every rank holds exactly its target column, owned experts first
            for r in range(world):
                assert set(slot_of[r]) == set(np.flatnonzero(target[:, r]).tolist())
                n_own = int((owner == r).sum())
                assert sorted(lr[r]["slot_expert"][:n_own]) == np.flatnonzero(owner == r).tolist()
            # SpAG copies: src is the owner, src_slot holds the expert there
            for r in range(world):
                for src, src_slot, dst_slot in lr[r]["spag"]:
                    e = lr[r]["slot_expert"][dst_slot]
                    assert owner[e] == src and lr[src]["slot_expert"][src_slot] == e
            # receive positions: source s's rows of expert e on d start where d expects
            for dd in range(world):
                for e, s_ in slot_of[dd].items():
                    st = lr[dd]["seg_start"][s_]
                    for s in range(world):
                        assert lr[s]["recv_base"][e][dd] == st + int(route[:s, e, dd].sum())
                    assert lr[dd]["seg_rows"][s_] == int(route[:, e, dd].sum())
            # SpRS: a holder's wgrad pushes into (owner, staging idx); the owner's job reads it
            for h in range(world):
                for j, (c_dest, c_off) in enumerate(lr[h]["wgrad"]):
                    if c_dest == 0:
                        continue
                    o = c_dest - 1
                    idx = c_off // (2 * f * d)
                    srcs = [tuple(x) for x in lr[o]["srcs"]]
                    assert (h, idx) in srcs, (it, layer, h, o, idx)
                    assert idx < lr[o]["n_stage"]
    assert moved > 0, "the skewed per-layer loads should trigger a re-shard"
    assert replicas > 0
