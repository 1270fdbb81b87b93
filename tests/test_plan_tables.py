"""Host-side plan tables (pure logic, CPU): every rank derives its tables from the same
global plan; the positions sources compute must tile each destination's receive
segments exactly, SpAG/SpRS jobs must follow the placement pair contract."""

import numpy as np

import paper_2502_02581_b200 as F
from oracle import tensor_oracle as TO
from oracle.plan_tables_oracle import build_rank_tables
from paper_2502_02581_b200.plan_tables import ROW_ALIGN


def _random_plan(rng, D, E, T, k):
    topo = F.ClusterTopology.for_nvswitch(D)
    cfg = F.ModelConfig(1, E, 2 ** 20, 512, 1e-3, 1e-6)
    pol = F.Policy(F.PolicyKind.FSSDP, overlap_override=int(rng.integers(1, E + 1)),
                   capacity_override=int(rng.integers(1, 4)))
    pl = F.FssdpPlanner(cfg, topo, pol)
    p = 1.0 / np.arange(1, E + 1) ** 1.2
    p = p[rng.permutation(E)]
    idxs = []
    for _ in range(D):
        idx = np.stack([rng.choice(E, size=k, replace=False, p=p / p.sum()) for _ in range(T)])
        idxs.append(idx.astype(np.int32))
    counts = np.stack([np.bincount(i.reshape(-1), minlength=E) for i in idxs])
    pl.history[0].append(counts * rng.uniform(0.8, 1.2, size=counts.shape))
    return pl.plan(0, counts), idxs


def test_positions_tile_receive_segments_exactly():
    rng = np.random.default_rng(0)
    for _ in range(25):
        D, E, T, k = int(rng.choice([1, 2, 4, 8])), int(rng.choice([8, 16])), 200, 2
        dec, idxs = _random_plan(rng, D, E, T, k)
        owner = dec.base.owners()
        tabs = [build_rank_tables(r, owner, dec.target.mask, dec.route, 256, 512) for r in range(D)]
        filled = [np.zeros(t.recv_rows, dtype=np.int64) for t in tabs]
        for s in range(D):
            dest, pos = TO.slot_positions(idxs[s], dec.route, s, tabs[s].recv_base)
            for (t, j), dd in np.ndenumerate(dest):
                e = idxs[s][t, j]
                assert dec.target.mask[e, dd], "slot routed to a non-holder"
                seg = tabs[dd].slots[e]
                st = tabs[dd].seg_start[seg]
                assert st <= pos[t, j] < st + tabs[dd].seg_rows[seg]
                filled[dd][pos[t, j]] += 1
        for d in range(D):
            t = tabs[d]
            want = np.zeros(t.recv_rows, dtype=np.int64)
            for s_ in range(len(t.seg_start)):
                want[t.seg_start[s_]:t.seg_start[s_] + t.seg_rows[s_]] = 1
            assert np.array_equal(filled[d], want)  # bijection onto the real rows
            assert np.all(t.seg_padded % ROW_ALIGN == 0)
            zr = {(int(a), int(b)) for a, b in t.zero_rows}
            assert zr == {(int(t.seg_start[i] + t.seg_rows[i]), int(t.seg_padded[i] - t.seg_rows[i]))
                          for i in range(len(t.seg_start)) if t.seg_padded[i] > t.seg_rows[i]}


def test_native_tables_equal_python_tables():
    """The C++ twin (product path) builds exactly the tables of oracle/plan_tables_oracle.py."""
    from paper_2502_02581_b200.plan_tables import GEMM_NAMES, NativeTables

    rng = np.random.default_rng(3)
    shapes = [(1024, 4096, 2), (256, 384, 2), (256, 384, 3), (2048, 1408, 3), (4096, 14336, 3)]
    for it in range(40):
        D, E = int(rng.choice([1, 2, 4, 8])), int(rng.choice([8, 16, 64]))
        d, f, nm = shapes[it % len(shapes)]
        dec, _ = _random_plan(rng, D, E, 300, 2)
        owner = dec.base.owners()
        # every other case: a model-level parameter region (owned_base, replica_base)
        lay = None if it % 2 == 0 else (int(rng.integers(0, 40)), int(rng.integers(40, 90)))
        for r in range(D):
            py = build_rank_tables(r, owner, dec.target.mask, dec.route, d, f, n_mats=nm,
                                   slot_layout=lay)
            nt = NativeTables(r, owner, dec.target.mask, dec.route, d, f, n_mats=nm,
                              slot_layout=lay)
            assert nt.slots == py.slots and nt.n_owned == py.n_owned
            assert nt.recv_rows == py.recv_rows
            for name in ("seg_start", "seg_rows", "seg_padded", "route_cum", "recv_base",
                         "zero_rows", "spag_copies", "sprs_jobs", "sprs_srcs", "sprs_pull"):
                assert np.array_equal(np.asarray(getattr(nt, name)),
                                      np.asarray(getattr(py, name))), name
            for name in GEMM_NAMES:
                arr, n_tiles, total = py.groups[name]
                assert nt.gemm[name] == (len(arr), n_tiles, total), name
                assert nt.groups(name).tobytes() == arr.tobytes(), name
            assert nt.wgrad_split == py.wgrad_split and nt.n_stage == py.n_stage


def test_early_spag_tables_compose_with_the_final_plan():
    """The estimate-based candidate (known before the gate) is contained in the final
    placement unless the final one fell back to the bare partition; its early tables put
    every prefetched replica in the slot the final tables use, and early + late SpAG
    copies are exactly the full SpAG schedule (native == python for both)."""
    from paper_2502_02581_b200.plan_tables import NativeTables

    rng = np.random.default_rng(5)
    checked = 0
    for _ in range(60):
        D, E = int(rng.choice([2, 4, 8])), int(rng.choice([8, 16]))
        topo = F.ClusterTopology.for_nvswitch(D)
        cfg = F.ModelConfig(1, E, 2 ** 20, 512, 1e-3, 1e-6)
        pol = F.Policy(F.PolicyKind.FSSDP, overlap_override=int(rng.integers(1, E + 1)),
                       capacity_override=int(rng.integers(1, 4)))
        pl = F.FssdpPlanner(cfg, topo, pol)
        p = 1.0 / np.arange(1, E + 1) ** 1.2
        p = p[rng.permutation(E)]
        hist = rng.multinomial(600, p / p.sum(), size=D)
        pl.history[0].append(hist.astype(np.float64))
        pre = pl.candidate(0)
        counts = rng.multinomial(600, p / p.sum(), size=D)
        dec = pl.plan(0, counts)
        target, base = dec.target.mask.astype(bool), dec.base.mask.astype(bool)
        if pre is None:
            assert not dec.adopted
            continue
        assert dec.adopted
        if np.any(pre.astype(bool) & ~target):
            assert np.array_equal(target, base), "final plan must be a superset or the partition"
            continue
        checked += 1
        owner = dec.base.owners()
        zero = np.zeros((D, E, D), dtype=np.int64)
        for r in range(D):
            early = build_rank_tables(r, owner, pre, zero, 256, 512)
            late = build_rank_tables(r, owner, dec.target.mask, dec.route, 256, 512, pre_mask=pre)
            full = build_rank_tables(r, owner, dec.target.mask, dec.route, 256, 512)
            for e, s in early.slots.items():
                assert late.slots[e] == s
            for py, args in ((early, (pre, zero, None)), (late, (dec.target.mask, dec.route, pre))):
                nt = NativeTables(r, owner, args[0], args[1], 256, 512, pre_mask=args[2])
                assert nt.slots == py.slots
                assert np.array_equal(np.asarray(nt.spag_copies), py.spag_copies)
            def copied(t):
                by_slot = {s: e for e, s in t.slots.items()}
                return [by_slot[int(s)] for _, _, s in t.spag_copies]

            ce, cl = copied(early), copied(late)
            assert not set(ce) & set(cl)
            assert sorted(ce + cl) == sorted(copied(full))
    assert checked > 5


def test_wgrad_shared_prefix_covers_every_sprs_input():
    """The wgrad groups list, first, exactly the slots SpRS reads or writes (experts with
    more than one holder), each launch starting at tile 0; a replica's groups write into
    its owner's staging slot (c_dest = owner + 1), the one the owner's SpRS job reads."""
    rng = np.random.default_rng(9)
    f_, d_ = 512, 256
    for _ in range(30):
        D, E = int(rng.choice([2, 4, 8])), 16
        dec, _ = _random_plan(rng, D, E, 300, 2)
        owner = dec.base.owners()
        tabs = [build_rank_tables(r, owner, dec.target.mask, dec.route, d_, f_) for r in range(D)]
        for r, t in enumerate(tabs):
            n_sh, t1, t2 = t.wgrad_split
            by_slot = {s: e for e, s in t.slots.items()}
            shared = [s for s in range(len(t.slots))
                      if np.count_nonzero(dec.target.mask[by_slot[s]]) > 1]
            rest = [s for s in range(len(t.slots)) if s not in shared]
            order = (sorted(shared, key=lambda s: -int(t.seg_padded[s])) +
                     sorted(rest, key=lambda s: -int(t.seg_padded[s])))
            assert n_sh == len(shared)
            for name, t_sh, extra in (("wgrad1", t1, 0), ("wgrad2", t2, f_ * d_)):
                arr, n_tiles, total = t.groups[name]
                assert len(arr) == len(t.slots)
                for g, s in zip(arr, order):
                    e = by_slot[s]
                    o = int(owner[e])
                    if o == r:
                        assert g["c_dest"] == 0 and g["c_off"] == s * 2 * f_ * d_ + extra
                        continue
                    assert g["c_dest"] == o + 1
                    j, rem = divmod(int(g["c_off"]) - extra, 2 * f_ * d_)
                    assert rem == 0 and 0 <= j < tabs[o].n_stage
                    jobs = {int(js): (b, c) for js, b, c in tabs[o].sprs_jobs}
                    b, c = jobs[tabs[o].slots[e]]
                    assert [int(x) for x in tabs[o].sprs_srcs[b:b + c][:, 1][
                        list(tabs[o].sprs_srcs[b:b + c][:, 0]).index(r)].reshape(-1)] == [j]
                for part in (arr[:n_sh], arr[n_sh:]):  # each launch starts at tile 0
                    if len(part):
                        assert part["tile_start"][0] == 0
                        assert np.all(np.diff(part["tile_start"]) ==
                                      (part["m_tiles"][:-1] * n_tiles))
                assert t_sh == int((arr[:n_sh]["m_tiles"] * n_tiles).sum())
                assert total == int((arr["m_tiles"] * n_tiles).sum())
        # staging slots on every owner are used exactly once
        for o, t in enumerate(tabs):
            got = sorted(int(i) for h, i in t.sprs_srcs if h != o)
            assert got == list(range(t.n_stage))


def test_spag_sprs_jobs_follow_the_pair_contract():
    rng = np.random.default_rng(1)
    for _ in range(25):
        D, E = int(rng.choice([2, 4, 8])), 16
        dec, _ = _random_plan(rng, D, E, 300, 2)
        owner = dec.base.owners()
        tabs = [build_rank_tables(r, owner, dec.target.mask, dec.route, 256, 512) for r in range(D)]
        spag_pairs = set()
        for r, t in enumerate(tabs):
            for src, src_slot, dst_slot in t.spag_copies:
                e = [x for x, s in t.slots.items() if s == dst_slot][0]
                assert owner[e] == src and tabs[src].slots[e] == src_slot
                spag_pairs.add((e, r))
        added = dec.target.entries - dec.base.entries
        assert spag_pairs == set(added)  # SpAG executes exactly spag_traffic's schedule
        tr, rep = F.spag_traffic(dec.base, dec.target, 1)
        assert rep.total_interdevice_bytes == len(spag_pairs)
        for r, t in enumerate(tabs):
            for dst_slot, b, n in t.sprs_jobs:
                e = [x for x, s in t.slots.items() if s == dst_slot][0]
                srcs = t.sprs_srcs[b:b + n]
                assert list(srcs[:, 0]) == sorted(np.flatnonzero(dec.target.mask[e]))
                assert all(sl == dst_slot for h, sl in srcs if h == r)  # own partial in place
            assert all(owner[e] == r for e, s in t.slots.items() if s < t.n_owned)
        # SpRS moves exactly sprs_traffic's schedule: one staging slot per (replica, holder)
        tr, rep = F.sprs_traffic(dec.target, dec.base, 1)
        assert rep.total_interdevice_bytes == sum(t.n_stage for t in tabs)
