"""Generate tests/golden/planner_goldens.json.gz by running the REAL reference moesim.

Run in the build container only (it imports /root/reference/pkg/src, which does not
exist on the GPU box):

    python tests/golden/make_goldens.py

The committed JSON pins both the CPU oracle (oracle/planner_oracle.py) and the
product's C++ planner to the reference's exact outputs on seeded random corpora,
including the float-order hazards of SURVEY.md §8a (nodes=1 x 8/9/16 devices, ties,
zero loads, fractional estimates).
"""

from __future__ import annotations

import gzip
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

import moesim  # noqa: E402
from moesim import engine as ref_engine  # noqa: E402
from moesim.planner import sparse_materialization  # noqa: E402

OUT = Path(__file__).resolve().parent / "planner_goldens.json.gz"

TOPOS = [(1, 2), (1, 4), (1, 8), (2, 2), (2, 1), (3, 2), (1, 9), (2, 4), (1, 16), (4, 1), (1, 1)]


def topo_of(rng, nodes=None, dpn=None):
    if nodes is None:
        nodes, dpn = TOPOS[int(rng.integers(0, len(TOPOS)))]
    intra = float(rng.choice([100e9, 150e9, 770e9]))
    inter = float(rng.choice([25e9, intra]))
    return moesim.ClusterTopology(nodes, dpn, intra, inter), [nodes, dpn, intra, inter, 10e-6]


def rand_loads(rng, E, D=None):
    kind = int(rng.integers(0, 4))
    shape = (D, E) if D is not None else (E,)
    if kind == 0:
        return rng.integers(0, 50, size=shape).astype(np.float64)
    if kind == 1:
        return rng.random(shape) * 100
    if kind == 2:  # many ties
        return rng.integers(0, 3, size=shape).astype(np.float64)
    return np.round(rng.random(shape) * 7, 1)  # fractional estimates


def rand_partition(rng, E, topo):
    if rng.random() < 0.5:
        return moesim.make_even_partition(E, topo)
    owner = rng.integers(0, topo.num_devices, size=E)
    return moesim.ChunkPlacement.from_pairs(E, topo.num_devices, [(e, int(d)) for e, d in enumerate(owner)])


def pairs(p):
    return [list(x) for x in sorted(p.entries)]


def gen_materialization(rng, n):
    out = []
    for _ in range(n):
        topo, tj = topo_of(rng)
        E = int(rng.integers(1, 65))
        base = rand_partition(rng, E, topo)
        loads = rand_loads(rng, E, topo.num_devices if rng.random() < 0.5 else None)
        t = int(rng.integers(0, E + 3))
        m = int(rng.integers(0, 6))
        plan = sparse_materialization(base, loads, t, m, topo)
        out.append(dict(topo=tj, E=E, base=pairs(base), loads=loads.tolist(), t=t, m=m,
                        target=pairs(plan.target), added=list(plan.added_per_device)))
    return out


def gen_calibrate(rng, n):
    out = []
    for _ in range(n):
        topo, tj = topo_of(rng)
        D = topo.num_devices
        E = int(rng.integers(1, 33))
        base = rand_partition(rng, E, topo)
        est = rand_loads(rng, E, D)
        plan = sparse_materialization(base, est, int(rng.integers(0, E + 1)), int(rng.integers(0, 4)), topo)
        actual = rng.integers(0, 200, size=(D, E)).astype(np.float64)
        if rng.random() < 0.5:
            actual[:, int(rng.integers(0, E))] += 1000
        rem_m = int(rng.integers(-1, 5))
        t_rem = float(rng.choice([0.0, 1e-5, 1e-4, 1e-3, 1.0]))
        cb = int(rng.choice([1000, 10 ** 6, 16 * 2 ** 20]))
        tb = int(rng.choice([8, 512, 2048]))
        ptt = float(rng.choice([1e-3, 1e-6, 12.2e-9]))
        o = moesim.calibrate(plan, actual, rem_m, t_rem, topo, cb, tb, ptt)
        out.append(dict(topo=tj, E=E, source=pairs(plan.source), target=pairs(plan.target),
                        actual=actual.tolist(), rem_m=rem_m, t_rem=t_rem, cb=cb, tb=tb, ptt=ptt,
                        accepted=o.accepted, out_target=pairs(o.plan.target),
                        added=list(o.plan.added_per_device), extra=o.extra_seconds,
                        before=o.estimate_before, after=o.estimate_after))
    return out


def gen_sharding(rng, n):
    out = []
    for _ in range(n):
        topo, tj = topo_of(rng)
        L = int(rng.integers(1, 6))
        E = int(rng.integers(1, 33))
        prof = rand_loads(rng, E, L)
        t = int(rng.integers(0, E + 2))
        plan = moesim.heterogeneous_sharding(moesim.GlobalLoadProfile(prof), t, topo)
        owners = [[plan.per_layer[l].owner(e) for e in range(E)] for l in range(L)]
        out.append(dict(topo=tj, profile=prof.tolist(), t=t, owners=owners,
                        slots=plan.slots_per_device))
    return out


def gen_dispatch(rng, n):
    out = []
    for _ in range(n):
        topo, tj = topo_of(rng)
        D = topo.num_devices
        E = int(rng.integers(1, 33))
        ent = set()
        for e in range(E):
            for d in rng.choice(D, size=int(rng.integers(1, D + 1)), replace=False):
                ent.add((e, int(d)))
        p = moesim.ChunkPlacement.from_pairs(E, D, ent)
        counts = rng.integers(0, 100, size=(D, E))
        if rng.random() < 0.3:
            counts[rng.random((D, E)) < 0.5] = 0
        plan = moesim.build_dispatch(counts, p, topo)
        out.append(dict(topo=tj, E=E, placement=pairs(p), counts=counts.tolist(),
                        route=plan.route.tolist()))
    return out


def gen_traffic(rng, n):
    out = []
    for _ in range(n):
        topo, tj = topo_of(rng)
        D = topo.num_devices
        E = int(rng.integers(1, 33))
        pre = rand_partition(rng, E, topo)
        extra = [(int(rng.integers(0, E)), int(rng.integers(0, D))) for _ in range(int(rng.integers(0, 2 * E + 1)))]
        post = pre.union(extra)
        case = dict(topo=tj, E=E, pre=pairs(pre), post=pairs(post), bytes=int(rng.choice([1, 4096, 16 * 2 ** 20])))
        if rng.random() < 0.15:  # corrupt: drop an owner entry or add a duplicate owner in pre
            bad = sorted(pre.entries)
            if rng.random() < 0.5 and bad:
                bad.pop(int(rng.integers(0, len(bad))))
            else:
                bad.append((int(rng.integers(0, E)), int(rng.integers(0, D))))
            case["pre"] = [list(x) for x in sorted(set(bad))]
            pre = moesim.ChunkPlacement.from_pairs(E, D, bad)
        for kind, fn, a, b in (("spag", moesim.spag_traffic, pre, post), ("sprs", moesim.sprs_traffic, post, pre)):
            try:
                tr, rep = fn(a, b, case["bytes"])
                case[kind] = dict(matrix=tr.data.tolist(), report=[rep.sparsity, rep.total_interdevice_bytes,
                                                                   rep.bottleneck_device, rep.bottleneck_bytes],
                                  latency=moesim.collective_latency(tr, topo))
            except moesim.InvalidPairError as exc:
                case[kind] = dict(error=str(exc))
        out.append(case)
    return out


def gen_estimate(rng, n):
    out = []
    for _ in range(n):
        D, E = int(rng.integers(1, 9)), int(rng.integers(1, 17))
        hist = [rng.integers(0, 1000, size=(D, E)) for _ in range(int(rng.integers(1, 9)))]
        w = int(rng.integers(1, 8))
        out.append(dict(history=[h.tolist() for h in hist], window=w,
                        mean=moesim.estimate_loads(hist, w).tolist()))
    return out


def gen_moe_latency(rng, n):
    out = []
    for _ in range(n):
        topo, tj = topo_of(rng)
        D = topo.num_devices
        E = int(rng.integers(1, 17))
        p = rand_partition(rng, E, topo).union(
            [(int(rng.integers(0, E)), int(rng.integers(0, D))) for _ in range(E)])
        tok = rng.integers(0, 500, size=(D, E))
        tb, ptt = int(rng.choice([8, 2048])), float(rng.choice([1e-6, 12.2e-9]))
        out.append(dict(topo=tj, E=E, placement=pairs(p), tokens=tok.tolist(), tb=tb, ptt=ptt,
                        latency=moesim.estimate_moe_latency(p, tok, topo, tb, ptt)))
    return out


def gen_replays(rng):
    """FssdpState.run_iteration decisions over synthetic traces (engine.py:457-557)."""
    captured = []
    orig = ref_engine.memory_report

    def spy(plan, mats, config, mode="retain"):
        captured.append((plan, mats))
        return orig(plan, mats, config, mode)

    ref_engine.memory_report = spy
    out = []
    try:
        specs = [
            # (layers, E, nodes, dpn, tokens, skew, drift, t, m, calib, remat, reshard, iters, attn, ptt)
            (1, 16, 1, 8, 2048, 0.5, 0.05, 4, 2, True, False, 10, 30, 1e-3, 12.2e-9),
            (1, 8, 1, 4, 1024, 1.0, 0.05, None, None, True, False, 100, 12, 1e-3, 1e-6),
            (4, 8, 1, 8, 4096, 0.5, 0.1, 2, 1, True, True, 5, 25, 2e-3, 255e-9),
            (2, 64, 1, 8, 4096, 0.4, 0.05, 8, 4, True, True, 7, 22, 1e-3, 12.5e-9),
            (3, 16, 2, 2, 512, 0.5, 0.05, 3, 2, False, False, 4, 20, 1e-3, 1e-6),
            (2, 12, 1, 8, 800, 0.3, 0.2, 6, 3, True, False, 3, 16, 1e-3, 5e-8),
        ]
        for (L, E, nodes, dpn, tok, skew, drift, t, m, calib, remat, rint, iters, attn, ptt) in specs:
            topo = moesim.ClusterTopology(nodes, dpn, 150e9, 25e9 if nodes > 1 else 150e9)
            cfg = moesim.ModelConfig(L, E, 16 * 2 ** 20, 2048, attn, ptt)
            pol = moesim.Policy(moesim.PolicyKind.FSSDP, calibration=calib, rematerialize=remat,
                                reshard_interval=rint, overlap_override=t, capacity_override=m)
            meta = moesim.TraceMeta(iters, L, E, nodes * dpn, tok)
            trace = moesim.gen_synthetic_trace(meta, skew=skew, drift=drift, seed=int(rng.integers(0, 1000)))
            state = moesim.make_policy_state(cfg, topo, pol)
            iters_out = []
            for step in trace.steps:
                captured.clear()
                state.run_iteration(step)
                plan, mats = captured[-1]
                layers_out = []
                for l, mat in enumerate(mats):
                    route = moesim.build_dispatch(step[l], mat.target, topo).route
                    layers_out.append(dict(target=pairs(mat.target), route=route.tolist()))
                owners = [[plan.per_layer[l].owner(e) for e in range(E)] for l in range(L)]
                iters_out.append(dict(counts=[s.tolist() for s in step], owners=owners, layers=layers_out))
            out.append(dict(spec=[L, E, nodes, dpn, tok, skew, drift, t, m, calib, remat, rint,
                                  iters, attn, ptt], state_t=state.t, state_m=state.m,
                            iterations=iters_out))
    finally:
        ref_engine.memory_report = orig
    return out


def gen_shard_score(rng, n):
    out = []
    for _ in range(n):
        nodes, dpn = [(1, 8), (1, 9), (1, 16), (2, 8), (1, 7), (1, 130)][int(rng.integers(0, 6))]
        topo = moesim.ClusterTopology(nodes, dpn, 150e9, 150e9)
        D = topo.num_devices
        L, E = int(rng.integers(1, 4)), D * int(rng.integers(1, 3))
        prof = rng.random((L, E)) * rng.choice([1.0, 1e3, 1e-3])
        owners = [list(rng.permutation(np.arange(E) % D)) for _ in range(L)]
        plan = moesim.ShardPlan(tuple(moesim.ChunkPlacement.from_pairs(E, D, list(enumerate(map(int, o))))
                                      for o in owners), (L * E) // D)
        cfg = moesim.ModelConfig(L, E, 1000, 8, 1e-3, 1e-6)
        st = ref_engine.FssdpState(cfg, topo, moesim.Policy(moesim.PolicyKind.FSSDP))
        score = st._shard_score(plan, moesim.GlobalLoadProfile(prof))
        out.append(dict(topo=[nodes, dpn, 150e9, 150e9, 10e-6], owners=[list(map(int, o)) for o in owners],
                        profile=prof.tolist(), score=list(score)))
    return out


def gen_traces(rng, n):
    """traces.py: the reference's own JSONL text of seeded synthetic traces."""
    import tempfile

    out = []
    for _ in range(n):
        meta = moesim.TraceMeta(int(rng.integers(1, 7)), int(rng.integers(1, 4)),
                                int(rng.choice([4, 8, 16, 64])), int(rng.choice([1, 2, 4, 8])),
                                int(rng.choice([1, 7, 128, 1000, 4096])))
        skew = float(rng.choice([0.25, 0.5, 1.0, 2.0]))
        drift = float(rng.choice([0.0, 0.02, 0.05, 0.3]))
        seed = int(rng.integers(0, 10_000))
        path = tempfile.mktemp(suffix=".jsonl")
        moesim.save_trace(moesim.gen_synthetic_trace(meta, skew=skew, drift=drift, seed=seed), path)
        out.append(dict(meta=meta.to_json_obj(), skew=skew, drift=drift, seed=seed,
                        jsonl=open(path).read()))
    return out


def main():
    rng = np.random.default_rng(20250204)
    data = dict(
        materialization=gen_materialization(rng, 400),
        calibrate=gen_calibrate(rng, 250),
        sharding=gen_sharding(rng, 250),
        dispatch=gen_dispatch(rng, 250),
        traffic=gen_traffic(rng, 250),
        estimate=gen_estimate(rng, 60),
        moe_latency=gen_moe_latency(rng, 150),
        shard_score=gen_shard_score(rng, 120),
        replays=gen_replays(rng),
    )
    data["traces"] = gen_traces(rng, 24)
    data["_meta"] = dict(generator="tests/golden/make_goldens.py", reference="/root/reference/pkg/src (moesim 0.1.0)",
                         numpy=np.__version__, seed=20250204)
    text = json.dumps(data, separators=(",", ":"))
    OUT.write_bytes(gzip.compress(text.encode(), compresslevel=9, mtime=0))
    print(OUT, len(text) // 1024, "KiB", hashlib.sha256(text.encode()).hexdigest()[:16])


if __name__ == "__main__":
    main()
