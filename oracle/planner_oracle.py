"""Pure-Python/numpy restatement of the reference moesim planner — TEST INFRASTRUCTURE.

Independent of the product's C++ planner; used as the checker for it and as the CPU
baseline.  Placements are plain Python: a placement is a tuple (C, D, frozenset of
(chunk, device)); a partition may also be given as an owner list.  Each function
cites the reference lines it restates.  PINNED against the reference's golden tables
(tests/test_oracle_goldens.py) and against reference-generated fixtures
(tests/golden/planner_goldens.json via tests/golden/make_goldens.py).
"""

from __future__ import annotations

import math
from collections import deque

import numpy as np

ERR_DIMENSION = "DimensionError"
ERR_INVALID_PAIR = "InvalidPairError"
ERR_ORPHAN = "OrphanExpertError"
ERR_INTERNAL = "InternalError"
ERR_INFEASIBLE = "InfeasibleSlotsError"
ERR_EMPTY_HISTORY = "EmptyHistoryError"


class OracleError(Exception):
    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


# ------------------------------------------------------------------ topology
class Topo:
    """ClusterTopology (topology.py:14-49) — value only."""

    def __init__(self, nodes, dpn, intra_bw, inter_bw, alpha=10e-6):
        self.nodes, self.dpn = int(nodes), int(dpn)
        self.intra, self.inter, self.alpha = float(intra_bw), float(inter_bw), float(alpha)

    @property
    def D(self):
        return self.nodes * self.dpn

    def node(self, d):
        return d // self.dpn

    def members(self, n):
        return list(range(n * self.dpn, (n + 1) * self.dpn))


# ------------------------------------------------------------------ placements
def holders_map(entries, C):
    h = [set() for _ in range(C)]
    for c, d in entries:
        h[c].add(d)
    return h


def even_owner(C, D):
    """make_even_partition (placement.py:155-170)."""
    q, r = divmod(C, D)
    owner = []
    for d in range(D):
        owner += [d] * (q + (1 if d < r else 0))
    return owner


def shard_plan_even_owners(L, E, D):
    """ShardPlan.even (placement.py:260-284): rotating remainder window."""
    q, r = divmod(E, D)
    start, out = 0, []
    for _ in range(L):
        per = [q] * D
        for j in range(r):
            per[(start + j) % D] += 1
        start = (start + r) % D
        row = []
        for d in range(D):
            row += [d] * per[d]
        out.append(row)
    return out


def owner_entries(owner):
    return frozenset((c, d) for c, d in enumerate(owner))


def verdict_partition(entries, C):
    """_check_partition (placement.py:181-190) -> (reason, chunk, device) or None."""
    h = holders_map(entries, C)
    for c in range(C):
        if not h[c]:
            return ("missing_chunk", c, None)
        if len(h[c]) > 1:
            return ("duplicate_owner", c, sorted(h[c])[1])
    return None


def verdict_subset(small, big):
    """_check_subset (placement.py:193-197)."""
    for c, d in sorted(small):
        if (c, d) not in big:
            return ("dropped_entry", c, d)
    return None


def check_spag(pre, post, C):
    return verdict_partition(pre, C) or verdict_subset(pre, post)


def check_sprs(pre, post, C):
    return verdict_partition(post, C) or verdict_subset(post, pre)


def describe(v):
    if v is None:
        return "valid"
    reason, c, d = v
    s = reason
    if c is not None:
        s += f" chunk={c}"
    if d is not None:
        s += f" device={d}"
    return s


# ------------------------------------------------------------------ traffic
def report(mat, touched, C):
    """_report (costmodel.py:75-84)."""
    per = np.maximum(mat.sum(axis=0), mat.sum(axis=1))
    b = int(np.argmax(per))
    return (touched / C if C else 0.0, float(mat.sum()), b, float(per[b]))


def spag_matrix(pre, post, C, D, nbytes):
    """spag_traffic (costmodel.py:87-108): owner -> every added holder."""
    v = check_spag(pre, post, C)
    if v is not None:
        raise OracleError(ERR_INVALID_PAIR, "invalid all-gather pair: " + describe(v))
    hpre, hpost = holders_map(pre, C), holders_map(post, C)
    mat = np.zeros((D, D))
    touched = 0
    for c in range(C):
        (own,) = tuple(hpre[c])
        new = hpost[c] - hpre[c]
        touched += bool(new)
        for d in new:
            mat[own, d] += nbytes
    return mat, report(mat, touched, C)


def sprs_matrix(pre, post, C, D, nbytes):
    """sprs_traffic (costmodel.py:111-132): every non-final replica -> final owner."""
    v = check_sprs(pre, post, C)
    if v is not None:
        raise OracleError(ERR_INVALID_PAIR, "invalid reduce-scatter pair: " + describe(v))
    hpre, hpost = holders_map(pre, C), holders_map(post, C)
    mat = np.zeros((D, D))
    touched = 0
    for c in range(C):
        (fin,) = tuple(hpost[c])
        snd = hpre[c] - {fin}
        touched += bool(snd)
        for s in snd:
            mat[s, fin] += nbytes
    return mat, report(mat, touched, C)


def latency(mat, topo):
    """collective_latency (costmodel.py:149-182)."""
    if not np.any(mat):
        return 0.0
    din, dout = np.zeros(topo.D), np.zeros(topo.D)
    nin, nout = np.zeros(topo.nodes), np.zeros(topo.nodes)
    rs, cs = np.nonzero(mat)
    for s, r in zip(rs.tolist(), cs.tolist()):
        v = mat[s, r]
        if topo.node(s) == topo.node(r):
            dout[s] += v
            din[r] += v
        else:
            nout[topo.node(s)] += v
            nin[topo.node(r)] += v
    dev_t = max(din.max(), dout.max()) / topo.intra
    node_t = max(nin.max(), nout.max()) / topo.inter
    return topo.alpha + max(dev_t, node_t)


def overlap(t_nonmoe, topo, nbytes):
    """overlap_degree (costmodel.py:185-194)."""
    if t_nonmoe <= 0 or nbytes <= 0:
        return 0
    bw = topo.inter if topo.inter < topo.intra else topo.intra
    return int(math.floor(t_nonmoe * bw / nbytes))


# ------------------------------------------------------------------ dispatch
def route_counts(counts, entries, E, topo):
    """build_dispatch (dispatch.py:49-97)."""
    cnt = np.asarray(counts).astype(np.int64)
    D = topo.D
    h = holders_map(entries, E)
    route = np.zeros((D, E, D), dtype=np.int64)
    load = [0] * D
    for s in range(D):
        for e in range(E):
            n = int(cnt[s, e])
            if n == 0:
                continue
            if not h[e]:
                raise OracleError(ERR_ORPHAN, f"expert {e} has tokens but is materialized nowhere")
            if s in h[e]:
                route[s, e, s] += n
                load[s] += n
                continue
            near = sorted(d for d in h[e] if topo.node(d) == topo.node(s))
            dests = near or sorted(h[e])
            q, r = divmod(n, len(dests))
            extra = set(sorted(dests, key=lambda d: (load[d], d))[:r])
            for d in dests:
                k = q + (1 if d in extra else 0)
                route[s, e, d] += k
                load[d] += k
    return route


def a2a_matrix(route, token_bytes):
    """dispatch_traffic (dispatch.py:100-104)."""
    m = route.sum(axis=1).astype(np.float64) * token_bytes
    np.fill_diagonal(m, 0.0)
    return m


def moe_latency(entries, tokens, E, topo, token_bytes, ptt):
    """estimate_moe_latency (planner.py:205-216)."""
    r = route_counts(tokens, entries, E, topo)
    busiest = int(r.sum(axis=(0, 1)).max())
    return busiest * ptt + latency(a2a_matrix(r, token_bytes), topo)


# ------------------------------------------------------------------ Alg. 1
def order_desc(vals):
    """_descending (planner.py:74-76)."""
    return sorted(range(len(vals)), key=lambda i: (-vals[i], i))


def extend(entries, per_expert, t, m, E, topo):
    """_extend_placement (planner.py:79-168); returns the new entry set."""
    D = topo.D
    t = min(t, E)
    m = min(m, t)
    if t <= 0 or m <= 0:
        return frozenset(entries)
    top = order_desc(per_expert)[:t]
    h = holders_map(entries, E)
    if t <= m:
        return frozenset(entries) | {(e, d) for e in top for d in range(D) if d not in h[e]}
    free = [m] * D
    new = set()

    def put(e):
        choice = None
        for n in range(topo.nodes):
            devs = topo.members(n)
            ok = [d for d in devs if free[d] > 0 and d not in h[e]]
            if not ok:
                continue
            key = (any(d in h[e] for d in devs), -sum(free[d] for d in devs), n)
            if choice is None or key < choice[0]:
                choice = (key, min(ok, key=lambda d: (-free[d], d)))
        if choice is None:
            return False
        d = choice[1]
        new.add((e, d))
        h[e].add(d)
        free[d] -= 1
        return True

    slots = D * m
    tot = 0
    for e in top:
        tot = tot + per_expert[e]
    tot = float(tot)
    left = slots
    for e in top:
        share = max(1, math.floor(slots * float(per_expert[e]) / tot)) if tot > 0 else \
            max(1, slots // t)
        want = min(share, D - len(h[e]), left)
        done = 0
        while done < want and put(e):
            done += 1
        left -= done
    moved = True
    while left > 0 and moved:
        moved = False
        for e in top:
            if left == 0:
                break
            if len(h[e]) < D and put(e):
                left -= 1
                moved = True
    return frozenset(entries) | new


def col_sums(a):
    a = np.asarray(a, dtype=np.float64)
    return a.sum(axis=0) if a.ndim == 2 else a


def materialize(owner, loads, t, m, topo):
    """sparse_materialization (planner.py:171-197) -> (target entries, added[D])."""
    E = len(owner)
    base = owner_entries(owner)
    tgt = extend(base, col_sums(loads), t, m, E, topo)
    return tgt, added_counts(base, tgt, topo.D)


def added_counts(src, tgt, D):
    a = [0] * D
    for _, d in tgt:
        a[d] += 1
    for _, d in src:
        a[d] -= 1
    return a


def calibrate(src, tgt, actual, rem_m, t_rem, topo, E, cbytes, tbytes, ptt):
    """calibrate (planner.py:228-276) -> (accepted, target, extra, before, after)."""
    act = np.asarray(actual, dtype=np.float64)
    tokens = act.astype(np.int64)
    before = moe_latency(tgt, tokens, E, topo, tbytes, ptt)
    tc = overlap(t_rem, topo, cbytes)
    if rem_m <= 0 or tc <= 0:
        return False, tgt, 0.0, before, before
    ext = extend(tgt, col_sums(act), tc, rem_m, E, topo)
    if ext == tgt:
        return False, tgt, 0.0, before, before
    d_new = spag_matrix(src, ext, E, topo.D, cbytes)[0]
    d_old = spag_matrix(src, tgt, E, topo.D, cbytes)[0]
    extra = latency(d_new - d_old, topo)
    after = moe_latency(ext, tokens, E, topo, tbytes, ptt)
    if after + extra < before:
        return True, ext, extra, before, after
    return False, tgt, 0.0, before, after


# ------------------------------------------------------------------ Alg. 2
def shard(profile, t, topo):
    """heterogeneous_sharding (planner.py:302-385) -> owners[L][E]."""
    prof = np.asarray(profile, dtype=np.float64)
    L, E = prof.shape
    D = topo.D
    q, r = divmod(L * E, D)
    free = [q + (1 if d < r else 0) for d in range(D)]
    t = max(0, min(t, E))
    held, rest = [], []
    for l in range(L):
        o = order_desc(prof[l])
        held.append(sorted(o[:t]))
        rest.append(o[t:])
    nload, dload = [0.0] * topo.nodes, [0.0] * D
    owners = [[-1] * E for _ in range(L)]

    def pick(v):
        best = None
        for n in range(topo.nodes):
            devs = topo.members(n)
            if not any(free[d] > 0 for d in devs):
                continue
            key = (nload[n], sum(free[d] for d in devs), n)
            if best is None or key < best:
                best = key
        if best is None:
            raise OracleError(ERR_INFEASIBLE, "no device slot left while placing experts")
        n = best[2]
        d = min((d for d in topo.members(n) if free[d] > 0),
                key=lambda d: (dload[d], free[d], d))
        free[d] -= 1
        dload[d] += v
        nload[n] += v
        return d

    heavy = [max((float(prof[l][e]) for e in rest[l]), default=float("-inf")) for l in range(L)]
    for l in sorted(range(L), key=lambda l: (-heavy[l], l)):
        for e in rest[l]:
            owners[l][e] = pick(float(prof[l][e]))
    cur = 0
    for l in range(L):
        for e in held[l]:
            tries = 0
            while free[cur] == 0:
                cur = (cur + 1) % D
                tries += 1
                if tries > D:
                    raise OracleError(ERR_INFEASIBLE, "slot accounting exhausted during fill")
            owners[l][e] = cur
            free[cur] -= 1
            cur = (cur + 1) % D
    return owners


def estimate(history, window=5):
    """estimate_loads (planner.py:32-42)."""
    if len(history) == 0 or window <= 0:
        raise OracleError(ERR_EMPTY_HISTORY, "bad history/window")
    last = [np.asarray(h, dtype=np.float64) for h in list(history)[-window:]]
    return np.mean(np.stack(last), axis=0)


# ------------------------------------------------------------------ FssdpState decisions
def shard_score(owners, profile, topo):
    """_shard_score (engine.py:431-442), numpy reductions included."""
    dev = np.zeros(topo.D)
    for l, row in enumerate(owners):
        for e, d in enumerate(row):
            dev[d] += profile[l][e]
    node = [dev[topo.members(n)].sum() for n in range(topo.nodes)]
    return (float(max(node)), float(dev.max()))


def plan_layer(owner, est, actual, topo, k):
    """Per-layer FSSDP decision (engine.py:491-553).  k: dict of knobs
    t, m, calibration, rematerialize, expert_bytes, token_bytes, attn_fwd_time, ptt.
    Returns dict(target, added, route, spag, sprs, remat, calib, adopted, calibrated)."""
    E, D = len(owner), topo.D
    base = owner_entries(owner)
    tgt = base
    spag = sprs = remat = calib = 0.0
    adopted = calibrated = False
    act = np.asarray(actual, dtype=np.int64)
    if not (k["t"] <= 0 or k["m"] <= 0):
        if est is not None:
            cand, _ = materialize(owner, est, k["t"], k["m"], topo)
            if cand != base:
                tok = np.clip(np.rint(est), 0, None).astype(np.int64)
                before = moe_latency(base, tok, E, topo, k["token_bytes"], k["ptt"])
                after = moe_latency(cand, tok, E, topo, k["token_bytes"], k["ptt"])
                s_lat = latency(spag_matrix(base, cand, E, D, k["expert_bytes"])[0], topo)
                r_lat = latency(sprs_matrix(cand, base, E, D, k["expert_bytes"])[0], topo)
                rm = s_lat if k["rematerialize"] else 0.0
                if after + s_lat + r_lat + rm < before:
                    tgt, adopted = cand, True
        if tgt != base:
            spag = latency(spag_matrix(base, tgt, E, D, k["expert_bytes"])[0], topo)
        if k["calibration"]:
            am = max(added_counts(base, tgt, D))
            ok, ext, extra, _, _ = calibrate(base, tgt, act.astype(np.float64), k["m"] - am,
                                             max(0.0, k["attn_fwd_time"] - spag), topo, E,
                                             k["expert_bytes"], k["token_bytes"], k["ptt"])
            if ok:
                tgt, calib, calibrated = ext, extra, True
            if tgt != base:
                kept = moe_latency(tgt, act, E, topo, k["token_bytes"], k["ptt"]) + calib
                if kept >= moe_latency(base, act, E, topo, k["token_bytes"], k["ptt"]):
                    tgt, calib = base, 0.0
        if tgt != base:
            sprs = latency(sprs_matrix(tgt, base, E, D, k["expert_bytes"])[0], topo)
            if k["rematerialize"]:
                remat = latency(spag_matrix(base, tgt, E, D, k["expert_bytes"])[0], topo)
    route = route_counts(act, tgt, E, topo)
    return dict(target=tgt, added=added_counts(base, tgt, D), route=route, spag=spag, sprs=sprs,
                remat=remat, calib=calib, adopted=adopted, calibrated=calibrated)


class FssdpReplay:
    """Oracle replay of FssdpState.run_iteration decisions over a trace (engine.py:389-557)."""

    def __init__(self, layers, experts, topo, knobs, window=5, reshard_interval=100):
        self.L, self.E, self.topo, self.k = layers, experts, topo, knobs
        self.window, self.interval = window, reshard_interval
        self.hist = [deque(maxlen=max(1, window)) for _ in range(layers)]
        self.owners = shard_plan_even_owners(layers, experts, topo.D)
        self.it = 0

    def step(self, counts_per_layer):
        resharded = False
        if self.k["t"] > 0 and self.k["m"] > 0:
            if (self.it > 0 and self.interval > 0 and self.it % self.interval == 0
                    and all(self.hist)):
                prof = np.stack([estimate(self.hist[l], self.window).sum(axis=0)
                                 for l in range(self.L)])
                cand = shard(prof, self.k["t"], self.topo)
                if shard_score(cand, prof, self.topo) < shard_score(self.owners, prof, self.topo):
                    self.owners = cand
                    resharded = True
        out = []
        for l, counts in enumerate(counts_per_layer):
            est = estimate(self.hist[l], self.window) if self.hist[l] else None
            out.append(plan_layer(self.owners[l], est, counts, self.topo, self.k))
        for l, counts in enumerate(counts_per_layer):
            self.hist[l].append(np.asarray(counts, dtype=np.int64))
        self.it += 1
        return out, resharded
