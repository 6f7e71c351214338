"""TEST INFRASTRUCTURE ONLY — CPU restatement of the reference analyzer path.

A plain-Python/numpy restatement of the collsight trigger + root-cause
analysis (the path of SURVEY.md §8(a)), written function by function from the
reference sources (citations are proj/... paths in /root/reference). It is
the independent specification the tests check the compiled reference
(oracle/_ref) and the B200 engine against; it is pinned by
tests/test_oracle.py, which requires it to reproduce the reference's own
reports on the catalog and the known-answer fixtures.

Never imported by the product (paper_2509_03018_b200/): only tests/ may use it.
Records are numpy arrays of paper_2509_03018_b200._abi.RECORD_DTYPE in store
(emission) order; the store index of a record is its array position.
"""
from __future__ import annotations

from collections import defaultdict, deque
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

M64 = (1 << 64) - 1
OP_SEND, OP_RECV = 3, 4
COMPLETION, STATE = 0, 1
# categories / sides / verdicts (proj/include/collsight/rca.hpp:16-37)
UNINIT, NOT_READY, RECV_FAILED, GPU_ISSUE, LATE_START, LATE_END, FLOW_INCOMPLETE, \
    FLOW_SKEWED = range(8)
LOCAL, REMOTE, UNDET = range(3)
V_SUSPECTS, V_UNDET, V_FALSE, V_INSUFF, V_NOSTRAG = range(5)
FAILURE, STRAGGLER = 0, 1


def mix64(x: int, b: Optional[int] = None) -> int:
    """proj/include/collsight/types.hpp:78-87"""
    if b is not None:
        return mix64(x ^ mix64(b))
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


class Store:
    """TraceStore (proj/src/trace.cpp:99) + RankIndex (proj/src/rca.cpp:77-90):
    per-rank record indices in store order."""

    def __init__(self, recs: np.ndarray):
        self.recs = recs
        self.ts = recs["ts"].astype(np.float64)
        self.op = recs["op_seq"].astype(np.int64)
        self.rank = recs["rank"].astype(np.int64)
        self.comm = recs["comm_id"].astype(np.int64)
        self.chan = recs["channel"].astype(np.int64)
        self.kind = recs["kind"].astype(np.int64)
        self.opname = recs["op_name"].astype(np.int64)
        self.start = recs["start_ms"].astype(np.float64)
        self.bytes = recs["msg_bytes"].astype(np.uint64)
        self.ready = recs["gpu_ready"].astype(np.int64)
        self.tx = recs["rdma_transmitted"].astype(np.int64)
        self.done = recs["rdma_done"].astype(np.int64)
        self.n = len(recs)
        order = np.argsort(self.rank, kind="stable")
        ranks, starts = np.unique(self.rank[order], return_index=True)
        bounds = list(starts) + [len(order)]
        self.by_rank: Dict[int, np.ndarray] = {
            int(r): order[bounds[i]:bounds[i + 1]] for i, r in enumerate(ranks)}
        self._runmax: Dict[int, np.ndarray] = {}

    def of(self, r: int) -> np.ndarray:
        return self.by_rank.get(int(r), np.zeros(0, dtype=np.int64))

    def prefix(self, r: int, t: float) -> np.ndarray:
        """The reference's prefix scans `for i in rank's records: if ts > t:
        break` (proj/src/rca.cpp:156,176,208,224,232,336,713)."""
        idx = self.of(r)
        if r not in self._runmax:
            self._runmax[r] = np.maximum.accumulate(self.ts[idx]) if len(idx) else idx
        rm = self._runmax[r]
        return idx[: int(np.searchsorted(rm, t, side="right"))] if len(idx) else idx


# ---- store queries (proj/src/trace.cpp:101-144) ---------------------------

def query(st: Store, ranks, t0: float, t1: float) -> List[int]:
    if t0 > t1:
        raise ValueError("query: t0 > t1")
    rs = set(int(r) for r in ranks)
    sel = [i for i in range(st.n) if not (st.ts[i] < t0 or st.ts[i] > t1)
           and int(st.rank[i]) in rs]
    return sorted(sel, key=lambda i: (st.ts[i], st.rank[i]))  # stable


def last_log_per_rank(st: Store, members, t: float) -> List[Tuple[int, int]]:
    if not len(members):
        raise ValueError("last_log_per_rank: empty group")
    out = []
    for m in members:
        best = None
        for i in st.of(m):
            if st.ts[i] > t:
                continue
            if best is None or st.ts[i] >= st.ts[best]:
                best = i
        if best is not None:
            out.append((int(m), int(best)))
    return out


# ---- trigger (proj/src/trigger.cpp) -------------------------------------

@dataclass
class Baseline:
    throughput: float = 0.0
    op_interval_ms: float = 0.0
    interval_defined: bool = False
    updates: int = 0


@dataclass
class TriggerState:
    baselines: Dict[int, Baseline] = field(default_factory=dict)
    had_records_prev: Dict[int, bool] = field(default_factory=dict)


def sample_ranks(groups, kinds, cap: int, seed: int) -> List[int]:
    """trigger.cpp:29-55; groups[g] = members, kinds[g] = 0 for DP."""
    dp = [g for g in range(len(groups)) if kinds[g] == 0]
    if len(dp) > cap:
        dp.sort(key=lambda g: (mix64(seed, g | (1 << 32)), g))
        dp = dp[:cap]
    out = {groups[g][mix64(seed, g) % len(groups[g])] for g in dp}
    return sorted(out)


def evaluate(st: Store, sampled, t: float, state: TriggerState, cfg) -> Optional[tuple]:
    """trigger.cpp:57-136. Python floats are IEEE doubles and the
    expressions below are evaluated in the reference's order (no FMA)."""
    tripped = None
    for r in sampled:
        idx = st.of(r)
        w = idx[~((st.ts[idx] < t - cfg.delta_ms) | (st.ts[idx] > t))]
        comps = w[st.kind[w] == COMPLETION]
        has_state = bool((st.kind[w] == STATE).any())
        had_prev = state.had_records_prev.get(r, False)
        state.had_records_prev[r] = len(w) > 0
        if len(comps) == 0:
            if (has_state or (len(w) == 0 and had_prev)) and tripped is None:
                tripped = (FAILURE, r, t)
            continue
        # sum in the query's (ts, rank) order
        order = sorted(comps, key=lambda i: st.ts[i])
        window_bytes = 0.0
        for i in order:
            window_bytes += float(int(st.bytes[i]))
        ends = sorted(float(st.ts[i]) for i in comps)
        throughput = window_bytes / cfg.delta_ms
        mean_interval, interval_defined = 0.0, False
        if len(ends) >= 2:
            mean_interval = (ends[-1] - ends[0]) / float(len(ends) - 1)
            interval_defined = True
        b = state.baselines.setdefault(r, Baseline())
        warmed = b.updates >= cfg.warmup_windows
        strag = False
        if warmed and b.throughput > 0 and throughput <= cfg.throughput_drop_factor * b.throughput:
            strag = True
        if (warmed and not strag and interval_defined and b.interval_defined
                and b.op_interval_ms > 0
                and mean_interval >= cfg.interval_inflation_factor * b.op_interval_ms):
            strag = True
        if strag:
            if tripped is None:
                tripped = (STRAGGLER, r, t)
            continue
        a = cfg.ema_alpha
        b.throughput = throughput if b.updates == 0 else (1 - a) * b.throughput + a * throughput
        if interval_defined:
            b.op_interval_ms = (mean_interval if not b.interval_defined
                                else (1 - a) * b.op_interval_ms + a * mean_interval)
            b.interval_defined = True
        b.updates += 1
    return tripped


# ---- RCA helpers (proj/src/rca.cpp) ---------------------------------------

class Model:
    """Topology groups (comm_id == index, ring order) + OpProgram."""

    def __init__(self, world: int, groups, kinds, ops):
        self.world = world
        self.groups = [list(g) for g in groups]
        self.kinds = list(kinds)
        self.ops = ops  # list of dicts: name, group, src, dst, deps
        self.opn = len(ops)

    def groups_of(self, r: int) -> List[int]:
        return [g for g, m in enumerate(self.groups) if r in m]

    def executing(self, op) -> List[int]:
        """program.cpp:11-16"""
        if op["name"] == OP_SEND:
            return [op["src"]]
        if op["name"] == OP_RECV:
            return [op["dst"]]
        return self.groups[op["group"]]


def progress_of(st: Store, r: int, op: int, t: float):
    """rca.cpp:167-196 -> (known, (ready, tx, done), evidence list)"""
    pre = st.prefix(r, t)
    sel = pre[(st.kind[pre] == STATE) & (st.op[pre] == op)]
    latest = {}
    for i in sel:  # later store index wins per channel
        latest[int(st.chan[i])] = i
    if not latest:
        return False, (0, 0, 0), []
    rd = tx = dn = 0
    ev = []
    for ch in sorted(latest):
        i = latest[ch]
        rd += int(st.ready[i])
        tx += int(st.tx[i])
        dn += int(st.done[i])
        ev.append({"rank": int(r), "channel": ch, "time_ms": float(st.ts[i]),
                   "op_seq": int(st.op[i])})
    M = (1 << 64) - 1
    return True, (rd & M, tx & M, dn & M), ev


def stall_onset_of(st: Store, r: int, op: int, t: float) -> float:
    """rca.cpp:202-212"""
    pre = st.prefix(r, t)
    hit = pre[st.op[pre] == op]
    return float(st.ts[hit[0]]) if len(hit) else 0.0


def stuck_on_incomplete(st: Store, r: int, ws: float, t: float):
    """rca.cpp:216-237 -> op or None"""
    pre = st.prefix(r, t)
    inw = pre[st.ts[pre] >= ws]
    if not len(inw) or st.kind[inw[-1]] == COMPLETION:
        return None
    op = st.op[inw[-1]]
    if np.any((st.kind[pre] == COMPLETION) & (st.op[pre] == op)):
        return None
    return int(op)


def check_min_op(pairs):
    """rca.cpp:249-261"""
    if not pairs:
        raise ValueError("check_min_op: no last logs supplied")
    mn = min(op for _, op in pairs)
    mins = [r for r, op in pairs if op == mn]
    if len(mins) == len(pairs):
        return None
    return sorted(mins)


def check_min_data(pairs):
    """rca.cpp:263-276; pairs of (rank, (ready, tx, done))"""
    if not pairs:
        raise ValueError("check_min_data: no progress supplied")
    key = lambda p: (p[2], p[1], p[0])
    mn = min(key(p) for _, p in pairs)
    return sorted(r for r, p in pairs if key(p) == mn)


def check_rc_table(c, peer=None):
    """rca.cpp:278-306; c = (ready, tx, done)"""
    ready, tx, done = c
    if not (ready >= tx >= done):
        raise ValueError("check_rc_table: counters violate the pipeline invariant")
    if ready == 0 and tx == 0 and done == 0:
        cat = UNINIT
    elif tx > done:
        cat = RECV_FAILED
    elif ready > tx:
        cat = NOT_READY
    else:
        cat = GPU_ISSUE
    side = UNDET
    if cat == GPU_ISSUE:
        side = LOCAL
    elif (peer is not None and cat == RECV_FAILED and ready == tx
          and peer[0] == peer[1] and peer[1] == peer[2]):
        side = REMOTE
    return cat, side


def lower_median(values):
    """rca.cpp:322-325"""
    v = sorted(values)
    return v[(len(v) - 1) // 2]


def group_iterations(st: Store, m: Model, g: int, t: float):
    """rca.cpp:327-349 -> {rank: {iter: [start, end]}}"""
    out = {}
    for r in m.groups[g]:
        if not len(st.of(r)):
            continue
        for i in st.prefix(r, t):
            if st.kind[i] != COMPLETION or st.comm[i] != g:
                continue
            it = int(np.trunc(st.op[i] / m.opn)) if st.op[i] < 0 else int(st.op[i] // m.opn)
            span = out.setdefault(r, {}).get(it)
            if span is None:
                out[r][it] = [float(st.start[i]), float(st.ts[i])]
            else:
                span[0] = min(span[0], float(st.start[i]))
                span[1] = max(span[1], float(st.ts[i]))
    return out


def complete_iterations(m: Model, g: int, table):
    """rca.cpp:352-372"""
    common = None
    for r in m.groups[g]:
        if r not in table:
            return []
        its = sorted(table[r])
        common = its if common is None else sorted(set(common) & set(its))
    return common or []


def group_has_late_member(st, m, g, cfg, t):
    """rca.cpp:374-396"""
    if len(m.groups[g]) < 2 or m.opn == 0:
        return False
    table = group_iterations(st, m, g, t)
    comp = complete_iterations(m, g, table)
    if not comp:
        return False
    j = comp[-1]
    starts = [table[r][j][0] for r in m.groups[g]]
    ends = [table[r][j][1] for r in m.groups[g]]
    ms, me = lower_median(starts), lower_median(ends)
    return any(s - ms >= cfg.straggler_threshold_ms or e - me >= cfg.straggler_threshold_ms
               for s, e in zip(starts, ends))


def affected_groups(st: Store, m: Model, cfg, trigger) -> List[int]:
    """rca.cpp:400-461"""
    kind, suspect, t = trigger
    ws = t - cfg.delta_ms
    flagged = [False] * len(m.groups)
    for g, members in enumerate(m.groups):
        for r in members:
            if stuck_on_incomplete(st, r, ws, t) is not None:
                flagged[g] = True
                break
        if not flagged[g] and kind == STRAGGLER and group_has_late_member(st, m, g, cfg, t):
            flagged[g] = True
    adj = defaultdict(list)

    def link(a, b):
        if a != b:
            adj[a].append(b)
            adj[b].append(a)
    for op in m.ops:
        for d in op["deps"]:
            link(op["group"], m.ops[d]["group"])
    for r in range(m.world):
        gs = m.groups_of(r)
        for a, b in zip(gs, gs[1:]):
            link(a, b)
    seen = set(m.groups_of(suspect))
    frontier = deque(sorted(seen))
    out = []
    while frontier:
        g = frontier.popleft()
        if flagged[g]:
            out.append(g)
        for nx in adj[g]:
            if nx not in seen:
                seen.add(nx)
                frontier.append(nx)
    return sorted(out)


class DepIndex:
    """rca.cpp:94-139: parents of each global op = depends_on + each executing
    rank's previous global op (carried across iterations)."""

    def __init__(self, m: Model, max_iteration: int):
        self.parents = defaultdict(list)
        prev = {}
        for it in range(max_iteration + 1):
            for s, op in enumerate(m.ops):
                gl = it * m.opn + s
                par = self.parents[gl]
                for d in op["deps"]:
                    par.append(it * m.opn + d)
                for r in m.executing(op):
                    if r in prev and prev[r] not in par:
                        par.append(prev[r])
                    prev[r] = gl

    def depends_on(self, down: int, up: int) -> bool:
        if down == up:
            return False
        seen = set()
        fr = deque([down])
        while fr:
            cur = fr.popleft()
            for p in self.parents.get(cur, ()):
                if p == up:
                    return True
                # pruning below `up` keeps the answer (every edge points to a
                # smaller global op) and bounds the search
                if p > up and p not in seen:
                    seen.add(p)
                    fr.append(p)
        return False


def _entry(c):
    return {"rank": c["rank"], "category": c["category"], "side": c["side"],
            "group": c["group"], "op_seq": c["op"], "onset_ms": c["onset"]}


def _finish(rep, cands_sorted, keep):
    seen = set()
    for c, k in zip(cands_sorted, keep):
        if not k:
            rep["exonerated"].append(_entry(c))
            continue
        if c["rank"] in seen:
            continue
        seen.add(c["rank"])
        rep["suspects"].append(_entry(c))
        rep["evidence"].extend(c["evidence"])
    rep["suspects"].sort(key=lambda e: e["rank"])


def _report(trigger, n):
    kind, suspect, t = trigger
    return {"verdict": V_UNDET, "kind": kind, "suspect_rank": suspect, "time_ms": t,
            "suspects": [], "exonerated": [], "affected_groups": [], "evidence": [],
            "records_scanned": n}


def analyze_failure(st: Store, m: Model, cfg, trigger) -> dict:
    """rca.cpp:540-631 (+ exonerate, rca.cpp:479-526)"""
    t = trigger[2]
    rep = _report(trigger, st.n)
    rep["affected_groups"] = affected_groups(st, m, cfg, trigger)
    if not rep["affected_groups"] or m.opn == 0:
        rep["verdict"] = V_FALSE
        return rep
    rep["records_scanned"] = 2 * st.n
    sel = st.op[st.ts <= t]
    max_iter = max(0, int(np.max(np.trunc(sel / m.opn)))) if len(sel) else 0
    deps = DepIndex(m, max_iter + 1)
    cands = []
    for g in rep["affected_groups"]:
        members = m.groups[g]
        logs = []
        for r in members:
            pre = st.prefix(r, t)
            if len(pre):
                logs.append((r, int(pre[-1])))
        if not logs:
            continue
        last_ops = [(r, int(st.op[i])) for r, i in logs]
        mins = check_min_op(last_ops)
        if mins is None:
            prog = []
            for r, op in last_ops:
                k, p, _ = progress_of(st, r, op, t)
                if k:
                    prog.append((r, p))
            if not prog:
                continue
            mins = check_min_data(prog)
        for r in mins:
            op = [o for rr, o in last_ops if rr == r][-1]
            known, p, ev = progress_of(st, r, op, t)
            peer = None
            if len(members) >= 2:
                succ = members[(members.index(r) + 1) % len(members)]
                pk, pp, pev = progress_of(st, succ, op, t)
                if pk:
                    peer = pp
                    ev = ev + pev
            if known:
                cat, side = check_rc_table(p, peer)
            else:
                cat, side = UNINIT, UNDET
            if not ev:
                for rr, i in logs:
                    if rr == r:
                        ev.append({"rank": r, "channel": int(st.chan[i]),
                                   "time_ms": float(st.ts[i]), "op_seq": int(st.op[i])})
            cands.append({"rank": r, "group": g, "op": op,
                          "onset": stall_onset_of(st, r, op, t), "known": known,
                          "prog": p, "category": cat, "side": side, "evidence": ev})
    order = sorted(range(len(cands)), key=lambda i: (cands[i]["op"], cands[i]["rank"], i))
    cs = [cands[i] for i in order]
    retained = []
    keep = []
    for c in cs:
        drop = False
        for u in retained:
            if u["rank"] == c["rank"]:
                continue
            if u["op"] == c["op"]:
                path = (u["known"] and c["known"] and
                        (u["prog"][2], u["prog"][1], u["prog"][0]) <
                        (c["prog"][2], c["prog"][1], c["prog"][0]))
            else:
                path = deps.depends_on(c["op"], u["op"])
            if path:
                drop = True
                break
        keep.append(not drop)
        if not drop:
            retained.append(c)
    _finish(rep, cs, keep)
    rep["verdict"] = V_SUSPECTS if rep["suspects"] else V_UNDET
    return rep


def _iter(op, opn):
    return int(np.trunc(op / opn)) if op < 0 else op // opn


def analyze_straggler(st: Store, m: Model, cfg, trigger) -> dict:
    """rca.cpp:633-877"""
    t = trigger[2]
    k = cfg.consecutive_iterations_k
    rep = _report(trigger, st.n)
    rep["affected_groups"] = affected_groups(st, m, cfg, trigger)
    if not rep["affected_groups"] or m.opn == 0:
        rep["verdict"] = V_FALSE
        return rep
    rep["records_scanned"] = 2 * st.n
    opn = m.opn
    any_history = False
    cands = []
    for g in rep["affected_groups"]:
        members = m.groups[g]
        if len(members) < 2:
            continue
        table = group_iterations(st, m, g, t)
        comp = complete_iterations(m, g, table)
        if len(comp) < k:
            continue
        any_history = True
        gfo = min([s for s, op in enumerate(m.ops) if op["group"] == g], default=opn)
        window = comp[-k:]
        for r in members:
            sl = el = True
            for j in window:
                starts = [table[x][j][0] for x in members]
                ends = [table[x][j][1] for x in members]
                if table[r][j][0] - lower_median(starts) < cfg.straggler_threshold_ms:
                    sl = False
                if table[r][j][1] - lower_median(ends) < cfg.straggler_threshold_ms:
                    el = False
            if not sl and not el:
                continue
            cands.append({"rank": r, "category": LATE_START if sl else LATE_END,
                          "side": LOCAL, "group": g, "op": window[-1] * opn + gfo,
                          "onset": table[r][window[0]][0], "lo": window[0],
                          "hi": window[-1],
                          "evidence": [{"rank": r, "channel": -1,
                                        "time_ms": table[r][j][0],
                                        "op_seq": j * opn + gfo} for j in window]})
        flows = defaultdict(list)
        states = defaultdict(set)
        completed = set()
        for r in members:
            for i in st.prefix(r, t):
                if st.comm[i] != g:
                    continue
                comp_rec = st.kind[i] == COMPLETION
                if comp_rec and st.opname[i] == OP_RECV:
                    continue
                if not comp_rec and m.ops[int(st.op[i]) % opn]["name"] == OP_RECV:
                    continue
                if comp_rec:
                    completed.add((r, int(st.op[i]), int(st.chan[i])))
                if st.ts[i] < t - cfg.delta_ms:
                    continue
                if comp_rec:
                    flows[(r, int(st.op[i]))].append(i)
                else:
                    states[(r, int(st.op[i]))].add(int(st.chan[i]))
        already = lambda r: any(c["rank"] == r for c in cands)
        for (r, op), comps in sorted(flows.items()):
            if already(r) or len(comps) < 2:
                continue
            durs = [float(st.ts[i]) - float(st.start[i]) for i in comps]
            med = lower_median(durs)
            for i, d in zip(comps, durs):
                if med > 0 and d > cfg.flow_skew_factor * med:
                    cands.append({"rank": r, "category": FLOW_SKEWED, "side": LOCAL,
                                  "group": g, "op": op, "onset": float(st.start[i]),
                                  "lo": 0, "hi": -1,
                                  "evidence": [{"rank": r, "channel": int(st.chan[i]),
                                                "time_ms": float(st.ts[i]), "op_seq": op}]})
                    break
        for (r, op), chans in sorted(states.items()):
            if already(r):
                continue
            if not any((r, op, ch) in completed for ch in chans):
                continue
            for ch in sorted(chans):
                if (r, op, ch) not in completed:
                    cands.append({"rank": r, "category": FLOW_INCOMPLETE, "side": LOCAL,
                                  "group": g, "op": op, "onset": t, "lo": 0, "hi": -1,
                                  "evidence": [{"rank": r, "channel": ch, "time_ms": t,
                                                "op_seq": op}]})
                    break
    if not cands:
        rep["verdict"] = V_NOSTRAG if any_history else V_INSUFF
        return rep
    by_op = defaultdict(lambda: defaultdict(list))
    cohort = defaultdict(list)
    for i in np.nonzero((st.ts <= t) & (st.kind == COMPLETION) & (st.opname != OP_RECV))[0]:
        d = float(st.ts[i]) - float(st.start[i])
        by_op[int(st.op[i])][int(st.rank[i])].append(d)
        cohort[(int(st.opname[i]), _iter(int(st.op[i]), opn))].append(d)
    rep["records_scanned"] += st.n

    def self_faulted(c):
        if c["hi"] < c["lo"]:
            return True
        for op, by_rank in sorted(by_op.items()):
            it = _iter(op, opn)
            if it < c["lo"] or it > c["hi"] or c["rank"] not in by_rank:
                continue
            sib = [d for rr, ds in by_rank.items() if rr != c["rank"] for d in ds]
            if not sib:
                co = cohort.get((m.ops[op % opn]["name"], it))
                if co is None or len(co) < 2:
                    continue
                sib = co
            med = lower_median(sib)
            if med <= 0:
                continue
            if any(d > cfg.flow_skew_factor * med for d in by_rank[c["rank"]]):
                return True
        return False

    sf = [self_faulted(c) for c in cands]
    any_self = any(sf)
    order = sorted(range(len(cands)), key=lambda i: (cands[i]["op"], cands[i]["rank"], i))
    _finish(rep, [cands[i] for i in order], [(not any_self) or sf[i] for i in order])
    rep["verdict"] = V_SUSPECTS if rep["suspects"] else V_NOSTRAG
    return rep


def analyze(st, m, cfg, trigger):
    """rca.cpp:879-884"""
    return (analyze_failure if trigger[0] == FAILURE else analyze_straggler)(st, m, cfg, trigger)


def run_detection(recs: np.ndarray, m: Model, tcfg, acfg, seed: int):
    """runner.cpp:47-81 -> list of structured reports"""
    st = Store(recs)
    last_ts = 0.0
    for x in st.ts:
        last_ts = max(last_ts, float(x))
    sampled = sample_ranks(m.groups, m.kinds, tcfg.max_sampled_ranks, seed)
    state = TriggerState()
    out = []
    t = tcfg.detect_interval_ms
    while t <= last_ts:
        if not (t < tcfg.delta_ms):
            trig = evaluate(st, sampled, t, state, tcfg)
            if trig is not None:
                out.append(analyze(st, m, acfg, trig))
        t += tcfg.detect_interval_ms
    return out, sampled


def model_from(topo, prog) -> Model:
    """From paper_2509_03018_b200.model Topology / OpProgram (plain data)."""
    return Model(topo.world_size, [g.members for g in topo.groups],
                 [g.kind for g in topo.groups],
                 [{"name": o.op_name, "group": o.group, "src": o.src, "dst": o.dst,
                   "deps": list(o.depends_on)} for o in prog.ops])
