"""ORACLE TEST INFRASTRUCTURE — CPU restatement of the spec-only modules.

Not product code: only tests/, __graft_entry__.smoke() and bench.py's CPU
baseline may import this file.  It restates, in plain Python on integer
ticks, the reference specification's memory / network / simulator /
costmodel / tuner operations:

    peak_memory            SPEC.md:218-226     enumerate_candidates
    transfer_duration      SPEC.md:276-284     record/estimate
    profile_links          SPEC.md:294-301     simulate
    bubble_report          SPEC.md:351-354     queue_analysis
    estimate_length        SPEC.md:400-408     rank_candidates
    run_adaptive           SPEC.md:453-461     switch_plan

with the ambiguity resolutions of SURVEY.md Appendix C.  The reference ships
no code for these modules, so "parity" here is pinned by the SPEC examples
and acceptance criteria (tests/test_spec_oracle.py) — this oracle is NOT
pinned to reference outputs beyond those examples.

The planner part (task graph ids, kFkB orders) is restated from
proj/src/taskgraph.cpp:35-106 and proj/src/plan.cpp:20-66 and is itself
checked against the compiled reference (oracle/_ref) in the tests.

Input/output: the same scenario dicts as libptk's ptk_scenario_json().
"""
from __future__ import annotations

import heapq
import math

TICKS = 1_000_000_000
F, B, SEND, RECV, GA = 0, 1, 2, 3, 4


class SpecError(Exception):
    def __init__(self, kind, msg=""):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


def llround(x: float) -> int:
    """C llround: round half away from zero."""
    if x >= 0:
        r = math.floor(x)
        return int(r + 1 if x - r >= 0.5 else r)
    r = math.ceil(x)
    return int(r - 1 if r - x >= 0.5 else r)


def to_ticks(units: float) -> int:
    return llround(units * 1e9)


def to_units(ticks: int) -> float:
    return ticks / 1e9


# ------------------------------------------------------------------ model / graph / plan
def stage_list(model):
    out = []
    for i, s in enumerate(model["stages"]):
        d = {"stage_id": i, "forward_fixed": 0.0, "forward_per_sample": 0.0, "backward_fixed": 0.0,
             "backward_per_sample": 0.0, "weight_bytes": 0, "activation_bytes_per_sample": 0,
             "output_bytes_per_sample_fwd": 0, "output_bytes_per_sample_bwd": 0}
        d.update(s)
        out.append(d)
    return out


def compute_ticks(st, b, fwd):
    if fwd:
        return to_ticks(st["forward_fixed"] + float(b) * st["forward_per_sample"])
    return to_ticks(st["backward_fixed"] + float(b) * st["backward_per_sample"])


class Graph:
    """Task graph with the reference id layout (taskgraph.cpp:43-90)."""

    def __init__(self, stages, b, M):
        S = len(stages)
        self.S, self.M, self.b = S, M, b
        self.nodes = []  # (kind, stage, mb, device, link, bytes)
        self.fwd = [[0] * M for _ in range(S)]
        self.bwd = [[0] * M for _ in range(S)]
        self.ga = [0] * S
        for s in range(S):
            for m in range(M):
                self.fwd[s][m] = self._add(F, s, m, s, -1, 0)
                self.bwd[s][m] = self._add(B, s, m, s, -1, 0)
            self.ga[s] = self._add(GA, s, -1, s, -1, 0)
        self.recv_of = {}
        self.send_of = {}
        self.pair = {}
        for m in range(M):
            for s in range(S - 1):
                self._link(self.fwd[s][m], self.fwd[s + 1][m], 2 * s,
                           b * stages[s]["output_bytes_per_sample_fwd"])
            for s in range(S - 1, 0, -1):
                self._link(self.bwd[s][m], self.bwd[s - 1][m], 2 * (s - 1) + 1,
                           b * stages[s]["output_bytes_per_sample_bwd"])

    def _add(self, kind, s, m, d, link, nbytes):
        self.nodes.append((kind, s, m, d, link, nbytes))
        return len(self.nodes) - 1

    def _link(self, src, dst, link, nbytes):
        ks, ss, ms, ds = self.nodes[src][:4]
        kd, sd, md, dd = self.nodes[dst][:4]
        snd = self._add(SEND, ss, ms, ds, link, nbytes)
        rcv = self._add(RECV, sd, md, dd, link, nbytes)
        self.send_of[src] = snd
        self.recv_of[dst] = rcv
        self.pair[snd] = rcv
        self.pair[rcv] = snd


def kfkb_orders(g: Graph, k: int, groups=None):
    """plan.cpp:20-59 walk: warm-up min(S-s, G) groups, alternate B/F groups, drain, GA."""
    if groups is None:
        groups = [(f, min(f + k, g.M) - 1) for f in range(0, g.M, k)]
    G = len(groups)
    orders = []
    for s in range(g.S):
        seq = []
        emit = lambda ids, gr: seq.extend(ids[m] for m in range(gr[0], gr[1] + 1))  # noqa: E731
        nf = nb = 0
        for _ in range(min(g.S - s, G)):
            emit(g.fwd[s], groups[nf])
            nf += 1
        while nf < G:
            emit(g.bwd[s], groups[nb])
            nb += 1
            emit(g.fwd[s], groups[nf])
            nf += 1
        while nb < G:
            emit(g.bwd[s], groups[nb])
            nb += 1
        seq.append(g.ga[s])
        orders.append(seq)
    return orders


def make_plan(model, plan_req):
    stages = stage_list(model)
    b = plan_req.get("micro_batch_size", 1)
    gb = model["global_batch"]
    if b < 1 or gb % b:
        raise SpecError("ConfigError", "b does not divide global_batch")
    M = gb // b
    g = Graph(stages, b, M)
    kind = plan_req.get("kind", "kfkb")
    if kind == "groups":  # B200 extension: explicit consecutive group sizes
        sizes = plan_req.get("groups")
        if not sizes or any(n < 1 for n in sizes):
            raise SpecError("ConfigError", "plan.groups sizes must be >= 1")
        if sum(sizes) != M:
            raise SpecError("PlanError", "groups must cover all micro-batches")
        groups, first = [], 0
        for n in sizes:
            groups.append((first, first + n - 1))
            first += n
        return stages, g, kfkb_orders(g, 0, groups), (max(sizes), b, M)
    if kind not in ("1f1b", "kfkb", "gpipe"):
        raise SpecError("ConfigError", "plan.kind must be 1f1b, kfkb, gpipe or groups")
    k = 1 if kind == "1f1b" else (M if kind == "gpipe" else plan_req.get("k", 1))
    if k < 1 or k > M:
        raise SpecError("PlanError", "k out of range")
    return stages, g, kfkb_orders(g, k), (k, b, M)


# ------------------------------------------------------------------ memory
def peak_memory(stages, g, orders):
    peaks = []
    for s, seq in enumerate(orders):
        act = stages[s]["activation_bytes_per_sample"] * g.b
        live = peak = stages[s]["weight_bytes"]
        for nid in seq:
            kind = g.nodes[nid][0]
            if kind == F:
                live += act
                peak = max(peak, live)
            elif kind == B:
                live -= act
        peaks.append(peak)
    lim = max(range(len(peaks)), key=lambda i: (peaks[i], -i))
    return peaks, lim


def divisors_desc(n):
    return [d for d in range(n, 0, -1) if n % d == 0]


def enumerate_candidates(model, limit, k_max, feasible=None):
    stages = stage_list(model)
    gb = model["global_batch"]
    out = []
    for k in range(1, k_max + 1):
        for b in divisors_desc(gb):
            M = gb // b
            if k > M:
                continue
            if feasible is not None:
                ok, peaks = feasible(k, b), []
            else:
                g = Graph(stages, b, M)
                peaks, _ = peak_memory(stages, g, kfkb_orders(g, k))
                ok = all(p <= limit for p in peaks)
            if ok:
                out.append((k, b, M, peaks))
                break
    if not out:
        raise SpecError("InfeasibleModel", "no candidate fits")
    return out


# ------------------------------------------------------------------ network
def _piece(trace, t):
    for s0, s1, a in trace.get("segments", []):
        a0, a1 = to_ticks(s0), to_ticks(s1)
        if t < a0:
            return 1.0, a0
        if t < a1:
            return a, a1
    return 1.0, None


def transfer_duration(trace, nbytes, start):
    lat = to_ticks(trace.get("latency", 0.0))
    if nbytes == 0:
        return lat
    eff = 1.0
    for bb, e in trace.get("utilization_curve", []):
        if bb == nbytes:
            eff = e
    left = float(nbytes)
    t = start
    while True:
        a, nxt = _piece(trace, t)
        rate = trace.get("base_bandwidth", 1.0) * a * eff
        if nxt is None:
            t += to_ticks(left / rate)
            break
        can = rate * to_units(nxt - t)
        if can >= left:
            t += to_ticks(left / rate)
            break
        left -= can
        t = nxt
    return (t - start) + lat


class Store:
    def __init__(self, window=8):
        self.window = window
        self.q = {}

    def record(self, link, nbytes, dur):
        q = self.q.setdefault((link, nbytes), [])
        q.append(dur)
        del q[:-self.window]

    def estimate(self, link, nbytes):
        q = self.q.get((link, nbytes))
        if not q:
            raise SpecError("NoProfileData", f"link {link} bytes {nbytes}")
        return (2 * sum(q) + len(q)) // (2 * len(q))


def plan_buckets(g):
    return sorted({(n[4], n[5]) for n in g.nodes if n[0] == SEND})


def profile(buckets, traces, clock, repeats, store):
    for link, nbytes in buckets:
        for _ in range(repeats):
            d = transfer_duration(traces[link], nbytes, clock)
            store.record(link, nbytes, d)
            clock += d
    return clock


# ------------------------------------------------------------------ simulator
def simulate(stages, g, orders, compute, transfer, start=0):
    """Event-driven twin of the executor (rules in include/pipetune/simulator.hpp)."""
    S = g.S
    b = g.b
    pc = [0] * S
    busy = [False] * S
    prev_end = [start] * S
    send_free = [start] * S
    recv_free = [start] * S
    sends = [[] for _ in range(S)]  # FIFO of (enqueue time, send id)
    buffered = [0] * S
    resident = [stages[s]["weight_bytes"] for s in range(S)]
    peak = list(resident)
    busy_sum = [0] * S
    first = [None] * S
    last = [None] * S
    arrival = {}
    timeline, qdepth, launches = [], [[] for _ in range(S)], [[] for _ in range(S)]
    ev = []
    seq = [0]

    def push(t, kind, dev, node):
        heapq.heappush(ev, (t, seq[0], kind, dev, node))
        seq[0] += 1

    def dispatch(now):
        moved = True
        while moved:
            moved = False
            for d in range(S):
                if busy[d] or pc[d] >= len(orders[d]):
                    continue
                nid = orders[d][pc[d]]
                r = g.recv_of.get(nid)
                if r is not None and (r not in arrival or arrival[r] > now):
                    continue
                kind = g.nodes[nid][0]
                act = stages[d]["activation_bytes_per_sample"] * b
                dur = 0
                if kind == F:
                    dur = compute(d, b, True)
                    resident[d] += act
                    peak[d] = max(peak[d], resident[d])
                elif kind == B:
                    dur = compute(d, b, False)
                    resident[d] -= act
                if r is not None:
                    launches[d].append([nid, 1 if arrival[r] < prev_end[d] else 0])
                    buffered[d] -= 1
                    qdepth[d].append([now, buffered[d]])
                busy[d] = True
                busy_sum[d] += dur
                if first[d] is None:
                    first[d] = now
                last[d] = now + dur
                timeline.append([nid, d, 0, now, now + dur])
                push(now + dur, 0, d, nid)
                pc[d] += 1
                moved = True
            heads = sorted((sends[d][0][0], sends[d][0][1], d) for d in range(S) if sends[d])
            for enq, sid, p in heads:
                rid = g.pair[sid]
                c = g.nodes[rid][3]
                if send_free[p] > now or recv_free[c] > now:
                    continue
                _, _, _, _, link, nbytes = g.nodes[sid]
                dur = transfer(link, nbytes, now)
                send_free[p] = recv_free[c] = now + dur
                sends[p].pop(0)
                timeline.append([sid, p, 1, now, now + dur])
                timeline.append([rid, c, 2, now, now + dur])
                push(now + dur, 1, c, sid)
                moved = True

    dispatch(start)
    end = start
    while ev:
        t, _, kind, d, nid = heapq.heappop(ev)
        end = max(end, t)
        if kind == 0:
            busy[d] = False
            prev_end[d] = t
            if nid in g.send_of:
                sends[d].append((t, g.send_of[nid]))
        else:
            arrival[g.pair[nid]] = t
            buffered[d] += 1
            qdepth[d].append([t, buffered[d]])
        if ev and ev[0][0] == t:
            continue
        dispatch(t)
    for d in range(S):
        if pc[d] < len(orders[d]) or sends[d]:
            raise SpecError("DeadlockDetected", f"device {d}")
    bubble = [((last[d] - first[d]) if first[d] is not None else 0) - busy_sum[d] for d in range(S)]
    frac = [0.0 if busy_sum[d] + bubble[d] == 0 else bubble[d] / (busy_sum[d] + bubble[d]) for d in range(S)]
    return {"start": start, "pipeline_length": end - start, "busy": busy_sum, "bubble": bubble,
            "bubble_fraction": frac, "peak": peak, "timeline": timeline, "queue_depth": qdepth,
            "launches": launches}


def simulate_true(stages, g, orders, traces, start=0):
    return simulate(stages, g, orders, lambda s, b, f: compute_ticks(stages[s], b, f),
                    lambda link, nb, t: transfer_duration(traces[link], nb, t), start)


# ------------------------------------------------------------------ cost model / tuner
def rank(model, cands, comp, store, mixed=()):
    """Uniform candidates [k, b, M, _] and mixed-k ones (b, [group sizes]) ranked by the simulated
    length over constant profiled durations; ties: smaller (max) k, larger b, group list (uniform
    first).  Mixed entries carry their sizes as a 5th element."""
    stages = stage_list(model)
    out = []

    def length(g, orders):
        return simulate(stages, g, orders, lambda s, bb, f: comp[(s, bb, 0 if f else 1)],
                        lambda link, nb, t: store.estimate(link, nb), 0)["pipeline_length"]

    for k, b, M, _ in cands:
        g = Graph(stages, b, M)
        out.append([k, b, M, length(g, kfkb_orders(g, k))])
    for b, sizes in mixed:
        M = model["global_batch"] // b
        g = Graph(stages, b, M)
        ranges, first = [], 0
        for n in sizes:
            ranges.append((first, first + n - 1))
            first += n
        if first != M:
            raise SpecError("PlanError", "groups do not tile [0, M)")
        out.append([max(sizes), b, M, length(g, kfkb_orders(g, max(sizes), ranges)), list(sizes)])
    out.sort(key=lambda e: (e[3], e[0], -e[1], e[4] if len(e) > 4 else []))
    return out


def decide(ranked, current, h, current_groups=None):
    """Returns (chosen [k, b, M], chosen groups or [], switched)."""
    best = ranked[0]
    groups = lambda e: e[4] if len(e) > 4 else []  # noqa: E731
    if current is None:
        return best[:3], groups(best), False
    cg = list(current_groups or [])
    cur = [e for e in ranked if e[:3] == list(current) and groups(e) == cg]
    if not cur:
        raise SpecError("UnknownCandidate", "current")
    better = float(best[3]) < float(cur[0][3]) * (1.0 - h)
    switched = better and not (best[:3] == list(current) and groups(best) == cg)
    return (best[:3] if switched else list(current)), (groups(best) if switched else cg), switched


def candidate_buckets(model, cands):
    stages = stage_list(model)
    out = set()
    for k, b, M, _ in cands:
        out.update(plan_buckets(Graph(stages, b, M)))
    return sorted(out)


def traces_by_link(req, S):
    n = 2 * (S - 1) if S > 1 else 0
    tr = [None] * n
    for t in req.get("traces", []):
        tr[t["link"]] = t
    if any(x is None for x in tr):
        raise SpecError("ConfigError", "missing trace")
    return tr


def run_adaptive(model, limit, traces, pol, horizon):
    stages = stage_list(model)
    interval = to_ticks(pol.get("interval", 1.0))
    reps = pol.get("profile_repeats", 3)
    h = pol.get("hysteresis", 0.02)
    overhead = to_ticks(pol.get("switch_overhead", 0.0))
    cands = enumerate_candidates(model, limit, pol.get("k_max", 6))
    comp = {}
    for _, b, _, _ in cands:
        for s, st in enumerate(stages):
            comp[(s, b, 0)] = compute_ticks(st, b, True)
            comp[(s, b, 1)] = compute_ticks(st, b, False)
    buckets = candidate_buckets(model, cands)
    store = Store(pol.get("window_size", 8))
    end = to_ticks(horizon)
    rounds, iters = [], []
    clock = 0
    t0 = clock
    clock = profile(buckets, traces, clock, reps, store)
    ranked = rank(model, cands, comp, store)
    cur, _, _ = decide(ranked, None, h)
    rounds.append({"time": t0, "estimates": ranked, "chosen": cur, "switched": False})
    while clock < end:
        rs = clock
        k, b, M = cur
        g = Graph(stages, b, M)
        orders = kfkb_orders(g, k)
        while True:
            r = simulate_true(stages, g, orders, traces, clock)
            L = r["pipeline_length"]
            iters.append([clock, clock + L, k, b, M, model["global_batch"] / to_units(L)])
            clock += L
            if not (clock - rs < interval and clock < end):
                break
        if clock >= end:
            break
        t = clock
        clock = profile(buckets, traces, clock, reps, store)
        ranked = rank(model, cands, comp, store)
        nxt, _, switched = decide(ranked, cur, h)
        if nxt != cur:
            clock += overhead
        cur = nxt
        rounds.append({"time": t, "estimates": ranked, "chosen": cur, "switched": switched})
    samples = sum(it[3] * it[4] for it in iters)
    span = iters[-1][1] - iters[0][0] if iters else 0
    thr = samples / to_units(span) if span > 0 else 0.0
    return {"rounds": rounds, "iterations": iters, "throughput": thr}


# ------------------------------------------------------------------ scenario front door
def run(req: dict) -> dict:
    op = req["op"]
    if op == "transfer":
        return {"duration": transfer_duration(req["trace"], req["bytes"], req.get("start", 0))}
    if op == "estimate":
        st = Store(req.get("window", 8))
        for link, nb, _, dur in req["samples"]:
            st.record(link, nb, dur)
        return {"estimate": st.estimate(*req["query"])}
    model = req["model"]
    S = len(model["stages"])
    if op in ("peak_memory", "simulate"):
        stages, g, orders, _ = make_plan(model, req["plan"])
        if op == "peak_memory":
            peaks, lim = peak_memory(stages, g, orders)
            return {"per_device_peak": peaks, "limiting_device": lim}
        return {"result": simulate_true(stages, g, orders, traces_by_link(req, S), req.get("start", 0))}
    if op == "enumerate":
        k_max = req.get("k_max", max(1, min(model["global_batch"], 6)))
        return {"entries": [[k, b, M, p] for k, b, M, p in
                            enumerate_candidates(model, req["cluster"]["device_memory_limit"], k_max)]}
    if op == "profile":
        stages, g, orders, _ = make_plan(model, req["plan"])
        st = Store(req.get("window", 8))
        clock = profile(plan_buckets(g), traces_by_link(req, S), req.get("clock", 0), req.get("repeats", 3), st)
        return {"clock": clock, "estimates": [[l, b, st.estimate(l, b)] for l, b in plan_buckets(g)]}
    if op == "compare":
        pol = req.get("policy", {})
        cands = enumerate_candidates(model, req["cluster"]["device_memory_limit"], pol.get("k_max", 6))
        stages = stage_list(model)
        comp = {}
        for _, b, _, _ in cands:
            for s, stg in enumerate(stages):
                comp[(s, b, 0)] = compute_ticks(stg, b, True)
                comp[(s, b, 1)] = compute_ticks(stg, b, False)
        st = Store(pol.get("window_size", 8))
        profile(candidate_buckets(model, cands), traces_by_link(req, S), req.get("clock", 0),
                pol.get("profile_repeats", 3), st)
        return {"ranked": rank(model, cands, comp, st)}
    if op == "decide":
        comp = {(s, b, d): t for s, b, d, t in req["compute_profile"]}
        st = Store(req.get("window", 8))
        for link, nb, _, dur in req["samples"]:
            st.record(link, nb, dur)
        cands = [(k, b, M, []) for k, b, M in req["candidates"]]
        mixed = [(b, list(sizes)) for b, sizes in req.get("group_candidates", [])]
        ranked = rank(model, cands, comp, st, mixed)
        cur = req.get("current")
        chosen, groups, switched = decide(ranked, cur, req.get("hysteresis", 0.02), req.get("current_groups"))
        out = {"time": req.get("clock", 0), "estimates": ranked, "chosen": chosen}
        if groups:
            out["chosen_groups"] = groups
        out["switched"] = switched
        return {"decision": out}
    if op == "tune":
        return run_adaptive(model, req["cluster"]["device_memory_limit"], traces_by_link(req, S),
                            req.get("policy", {}), req["horizon"])
    raise SpecError("ConfigError", f"unknown op {op}")
