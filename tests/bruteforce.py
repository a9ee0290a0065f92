"""Independent brute-force references used by the oracle pin tests (pure Python, written from the definitions in
PAPER.md; shares nothing with oracle/oracle.cpp or the CUDA path).

* geometry tables by exhaustive subset enumeration (Alg. 1 by definition);
* a replay checker that rebuilds the partition state from a decision-record stream and re-derives every placement
  decision by brute force over all candidate successors (Alg. 2, Scheme B PAPER.md:577-617,
  fusion/fission PAPER.md:580).
"""
import itertools

FULL = object()


def placements(spec):
    return [(p, s, prof["memory_slots"]) for p, prof in enumerate(spec["profiles"]) for s in prof["starts"]]


def slots_of(spec, p, s):
    return set(range(s, s + spec["profiles"][p]["memory_slots"]))


def valid_states(spec):
    pl = placements(spec)
    comp = [p["compute_slices"] for p in spec["profiles"]]
    out = set()
    for k in range(spec["total_memory_slots"] + 1):
        for combo in itertools.combinations(pl, k):
            used = set()
            ok = True
            for p, s, ln in combo:
                r = set(range(s, s + ln))
                if r & used:
                    ok = False
                    break
                used |= r
            if ok and sum(comp[p] for p, _, _ in combo) <= spec["total_compute_slices"]:
                out.add(frozenset((p, s) for p, s, _ in combo))
    return out


def fcr_table(spec):
    S = valid_states(spec)
    pl = placements(spec)
    finals = [s for s in S if not any((s | {(p, st)}) in S and (p, st) not in s for p, st, _ in pl)]
    return S, {s: sum(1 for f in finals if s <= f) for s in S}


class Replay:
    """Rebuild instance state from records and check each decision is the brute-force optimum."""

    def __init__(self, spec, kind, fcr):
        self.spec, self.kind, self.fcr = spec, kind, fcr
        self.mem = [p["memory_slots"] * spec["slot_mib"] for p in spec["profiles"]]
        self.comp = [p["compute_slices"] for p in spec["profiles"]]
        self.inst = {}  # start -> [prof, busy]
        if kind == 1:  # STATIC layout
            names = [p["name"] for p in spec["profiles"]]
            for n, s in spec["static_layout"]:
                self.inst[s] = [names.index(n), False]
        if kind == 0:
            self.inst[0] = [len(spec["profiles"]) - 1, False]
        self.visited = []

    def state(self):
        return frozenset((p, s) for s, (p, _) in self.inst.items())

    def overlap(self, p, s):
        q = slots_of(self.spec, p, s)
        return [st for st, (pp, _) in self.inst.items() if slots_of(self.spec, pp, st) & q]

    def best_alloc(self, need):
        cands = []
        for st in self.spec["profiles"][need]["starts"]:
            if not self.overlap(need, st):
                t = self.state() | {(need, st)}
                if t in self.fcr:
                    cands.append((self.fcr[t], st))
        return max(cands)[1] if cands else None

    def best_reconf(self, need):
        cands = []
        for st in self.spec["profiles"][need]["starts"]:
            ov = self.overlap(need, st)
            if not ov or any(self.inst[o][1] for o in ov):
                continue
            t = frozenset((p, s) for s, (p, _) in self.inst.items() if s not in ov) | {(need, st)}
            if t in self.fcr:
                cands.append((self.fcr[t], -len(ov), st))
        return max(cands) if cands else None

    def best_reuse(self, need):
        c = [st for st, (p, busy) in self.inst.items()
             if not busy and self.mem[p] == self.mem[need] and self.comp[p] >= self.comp[need]]
        return max(c) if c else None

    def step(self, r):
        k, st, p, nd = r["kind"], r["start"], r["profile"], r["n_destroyed"]
        if k in ("COMPLETE", "OOM", "PREEMPT"):
            assert self.inst[st][1], r
            self.inst[st][1] = False
            if self.kind == 2:
                del self.inst[st]
        elif k == "ALLOC":
            if self.kind == 3:
                assert self.best_reuse(p) is None, r
            assert self.best_alloc(p) == st, (r, self.inst)
            self.inst[st] = [p, True]
        elif k == "RECONF":
            assert self.kind == 3 and self.best_reuse(p) is None and self.best_alloc(p) is None, r
            best = self.best_reconf(p)
            assert best is not None and best[2] == st and -best[1] == nd, (r, best, self.inst)
            for o in self.overlap(p, st):
                del self.inst[o]
            self.inst[st] = [p, True]
        elif k == "REUSE":
            assert self.best_reuse(p) == st, r
            self.inst[st][1] = True
        elif k == "WAIT":
            if self.kind == 3:
                assert self.best_reuse(p) is None and self.best_alloc(p) is None and self.best_reconf(p) is None, r
            elif self.kind == 2:
                assert self.best_alloc(p) is None, r
            elif self.kind == 0:
                assert self.inst[0][1], r
        elif k in ("PLACE_STATIC", "PLACE_BASELINE"):
            assert not self.inst[st][1], r
            self.inst[st][1] = True
        self.visited.append(self.state())
        assert self.state() in self.fcr, (r, self.inst)  # only valid partition states are ever visited
        # invariants: no overlap, memory within capacity
        used = set()
        for s0, (pp, _) in self.inst.items():
            sl = slots_of(self.spec, pp, s0)
            assert not (sl & used)
            used |= sl
        assert sum(self.mem[pp] for pp, _ in self.inst.values()) <= self.spec["total_memory_slots"] * self.spec["slot_mib"]


def reach_counts(n_slots, masks):
    """Alg. 1 by definition on occupancy masks (pure Python): D[t] = number of distinct sets of
    disjoint placements with union t (by brute-force recursion on the lowest occupied slot), finals = states where
    no placement fits, fcr[m] = number of distinct final placement sets reachable from a state with occupancy m
    (sum of D[t] over t in the free slots of m with m | t final). Returns (|S|, |F|, fcr list)."""
    N = 1 << n_slots
    D = [0] * N
    D[0] = 1
    for t in range(1, N):
        low = t & -t
        D[t] = sum(D[t ^ q] for q in masks if (q & low) and (q & ~t) == 0)
    final = [D[m] > 0 and all(q & m for q in masks) for m in range(N)]
    fcr = [0] * N
    for m in range(N):
        if D[m]:
            free = (N - 1) & ~m
            fcr[m] = sum(D[t] for t in range(N) if (t & ~free) == 0 and final[m | t])
    return sum(D), sum(D[m] for m in range(N) if final[m]), fcr


def geometry_masks(spec):
    """Placement masks (bit i = memory slot i) of a geometry JSON spec."""
    return [((1 << prof["memory_slots"]) - 1) << s for prof in spec["profiles"] for s in prof["starts"]]
