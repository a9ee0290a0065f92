"""Pins for the oracle's geometry, Alg. 1 (precompute_reachability) and Alg. 2
(allocate_partition).

Independent checks (none re-uses the oracle's code):
  * a Python brute force over all subsets of placements (maximal sets, superset counting) — Alg. 1 by definition;
  * the paper's own facts: five A100 profiles, the legality example, seven 5 GB
    partitions, the 4/7 + 3/7 pair of 20 GB halves, "1/7 Compute, 1/8 Memory"
    (PAPER.md:1024), "last slice" argmax;
  * the vendor-table derived counts of SURVEY.md §8(c) (A30 |S|=26 |F|=5; A100 |S|=298 |F|=19; 1g.10gb variant
    723/78) and SURVEY.md Appendix A (A100 fcr table) — tests/golden/a100_fcr_table.txt.
"""
import itertools
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR, geom_path
from oracle import oracle as orc


def load(name):
    with open(geom_path(name)) as f:
        return json.load(f)


def placements(spec):
    out = []
    for p, prof in enumerate(spec["profiles"]):
        for s in prof["starts"]:
            out.append((p, s, prof["memory_slots"]))
    return out


def brute_states(spec):
    """All sets of pairwise non-overlapping placements with compute within the GPU (= S, reading R2)."""
    pl = placements(spec)
    comp = [p["compute_slices"] for p in spec["profiles"]]
    states = []
    for k in range(0, spec["total_memory_slots"] + 1):
        for combo in itertools.combinations(range(len(pl)), k):
            slots = set()
            ok = True
            c = 0
            for i in combo:
                p, s, ln = pl[i]
                rng = set(range(s, s + ln))
                if rng & slots:
                    ok = False
                    break
                slots |= rng
                c += comp[p]
            if ok and c <= spec["total_compute_slices"]:
                states.append(frozenset((pl[i][0], pl[i][1]) for i in combo))
    return states


def brute_tables(spec):
    S = brute_states(spec)
    Sset = set(S)
    pl = placements(spec)

    def succ(s):
        out = []
        for p, st, _ in pl:
            t = s | {(p, st)}
            if t != s and t in Sset:
                out.append(t)
        return out

    finals = [s for s in S if not succ(s)]
    fcr = {s: sum(1 for f in finals if s <= f) for s in S}  # reachable finals = maximal supersets
    return S, finals, fcr


@pytest.mark.parametrize("name,nS,nF", [("a30-24gb", 26, 5), ("a100-40gb", 298, 19), ("a100-80gb", 298, 19),
                                         ("h100-80gb", 298, 19), ("a100-40gb-1g10", 723, 78),
                                         ("b200-180gb", 723, 78)])
def test_state_counts_match_bruteforce(name, nS, nF):
    spec = load(name)
    g = orc.Geometry(spec)
    S, F, fcr = brute_tables(spec)
    assert (len(S), len(F)) == (nS, nF)
    n_states, n_finals, _ = g.counts()
    assert (n_states, n_finals) == (nS, nF)
    got = {frozenset(inst): (f, fin) for inst, f, fin in g.states()}
    assert set(got) == set(S)
    for s in S:
        assert got[s][0] == fcr[s], (name, sorted(s))
        assert got[s][1] == (s in set(F))
    assert g.fcr([]) == nF  # fcr(s0) = |F| (every final reachable from the empty GPU)


def test_a30_fcr_table():
    # SURVEY.md §8(c) "fcr table": A30 fcr[occ] (bit i = slot i)
    g = orc.Geometry(load("a30-24gb"))
    want = {0b0000: 5, 0b0001: 2, 0b0010: 2, 0b0100: 2, 0b1000: 2, 0b0011: 2, 0b1100: 2}
    spec = load("a30-24gb")
    for inst, f, _ in g.states():
        m = 0
        for p, s in inst:
            m |= ((1 << spec["profiles"][p]["memory_slots"]) - 1) << s
        assert f == want.get(m, 1), (bin(m), f)


def test_a100_fcr_table_appendix_a():
    # SURVEY.md Appendix A (derived A100 fcr table); also the factorisation fcr = L(low nibble) * R(high nibble).
    table = {}
    with open(os.path.join(GOLDEN_DIR, "a100_fcr_table.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            for tok in line.split():
                m, v = tok.split(":")
                table[int(m, 16)] = int(v)
    spec = load("a100-40gb")
    g = orc.Geometry(spec)
    seen = {}
    for inst, f, _ in g.states():
        m = 0
        for p, s in inst:
            m |= ((1 << spec["profiles"][p]["memory_slots"]) - 1) << s
        seen.setdefault(m, set()).add(f)
    assert all(len(v) == 1 for v in seen.values())  # fcr depends only on the occupancy mask
    assert {m: next(iter(v)) for m, v in seen.items()} == table
    assert len(table) == 144


def test_fcr_invariants():
    # fcr(final) = 1; fcr non-increasing along every alloc edge
    for name in ["a30-24gb", "a100-40gb", "a100-40gb-1g10"]:
        spec = load(name)
        g = orc.Geometry(spec)
        states = {frozenset(i): (f, fin) for i, f, fin in g.states()}
        for s, (f, fin) in states.items():
            if fin:
                assert f == 1
            for p, st, _ in placements(spec):
                t = s | {(p, st)}
                if t != s and t in states:
                    assert states[t][0] <= f


def test_a100_profiles_paper_sizes():
    # 1/7+5GB, 2/7+10GB, 3/7+20GB, 4/7+20GB, full; "1/7 Compute, 1/8 Memory"
    spec = load("a100-40gb")
    g = orc.Geometry(spec)
    assert g.compute == [1, 2, 3, 4, 7]
    assert g.mem == [5120, 10240, 20480, 20480, 40960]
    assert spec["total_memory_slots"] == 8 and g.compute[0] / 7 == 1 / 7 and g.mem[0] / g.full_mem == 1 / 8


def test_legality_example_paper_438():
    # (5GB, 5GB, 30GB-unallocated) + 20GB -> only (5,5,10 unalloc,20): 3g@4; the 4g (start 0 only) FAILs;
    # "(5GB, 5GB, 20GB, 10GB unallocated)" is illegal: nothing 20 GB starts at slot 2.
    g = orc.Geometry(load("a100-40gb"))
    s = [(0, 0), (0, 1)]
    assert g.allocate(s, 2) == 4
    assert g.allocate(s, 3) == -1
    assert g.fcr(s + [(2, 2)]) == 0  # not a valid state
    assert g.fcr(s + [(2, 4)]) > 0


def test_seven_5gb_and_halves():
    g = orc.Geometry(load("a100-40gb"))
    s = []
    starts = []
    for _ in range(7):  # PAPER.md:573 "creates seven 5gb partitions"
        st = g.allocate(s, 0)
        assert st >= 0
        starts.append(st)
        s.append((0, st))
    assert starts == [6, 5, 4, 3, 2, 1, 0]  # SURVEY.md §8(c) Alg 2 pin
    assert g.allocate(s, 0) == -1  # 8th memory slot unusable by a 1g (fully configured)
    # two 20 GB halves, 4/7 + 3/7 compute
    assert g.allocate([], 3) == 0
    assert g.allocate([(3, 0)], 2) == 4


def test_alg2_argmax_pins():
    g = orc.Geometry(load("a100-40gb"))
    assert g.allocate([], 0) == 6  # fcr 12 vs 6: the last slice is best
    assert g.allocate([], 1) == 4  # 6,6,6 tie -> highest start (R5)
    assert g.allocate([], 2) == 4  # 6 vs 3
    a30 = orc.Geometry(load("a30-24gb"))
    assert a30.allocate([], 1) == 2  # tie 2,2 -> highest start
    assert a30.allocate([(1, 2)], 0) == 1
    assert a30.allocate([(1, 2), (0, 1)], 0) == 0


def test_paper_534_example_recorded_discrepancy():
    # PAPER.md:534-537 prints 7 / 7 / 9 for the first, second and last 5 GB placement from s0. Under the vendor
    # table (R1) the counts are 6 / 6 / 12 (R4: not reproducible; recorded, not patched). The paper's ordering
    # (first = second < last) and its argmax (the last slice) hold.
    g = orc.Geometry(load("a100-40gb"))
    f = [g.fcr([(0, s)]) for s in range(7)]
    assert f == [6, 6, 6, 6, 6, 6, 12]
    assert f[0] == f[1] < f[6]


def test_alg2_equals_bruteforce_argmax_everywhere():
    # allocate_partition = brute-force argmax over enumerate_placements on every state x profile
    for name in ["a30-24gb", "a100-40gb", "a100-40gb-1g10"]:
        spec = load(name)
        g = orc.Geometry(spec)
        S, F, fcr = brute_tables(spec)
        Sset = set(S)
        for s in S:
            for p in range(len(spec["profiles"])):
                cands = [(fcr[s | {(p, st)}], st) for st in spec["profiles"][p]["starts"]
                         if (s | {(p, st)}) in Sset and (p, st) not in s]
                want = max(cands)[1] if cands else -1
                assert g.allocate(sorted(s), p) == want, (name, sorted(s), p)


def test_tight_fit_and_warp_folding():
    g = orc.Geometry(load("a100-40gb"))
    pol = orc.policy()
    assert g.tight_fit(3 * 1024, 0, pol) == 0  # SPEC.md:51 (A100, 3 GB) -> 5GB profile
    assert g.tight_fit(45 * 1024, 0, pol) == -1  # SPEC.md:53 NoFit
    assert g.tight_fit(20 * 1024, 0, pol) == 2  # 20 GB -> 3g (fewer compute), R6
    assert g.tight_fit(10 * 1024 + 1, 0, pol) == 2
    # warp folding (R30): W warps; capacity per slice 14 SMs * 64 warps = 896; full = 7*896 = 6272.
    fold = orc.policy(flags=orc.WARP_FOLD)
    W = 6272 + 1  # 2 waves on the full GPU; 3g (2688) -> 3 waves, 4g (3584) -> 2 waves
    assert g.tight_fit(1024, W, fold) == 3
    assert g.tight_fit(1024, W, pol) == 0  # folding off: memory only
    assert g.tight_fit(1024, 100, fold) == 0  # 1 wave everywhere


def test_geometry_validation_errors():
    spec = load("a100-40gb")
    bad = json.loads(json.dumps(spec))
    bad["profiles"][1]["starts"] = [7]  # 2-slot profile starting at slot 7 of 8
    with pytest.raises(ValueError):
        orc.Geometry(bad)


def test_reach_counts_reference_pins():
    # the brute-force Alg. 1 on occupancy masks (tests/bruteforce.py reach_counts, the reference of the device
    # mig_reachability) reproduces the instance-set enumeration's |S| / |F| and Appendix A on the vendor tables
    import bruteforce as bf

    for name, nS, nF in [("a30-24gb", 26, 5), ("a100-40gb", 298, 19), ("a100-40gb-1g10", 723, 78)]:
        spec = json.load(open(geom_path(name)))
        S, F, fcr = bf.reach_counts(spec["total_memory_slots"], bf.geometry_masks(spec))
        assert (S, F, fcr[0]) == (nS, nF, nF), name
    spec = json.load(open(geom_path("a100-40gb")))
    _, _, fcr = bf.reach_counts(8, bf.geometry_masks(spec))
    for line in open(os.path.join(GOLDEN_DIR, "a100_fcr_table.txt")):
        if line.startswith("#"):
            continue
        for tok in line.split():
            if ":" in tok:
                k, v = tok.split(":")
                assert fcr[int(k, 16)] == int(v), tok
    # binary-aligned slots (lengths 1, 2, 4, ..., n at aligned starts): |S| = f(n) = f(n/2)^2 + 1, f(1) = 2 and
    # |F| = g(n) = g(n/2)^2 + 1, g(1) = 1 (a block is one instance, or two independent halves)
    masks = [((1 << L) - 1) << s for L in (1, 2, 4, 8) for s in range(0, 8, L)]
    S, F, fcr = bf.reach_counts(8, masks)
    assert (S, F, fcr[0], fcr[255]) == (677, 26, 26, 1)


def test_oracle_reach_pins():
    # the oracle's literal Alg. 1 on placement masks (or_reach: every set of disjoint placements, finals, fcr =
    # finals containing the state) against the vendor tables' |S| / |F| / fcr(s0), Appendix A, the closed forms of
    # aligned power-of-two slots, and the independent pure-Python definition (tests/bruteforce.py) on random
    # geometries
    import bruteforce as bf

    for name, nS, nF in [("a30-24gb", 26, 5), ("a100-40gb", 298, 19), ("a100-40gb-1g10", 723, 78)]:
        spec = json.load(open(geom_path(name)))
        fcr, S, F = orc.reach(spec["total_memory_slots"], bf.geometry_masks(spec))
        assert (S, F, int(fcr[0])) == (nS, nF, nF), name
    spec = json.load(open(geom_path("a100-40gb")))
    fcr, _, _ = orc.reach(8, bf.geometry_masks(spec))
    for line in open(os.path.join(GOLDEN_DIR, "a100_fcr_table.txt")):
        if line.startswith("#"):
            continue
        for tok in line.split():
            if ":" in tok:
                k, v = tok.split(":")
                assert int(fcr[int(k, 16)]) == int(v), tok
    for n, S, F in [(8, 677, 26), (16, 458330, 677)]:
        masks = [((1 << L) - 1) << s for L in [1 << k for k in range(5)] if L <= n for s in range(0, n, L)]
        fcr, s_, f_ = orc.reach(n, masks)
        assert (s_, f_, int(fcr[0]), int(fcr[(1 << n) - 1])) == (S, F, F, 1)
    rng = np.random.default_rng(2)
    for _ in range(10):
        n = int(rng.integers(4, 10))
        masks = sorted({((1 << L) - 1) << s for L, s in
                        [(L, int(rng.integers(0, n - L + 1))) for L in rng.integers(1, min(n, 5) + 1, 3 * n)]})
        S, F, ref = bf.reach_counts(n, masks)
        fcr, s_, f_ = orc.reach(n, masks)
        assert (s_, f_) == (S, F) and fcr.tolist() == ref
