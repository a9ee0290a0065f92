"""ctypes binding of the CPU oracle (oracle/oracle.cpp). TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference`` legs may import this module.
It never touches the CUDA path: the oracle is an independent, single-threaded C++ simulator written from
PAPER.md (see the header of oracle.cpp for the passage each part follows).
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

BASELINE, STATIC, DYNAMIC, FUSION_FISSION, SCHEME_A = 0, 1, 2, 3, 4
EARLY_RESTART, WARP_FOLD, EWMA_REUSE, WAVE_TIME, PCIE = 1, 2, 4, 8, 16

KIND_NAMES = {1: "REUSE", 2: "ALLOC", 3: "RECONF", 4: "WAIT", 5: "REJECT", 6: "COMPLETE", 7: "OOM", 8: "PREEMPT",
              9: "FAILED", 10: "PLACE_STATIC", 11: "PLACE_BASELINE", 12: "LAYOUT", 13: "PLACE_GROUP"}

RESULT_DTYPE = np.dtype([
    ("makespan", "<u4"), ("n_jobs", "<u4"), ("completed", "<u4"), ("rejected", "<u4"), ("failed", "<u4"),
    ("ooms", "<u4"), ("preempts", "<u4"), ("restarts", "<u4"), ("placements", "<u4"), ("waits", "<u4"),
    ("creates", "<u4"), ("destroys", "<u4"), ("energy_wticks", "<u8"), ("turnaround_sum", "<u8"),
    ("busy_slice_ticks", "<u8"), ("decision_hash", "<u8"), ("mem_mib_ticks", "<u8"), ("wasted_ticks", "<u8")])
ESTIMATE_DTYPE = np.dtype([
    ("req0_mib", "<u4"), ("pred_mib", "<u4"), ("conv_iter", "<u2"), ("n_levels", "<u2"), ("fe", "<u2", (6,)),
    ("phi", "<f8"), ("a", "<f8"), ("sigma", "<f8"), ("mem_fe", "<u4", (5,)), ("mem_conv", "<u4"),
    ("mem_T", "<u4"), ("pad", "<u4")])
assert RESULT_DTYPE.itemsize == 96 and ESTIMATE_DTYPE.itemsize == 80


class OrGeomDesc(C.Structure):
    _fields_ = [("n_slots", C.c_uint32), ("slot_mib", C.c_uint32), ("n_compute", C.c_uint32),
                ("sms_per_slice", C.c_uint32), ("warps_per_sm", C.c_uint32), ("n_prof", C.c_uint32),
                ("prof_compute", C.c_uint32 * 16), ("prof_len", C.c_uint32 * 16), ("prof_nstart", C.c_uint32 * 16),
                ("prof_start", (C.c_uint32 * 8) * 16), ("n_layout", C.c_uint32), ("layout_prof", C.c_uint32 * 8),
                ("layout_start", C.c_uint32 * 8), ("n_alay", C.c_uint32 * 8), ("alay_prof", (C.c_uint32 * 8) * 8),
                ("alay_start", (C.c_uint32 * 8) * 8)]


class OrPolicy(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("flags", C.c_uint32), ("ctx_mib", C.c_uint32),
                ("reconfig_ticks", C.c_uint32), ("idle_w", C.c_uint32), ("w_per_slice", C.c_uint32),
                ("z", C.c_double), ("eps_num", C.c_uint32), ("eps_den", C.c_uint32), ("conv_k", C.c_uint32),
                ("min_n", C.c_uint32)]


def policy(kind=FUSION_FISSION, flags=0, ctx_mib=512, reconfig_ticks=500, idle_w=30, w_per_slice=25, z=2.326,
           eps_num=1, eps_den=100, conv_k=3, min_n=3) -> OrPolicy:
    if min_n < 3:
        raise ValueError("min_n must be >= 3 (sigma needs n-2 >= 1)")
    return OrPolicy(kind, flags, ctx_mib, reconfig_ticks, idle_w, w_per_slice, z, eps_num, eps_den, conv_k, min_n)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        L.or_last_error.restype = C.c_char_p
        L.or_geometry_new.restype = C.c_void_p
        L.or_geometry_new.argtypes = [C.POINTER(OrGeomDesc)]
        L.or_geometry_free.argtypes = [C.c_void_p]
        L.or_geometry_counts.argtypes = [C.c_void_p] + [C.POINTER(C.c_uint32)] * 3
        L.or_geometry_state.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint32),
                                        C.POINTER(C.c_int32)]
        L.or_state_fcr.restype = C.c_uint32
        L.or_state_fcr.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32]
        L.or_allocate.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32]
        L.or_tight_fit.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(OrPolicy)]
        L.or_reach.argtypes = [C.c_uint32, C.c_void_p, C.c_uint32, C.c_void_p, C.POINTER(C.c_uint64),
                               C.POINTER(C.c_uint64)]
        L.or_predict_series.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.POINTER(OrPolicy), C.c_uint32,
                                        C.c_void_p]
        L.or_fit_once.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(OrPolicy), C.c_uint32,
                                  C.POINTER(C.c_int64)] + [C.POINTER(C.c_double)] * 3
        L.or_estimate.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                                  C.c_uint64, C.POINTER(OrPolicy), C.c_void_p, C.c_void_p, C.c_void_p]
        L.or_simulate.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                                  C.c_uint64, C.c_uint64, C.POINTER(OrPolicy), C.c_uint32, C.c_void_p, C.c_void_p,
                                  C.c_uint64, C.POINTER(C.c_uint64), C.c_void_p, C.c_void_p, C.c_void_p]
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Geometry:
    """Oracle geometry: Alg. 1 run literally over instance sets."""

    def __init__(self, spec: dict | str):
        if isinstance(spec, str):
            with open(spec) as f:
                spec = json.load(f)
        self.spec = spec
        d = OrGeomDesc()
        d.n_slots = spec["total_memory_slots"]
        d.slot_mib = spec["slot_mib"]
        d.n_compute = spec["total_compute_slices"]
        d.sms_per_slice = spec.get("sms_per_slice", 14)
        d.warps_per_sm = spec.get("warps_per_sm", 64)
        profs = spec["profiles"]
        d.n_prof = len(profs)
        self.names = [p["name"] for p in profs]
        for i, p in enumerate(profs):
            d.prof_compute[i] = p["compute_slices"]
            d.prof_len[i] = p["memory_slots"]
            d.prof_nstart[i] = len(p["starts"])
            for k, s in enumerate(p["starts"]):
                d.prof_start[i][k] = s
        lay = spec.get("static_layout", [])
        d.n_layout = len(lay)
        for i, (name, st) in enumerate(lay):
            d.layout_prof[i] = self.names.index(name)
            d.layout_start[i] = st
        mems = sorted({p["memory_slots"] * spec["slot_mib"] for p in profs})
        for entry in spec.get("scheme_a_layouts", []):
            lvl = mems.index(entry["memory_mib"])
            d.n_alay[lvl] = len(entry["slices"])
            for i, (name, st) in enumerate(entry["slices"]):
                d.alay_prof[lvl][i] = self.names.index(name)
                d.alay_start[lvl][i] = st
        self.desc = d
        h = lib().or_geometry_new(C.byref(d))
        if not h:
            raise ValueError(lib().or_last_error().decode())
        self.h = h
        self.mem = [p["memory_slots"] * spec["slot_mib"] for p in profs]
        self.compute = [p["compute_slices"] for p in profs]
        self.full_mem = spec["total_memory_slots"] * spec["slot_mib"]

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.or_geometry_free(self.h)
            self.h = None

    def counts(self):
        a, b, c = C.c_uint32(), C.c_uint32(), C.c_uint32()
        lib().or_geometry_counts(self.h, C.byref(a), C.byref(b), C.byref(c))
        return a.value, b.value, c.value

    def states(self):
        """All valid states: list of (instances [(prof, start)], fcr, is_final)."""
        n, _, _ = self.counts()
        out = []
        prof = np.zeros(8, np.uint32)
        start = np.zeros(8, np.uint32)
        for i in range(n):
            f, fin = C.c_uint32(), C.c_int32()
            k = lib().or_geometry_state(self.h, i, _ptr(prof), _ptr(start), C.byref(f), C.byref(fin))
            out.append(([(int(prof[j]), int(start[j])) for j in range(k)], f.value, bool(fin.value)))
        return out

    @staticmethod
    def _arrs(instances):
        prof = np.array([p for p, _ in instances] + [0], np.uint32)
        start = np.array([s for _, s in instances] + [0], np.uint32)
        return prof, start

    def fcr(self, instances):
        prof, start = self._arrs(instances)
        return lib().or_state_fcr(self.h, _ptr(prof), _ptr(start), len(instances))

    def allocate(self, instances, prof_idx):
        prof, start = self._arrs(instances)
        return lib().or_allocate(self.h, _ptr(prof), _ptr(start), len(instances), prof_idx)

    def tight_fit(self, req, warps=0, pol=None):
        pol = pol or policy()
        return lib().or_tight_fit(self.h, req, warps, C.byref(pol))


def predict_series(y, q, pol=None, ws=0):
    """Alg. 3 over an explicit series (y MiB, q Q16). Returns a numpy record of ESTIMATE_DTYPE."""
    pol = pol or policy(ctx_mib=0)
    y = np.ascontiguousarray(y, np.uint32)
    q = np.ascontiguousarray(q, np.uint32)
    out = np.zeros(1, ESTIMATE_DTYPE)
    lib().or_predict_series(_ptr(y), _ptr(q), len(y), C.byref(pol), ws, _ptr(out))
    return out[0]


def reach(n_slots, masks):
    """Alg. 1 by its literal definition for a slot geometry of placement masks (oracle.cpp or_reach): returns
    (fcr per occupancy, uint32 [2^n_slots]; |S|; |F|)."""
    m = np.ascontiguousarray(masks, np.uint32)
    out = np.zeros(1 << n_slots, np.uint32)
    ns, nf = C.c_uint64(), C.c_uint64()
    rc = lib().or_reach(n_slots, _ptr(m), len(m), _ptr(out), C.byref(ns), C.byref(nf))
    if rc != 0:
        raise RuntimeError(f"or_reach failed ({rc})")
    return out, ns.value, nf.value


def fit_once(y, q, T, pol=None, ws=0):
    pol = pol or policy(ctx_mib=0)
    y = np.ascontiguousarray(y, np.uint32)
    q = np.ascontiguousarray(q, np.uint32)
    P, phi, a, s = C.c_int64(), C.c_double(), C.c_double(), C.c_double()
    lib().or_fit_once(_ptr(y), _ptr(q), len(y), T, C.byref(pol), ws, C.byref(P), C.byref(phi), C.byref(a),
                      C.byref(s))
    return P.value, phi.value, a.value, s.value


def _samples(samples, sample_off):
    if samples is None:
        return None, None
    return np.ascontiguousarray(samples, np.uint32), np.ascontiguousarray(sample_off, np.uint64)


def estimate(geom: Geometry, jobs, ext, trace_off, pol, seed=0, trace_id0=0, samples=None, sample_off=None):
    n_traces = len(trace_off) - 1
    out = np.zeros(int(trace_off[-1]), ESTIMATE_DTYPE)
    jobs = np.ascontiguousarray(jobs, np.uint32)
    ext = None if ext is None else np.ascontiguousarray(ext, np.uint32)
    off = np.ascontiguousarray(trace_off, np.uint64)
    smp, soff = _samples(samples, sample_off)
    lib().or_estimate(geom.h, _ptr(jobs), _ptr(ext), _ptr(off), n_traces, trace_id0, seed, C.byref(pol), _ptr(out),
                      _ptr(smp), _ptr(soff))
    return out


def simulate(geom: Geometry, jobs, ext, trace_off, pols, seed=0, trace_id0=0, t0=0, t1=None, records=False,
             samples=None, sample_off=None, arrival=None):
    """Run the oracle on traces [t0, t1). Returns results[(t1-t0), n_pol] (and the record list if records).
    arrival: per-job arrival ticks (reading R40) or None (batch: all at t = 0)."""
    if not isinstance(pols, (list, tuple)):
        pols = [pols]
    n_traces = len(trace_off) - 1
    t1 = n_traces if t1 is None else t1
    parr = (OrPolicy * len(pols))(*pols)
    out = np.zeros((t1 - t0, len(pols)), RESULT_DTYPE)
    jobs = np.ascontiguousarray(jobs, np.uint32)
    ext = None if ext is None else np.ascontiguousarray(ext, np.uint32)
    off = np.ascontiguousarray(trace_off, np.uint64)
    rec = None
    rec_n = C.c_uint64(0)
    if records:
        assert t1 - t0 == 1 and len(pols) == 1
        rec = np.zeros(1 << 16, np.uint64)
    smp, soff = _samples(samples, sample_off)
    rc = lib().or_simulate(geom.h, _ptr(jobs), _ptr(ext), _ptr(off), t0, t1, trace_id0, seed, parr, len(pols),
                           _ptr(out), _ptr(rec), 0 if rec is None else len(rec), C.byref(rec_n), _ptr(smp),
                           _ptr(soff), _ptr(None if arrival is None else np.ascontiguousarray(arrival, np.uint32)))
    if rc != 0:
        raise RuntimeError(lib().or_last_error().decode())
    if records:
        return out, [decode_record(int(r)) for r in rec[: rec_n.value]]
    return out


def decode_record(r: int):
    return dict(tick=r >> 32, job=(r >> 16) & 0xFFFF, kind=KIND_NAMES.get((r >> 12) & 0xF, "?"),
                start=(r >> 8) & 0xF, profile=(r >> 4) & 0xF, n_destroyed=r & 0xF)
