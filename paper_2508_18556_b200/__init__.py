"""paper_2508_18556_b200 — Python binding of libmig.so (include/mig.h).

Argument marshalling only: every step of the hot path (memory estimation, tight fit, Alg. 2 placement,
fusion/fission, OOM and early restart, event loop, metric reduction) runs in the sm_100a kernels of libmig.so.
PyTorch is used for device memory and streams. There is no CPU fallback: importing this package fails loudly if
libmig.so has not been built, and the device entry points fail without a CUDA device.

Names follow the C ABI: mig_geometry_load, mig_estimate_memory, mig_simulate, mig_simulate_host, ...
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmig.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python __graft_entry__.py` (no CPU fallback exists)")
_lib = C.CDLL(LIB_PATH)

MIG_BASELINE, MIG_STATIC, MIG_DYNAMIC, MIG_FUSION_FISSION, MIG_SCHEME_A = 0, 1, 2, 3, 4
MIG_EARLY_RESTART, MIG_WARP_FOLD, MIG_EWMA_REUSE, MIG_WAVE_TIME, MIG_PCIE_CONTENTION = 1, 2, 4, 8, 16
MIG_MAX_JOBS_PER_TRACE = 768
MIG_TRACES_NO_DYNAMIC = 1  # mig_traces.flags: no DYNAMIC-class job (the estimator pass is skipped)
MIG_NEVER = 0xFFFF
STATUS = {0: "MIG_OK", 1: "MIG_E_INVALID_ARG", 2: "MIG_E_IO", 3: "MIG_E_PARSE", 4: "MIG_E_VALIDATION",
          5: "MIG_E_CAPACITY", 6: "MIG_E_CUDA", 7: "MIG_E_UNSUPPORTED"}

RESULT_DTYPE = np.dtype([
    ("makespan", "<u4"), ("n_jobs", "<u4"), ("completed", "<u4"), ("rejected", "<u4"), ("failed", "<u4"),
    ("ooms", "<u4"), ("preempts", "<u4"), ("restarts", "<u4"), ("placements", "<u4"), ("waits", "<u4"),
    ("creates", "<u4"), ("destroys", "<u4"), ("energy_wticks", "<u8"), ("turnaround_sum", "<u8"),
    ("busy_slice_ticks", "<u8"), ("decision_hash", "<u8"), ("mem_mib_ticks", "<u8"), ("wasted_ticks", "<u8")])
ESTIMATE_DTYPE = np.dtype([
    ("req0_mib", "<u4"), ("pred_mib", "<u4"), ("conv_iter", "<u2"), ("n_levels", "<u2"), ("fe", "<u2", (6,)),
    ("phi", "<f8"), ("a", "<f8"), ("sigma", "<f8"), ("mem_fe", "<u4", (5,)), ("mem_conv", "<u4"),
    ("mem_T", "<u4"), ("pad", "<u4")])
TOTALS_FIELDS = ["n_traces", "n_jobs", "completed", "rejected", "failed", "ooms", "preempts", "restarts",
                 "placements", "waits", "creates", "destroys", "makespan_sum", "makespan_max", "energy_wticks",
                 "turnaround_sum", "busy_slice_ticks", "decision_hash_sum", "mem_mib_ticks", "wasted_ticks",
                 "error_flags", "reserved0", "reserved1", "reserved2"]
TOTALS_DTYPE = np.dtype([(f, "<u8") for f in TOTALS_FIELDS])
assert RESULT_DTYPE.itemsize == 96 and ESTIMATE_DTYPE.itemsize == 80 and TOTALS_DTYPE.itemsize == 192


class MigError(RuntimeError):
    pass


class mig_geometry_info(C.Structure):
    _fields_ = [("gpu_name", C.c_char * 64)] + [(n, C.c_uint32) for n in (
        "n_slots", "slot_mib", "n_compute", "n_profiles", "n_levels", "n_placements", "n_states", "n_finals",
        "fcr_s0", "full_mem_mib", "n_layout", "scheme_a", "idle_w", "w_per_slice")]


class mig_traces(C.Structure):
    _fields_ = [("jobs", C.c_void_p), ("jobs_ext", C.c_void_p), ("trace_off", C.c_void_p), ("n_traces", C.c_uint64),
                ("trace_id0", C.c_uint64), ("seed", C.c_uint64), ("n_jobs", C.c_uint64), ("max_jobs", C.c_uint32),
                ("flags", C.c_uint32), ("samples", C.c_void_p), ("sample_off", C.c_void_p),
                ("arrival", C.c_void_p)]


class mig_policy(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("flags", C.c_uint32), ("ctx_mib", C.c_uint32),
                ("reconfig_ticks", C.c_uint32), ("idle_w", C.c_uint32), ("w_per_slice", C.c_uint32),
                ("z", C.c_double), ("eps_num", C.c_uint32), ("eps_den", C.c_uint32), ("conv_k", C.c_uint32),
                ("min_n", C.c_uint32)]


_lib.mig_last_error.restype = C.c_char_p
_lib.mig_last_launch_count.restype = C.c_uint32
_lib.mig_release_scratch.restype = C.c_int
_lib.mig_geometry_load.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
_lib.mig_geometry_free.argtypes = [C.c_void_p]
_lib.mig_geometry_query.argtypes = [C.c_void_p, C.POINTER(mig_geometry_info)]
_lib.mig_geometry_profile.argtypes = [C.c_void_p, C.c_uint32, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                      C.POINTER(C.c_uint32), C.c_char_p]
_lib.mig_geometry_fcr.argtypes = [C.c_void_p, C.c_uint32, C.POINTER(C.c_uint32)]
_lib.mig_geometry_place.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(C.c_int32)]
_lib.mig_geometry_fusion.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                     C.POINTER(C.c_int32), C.POINTER(C.c_uint32)]
_lib.mig_estimate_memory.argtypes = [C.c_void_p, C.POINTER(mig_traces), C.POINTER(mig_policy), C.c_void_p,
                                     C.c_void_p]
_lib.mig_simulate.argtypes = [C.c_void_p, C.POINTER(mig_traces), C.POINTER(mig_policy), C.c_uint32, C.c_void_p,
                              C.c_void_p, C.c_void_p, C.c_void_p]
_lib.mig_simulate_host.argtypes = [C.c_void_p, C.POINTER(mig_traces), C.POINTER(mig_policy), C.c_uint32,
                                   C.c_void_p, C.c_void_p]


def _check(status):
    if status != 0:
        raise MigError(f"{STATUS.get(status, status)}: {_lib.mig_last_error().decode()}")


def mig_last_launch_count() -> int:
    return int(_lib.mig_last_launch_count())


class mig_reach_info(C.Structure):
    _fields_ = [("n_states", C.c_uint64), ("n_finals", C.c_uint64), ("fcr_s0", C.c_uint64)]


_lib.mig_reachability.argtypes = [C.c_uint32, C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p,
                                  C.POINTER(mig_reach_info), C.c_void_p]


def mig_reachability(n_slots: int, placement_masks, flags=True, stream=None):
    """Alg. 1 on the device (include/mig.h mig_reachability): returns (fcr uint32 CUDA tensor [2^n_slots],
    state flags uint8 CUDA tensor or None, info dict)."""
    import torch

    masks = np.ascontiguousarray(placement_masks, np.uint32)
    dev = torch.device("cuda", torch.cuda.current_device())
    fcr = torch.empty(1 << n_slots, dtype=torch.int32, device=dev)
    fl = torch.empty(1 << n_slots, dtype=torch.uint8, device=dev) if flags else None
    info = mig_reach_info()
    _check(_lib.mig_reachability(n_slots, masks.ctypes.data, len(masks), C.c_void_p(fcr.data_ptr()),
                                 None if fl is None else C.c_void_p(fl.data_ptr()), C.byref(info), _stream_ptr(stream)))
    return fcr, fl, {"n_states": info.n_states, "n_finals": info.n_finals, "fcr_s0": info.fcr_s0}


def mig_release_scratch() -> None:
    """Return the library's unused device scratch (its private pools) to the devices (include/mig.h)."""
    _check(_lib.mig_release_scratch())


class mig_kernel_time(C.Structure):
    _fields_ = [("name", C.c_char * 16), ("ms", C.c_double), ("launches", C.c_uint32), ("reserved", C.c_uint32)]


_lib.mig_timing_enable.argtypes = [C.c_int]
_lib.mig_timing_query.argtypes = [C.POINTER(mig_kernel_time), C.c_uint32, C.POINTER(C.c_uint32)]


def mig_timing_enable(on: bool = True) -> None:
    """Bracket this thread's kernel launches with CUDA events (include/mig.h: mig_timing_enable)."""
    _lib.mig_timing_enable(1 if on else 0)


def mig_timing_query() -> dict:
    """{kernel group name: (total ms, launches)} since the last enable/query (synchronises the events)."""
    buf = (mig_kernel_time * 32)()
    n = C.c_uint32(0)
    _check(_lib.mig_timing_query(buf, 32, C.byref(n)))
    return {buf[i].name.decode(): (buf[i].ms, int(buf[i].launches)) for i in range(min(n.value, 32))}


class Geometry:
    """A loaded geometry (opaque mig_geometry*), with its info and profile table."""

    def __init__(self, handle):
        self.h = handle
        info = mig_geometry_info()
        _check(_lib.mig_geometry_query(self.h, C.byref(info)))
        self.info = info
        self.name = info.gpu_name.decode()
        self.profiles = []
        for p in range(info.n_profiles):
            m, c, s = C.c_uint32(), C.c_uint32(), C.c_uint32()
            nm = C.create_string_buffer(32)
            _check(_lib.mig_geometry_profile(self.h, p, C.byref(m), C.byref(c), C.byref(s), nm))
            self.profiles.append(dict(name=nm.value.decode(), mem_mib=m.value, compute=c.value, slots=s.value))

    def __del__(self):
        if getattr(self, "h", None):
            _lib.mig_geometry_free(self.h)
            self.h = None


def mig_geometry_load(path_or_builtin: str) -> Geometry:
    h = C.c_void_p()
    _check(_lib.mig_geometry_load(path_or_builtin.encode(), C.byref(h)))
    return Geometry(h)


def mig_geometry_fcr(g: Geometry, occ: int) -> int:
    out = C.c_uint32()
    _check(_lib.mig_geometry_fcr(g.h, occ, C.byref(out)))
    return out.value


def mig_geometry_place(g: Geometry, occ: int, profile: int) -> int:
    out = C.c_int32()
    _check(_lib.mig_geometry_place(g.h, occ, profile, C.byref(out)))
    return out.value


def mig_geometry_fusion(g: Geometry, occ: int, starts: int, busy: int, profile: int):
    """Fusion/fission test hook (include/mig.h): (start or -1, destroyed-slot mask)."""
    st, dm = C.c_int32(), C.c_uint32()
    _check(_lib.mig_geometry_fusion(g.h, occ, starts, busy, profile, C.byref(st), C.byref(dm)))
    return st.value, dm.value


def policy(g: Geometry | None = None, kind=MIG_FUSION_FISSION, flags=0, ctx_mib=512, reconfig_ticks=500,
           idle_w=None, w_per_slice=None, z=2.326, eps_num=1, eps_den=100, conv_k=3, min_n=3) -> mig_policy:
    """A mig_policy; the power model defaults to the geometry's (idle_w, w_per_slice)."""
    if idle_w is None:
        idle_w = g.info.idle_w if g is not None else 30
    if w_per_slice is None:
        w_per_slice = g.info.w_per_slice if g is not None else 25
    return mig_policy(kind, flags, ctx_mib, reconfig_ticks, idle_w, w_per_slice, z, eps_num, eps_den, conv_k,
                      min_n)


class Traces:
    """Device-resident traces: keeps the tensors alive and carries the mig_traces descriptor."""

    def __init__(self, jobs, ext, trace_off, n_traces, seed=0, trace_id0=0, max_jobs=None, n_jobs=None,
                 samples=None, sample_off=None, arrival=None, flags=0):
        self.jobs, self.ext, self.trace_off = jobs, ext, trace_off
        self.arrival = arrival
        self.samples, self.sample_off = samples, sample_off
        self.n_traces = int(n_traces)
        self.n_jobs = int(jobs.shape[0]) if n_jobs is None else int(n_jobs)
        if max_jobs is None:
            if self.n_traces:
                max_jobs = int((trace_off[1:] - trace_off[:-1]).max().item())
            max_jobs = max(1, max_jobs or 1)
        self.max_jobs = int(max_jobs)
        self.desc = mig_traces(jobs.data_ptr() if self.n_jobs else None,
                               ext.data_ptr() if ext is not None else None, trace_off.data_ptr(), self.n_traces,
                               trace_id0, seed, self.n_jobs, self.max_jobs, flags,
                               None if samples is None else samples.data_ptr(),
                               None if sample_off is None else sample_off.data_ptr(),
                               None if arrival is None else arrival.data_ptr())


def traces_from_numpy(jobs, ext, trace_off, seed=0, trace_id0=0, device=None, max_jobs=None, samples=None,
                      sample_off=None, arrival=None) -> Traces:
    import torch

    dev = device or torch.device("cuda", torch.cuda.current_device())
    j = torch.from_numpy(np.ascontiguousarray(jobs, np.uint32).view(np.int32)).reshape(-1, 4).to(dev)
    e = None if ext is None else torch.from_numpy(np.ascontiguousarray(ext, np.uint32).view(np.int32)).reshape(-1, 4).to(dev)
    o = torch.from_numpy(np.ascontiguousarray(trace_off, np.uint64).view(np.int64)).to(dev)
    if max_jobs is None:
        lens = np.diff(np.asarray(trace_off, np.int64))
        max_jobs = max(1, int(lens.max())) if len(lens) else 1
    smp = soff = None
    if samples is not None:
        smp = torch.from_numpy(np.ascontiguousarray(samples, np.uint32).view(np.int32).reshape(-1, 2)).to(dev)
        soff = torch.from_numpy(np.ascontiguousarray(sample_off, np.uint64).view(np.int64)).to(dev)
    arr = None
    if arrival is not None:
        arr = torch.from_numpy(np.ascontiguousarray(arrival, np.uint32).view(np.int32)).to(dev)
    return Traces(j, e, o, len(trace_off) - 1, seed, trace_id0, max_jobs, samples=smp, sample_off=soff, arrival=arr)


def _stream_ptr(stream):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _policies(pols):
    if isinstance(pols, mig_policy):
        pols = [pols]
    return (mig_policy * len(pols))(*pols), len(pols)


def mig_estimate_memory(g: Geometry, tr: Traces, pol: mig_policy, out=None, stream=None):
    """Per-job estimates on the device. Returns a uint8 CUDA tensor [n_jobs, 80] (view with ESTIMATE_DTYPE)."""
    import torch

    if out is None:
        out = torch.empty((tr.n_jobs, 80), dtype=torch.uint8, device=tr.jobs.device)
    _check(_lib.mig_estimate_memory(g.h, C.byref(tr.desc), C.byref(pol), C.c_void_p(out.data_ptr()),
                                    _stream_ptr(stream)))
    return out


def mig_simulate(g: Geometry, tr: Traces, pols, est=None, out=None, totals=None, write_results=True, stream=None):
    """Simulate every trace under each policy on the device. Returns (results uint8 [n_traces*n_pol, 96] or None,
    totals uint8 [n_pol, 192]); view on the host with RESULT_DTYPE / TOTALS_DTYPE."""
    import torch

    parr, n = _policies(pols)
    dev = tr.jobs.device
    if out is None and write_results:
        out = torch.empty((tr.n_traces * n, 96), dtype=torch.uint8, device=dev)
    if totals is None:
        totals = torch.empty((n, 192), dtype=torch.uint8, device=dev)
    _check(_lib.mig_simulate(g.h, C.byref(tr.desc), parr, n,
                             None if est is None else C.c_void_p(est.data_ptr()),
                             None if out is None else C.c_void_p(out.data_ptr()), C.c_void_p(totals.data_ptr()),
                             _stream_ptr(stream)))
    return out, totals


def mig_simulate_host(g: Geometry, jobs, ext, trace_off, pols, seed=0, trace_id0=0, max_jobs=None, out=None,
                      totals=None, samples=None, sample_off=None, arrival=None, results=True):
    """HOST buffers in, HOST results out (page-locked numpy views recommended). Returns (results [n_traces, n_pol]
    RESULT_DTYPE, or None with results=False: only the per-policy totals come back, totals [n_pol] TOTALS_DTYPE)."""
    parr, n = _policies(pols)
    n_traces = len(trace_off) - 1
    if max_jobs is None:
        lens = np.diff(np.asarray(trace_off, np.int64))
        max_jobs = max(1, int(lens.max())) if len(lens) else 1
    if out is None and results:
        out = np.zeros((n_traces, n), RESULT_DTYPE)
    if totals is None:
        totals = np.zeros(n, TOTALS_DTYPE)
    if samples is not None:
        samples = np.ascontiguousarray(samples, np.uint32)
        sample_off = np.ascontiguousarray(sample_off, np.uint64)
    if arrival is not None:
        arrival = np.ascontiguousarray(arrival, np.uint32)
    desc = mig_traces(jobs.ctypes.data if len(jobs) else None, None if ext is None else ext.ctypes.data,
                      trace_off.ctypes.data, n_traces, trace_id0, seed, int(trace_off[-1] - trace_off[0]), max_jobs, 0,
                      None if samples is None else samples.ctypes.data,
                      None if sample_off is None else sample_off.ctypes.data,
                      None if arrival is None else arrival.ctypes.data)
    _check(_lib.mig_simulate_host(g.h, C.byref(desc), parr, n, None if out is None else out.ctypes.data,
                                  totals.ctypes.data))
    return out, totals


def results_numpy(res_tensor, n_pol):
    """Device results tensor -> numpy [n_traces, n_pol] RESULT_DTYPE."""
    a = res_tensor.cpu().numpy()
    return a.view(RESULT_DTYPE).reshape(-1, n_pol)


def totals_numpy(tot_tensor):
    return tot_tensor.cpu().numpy().view(TOTALS_DTYPE).reshape(-1)


def estimates_numpy(est_tensor):
    return est_tensor.cpu().numpy().view(ESTIMATE_DTYPE).reshape(-1)


def mig_debug_phys_div(y, q, out=None, stream=None):
    """Test hook (include/mig.h): floor(y * 2^16 / q) on the device the way k_estimate's fast path computes it.
    y, q: uint32 data in int32 CUDA tensors of equal length."""
    import torch

    if out is None:
        out = torch.empty_like(y)
    _check(_lib.mig_debug_phys_div(C.c_void_p(y.data_ptr()), C.c_void_p(q.data_ptr()), C.c_void_p(out.data_ptr()),
                                   y.numel(), _stream_ptr(stream)))
    return out


_lib.mig_debug_phys_div.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]


def mig_workspace_bytes(cublas_workspace_config: str, n_layers: int = 1) -> int:
    """Third-party workspace bytes from a CUBLAS_WORKSPACE_CONFIG string."""
    out = C.c_uint64()
    _check(_lib.mig_workspace_bytes(cublas_workspace_config.encode(), n_layers, C.byref(out)))
    return out.value


_lib.mig_workspace_bytes.argtypes = [C.c_char_p, C.c_uint32, C.POINTER(C.c_uint64)]
_lib.mig_samples_load_csv.argtypes = [C.c_char_p, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]


def mig_samples_load_csv(path: str):
    """One job's recorded per-iteration samples from a CSV trace file (include/mig.h): uint32 [n, 2] rows
    {req_mib, inv_reuse_q16}, the mig_traces.samples format."""
    n = C.c_uint64()
    _check(_lib.mig_samples_load_csv(str(path).encode(), None, 0, C.byref(n)))
    out = np.zeros((max(n.value, 1), 2), np.uint32)
    _check(_lib.mig_samples_load_csv(str(path).encode(), out.ctypes.data, n.value, C.byref(n)))
    return out[: n.value]


def samples_from_series(jobs, series):
    """Assemble mig_traces.samples / sample_off (host arrays) from per-job recorded series: series[k] = uint32
    [n_k, 2] samples of job k, or None for a job without samples. Argument marshalling only."""
    off = [0]
    parts = []
    for k in range(len(jobs)):
        s = series[k] if k < len(series) else None
        n = 0 if s is None else len(s)
        if n:
            parts.append(np.ascontiguousarray(s, np.uint32).reshape(-1, 2))
        off.append(off[-1] + n)
    smp = np.concatenate(parts) if parts else np.zeros((1, 2), np.uint32)
    return smp, np.array(off, np.uint64)
