"""Python binding of the seeded trace generator (tracegen.h / libtracegen.so). Input generation only.

Host generation returns numpy arrays in the trace format of tracegen.h; device generation fills torch CUDA tensors
(used by bench.py and the GPU tests so 10^6..10^8-trace inputs never cross PCIe).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtracegen.so")

# Config -> geometry name; cfg 1 is the fixed hand-worked A30 trace (tests/golden/config1_w.json).
CONFIG_GEOMETRY = {1: "a30-24gb", 2: "a100-40gb", 3: "a100-80gb", 4: "h100-80gb", 5: "a100-40gb"}
CONFIG_TRACES = {1: 1, 2: 1_000_000, 3: 1_000_000, 4: 10_000_000, 5: 100_000_000}
# Configs whose generator emits DYNAMIC-class jobs (tracegen.h tg_gen_trace: config 2 is Rodinia STATIC only); the
# others let a caller pass mig_traces.flags = MIG_TRACES_NO_DYNAMIC.
CONFIG_HAS_DYNAMIC = {1: False, 2: False, 3: True, 4: True, 5: True}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        L.tg_cfg_jobs_per_trace.restype = C.c_uint32
        L.tg_cfg_jobs_per_trace.argtypes = [C.c_uint32]
        L.tg_cfg_has_ext.restype = C.c_uint32
        L.tg_cfg_has_ext.argtypes = [C.c_uint32]
        L.tg_cfg_seed.restype = C.c_uint64
        L.tg_cfg_seed.argtypes = [C.c_uint32]
        L.tg_generate_host.argtypes = [C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p,
                                       C.c_void_p]
        L.tg_dyn_samples_host.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_void_p, C.c_void_p, C.c_uint32,
                                          C.c_void_p, C.c_void_p]
        L.tg_dyn_samples_host_fast.argtypes = L.tg_dyn_samples_host.argtypes
        L.tg_generate_device.argtypes = [C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_void_p]
        _lib = L
    return _lib


def seed_of(cfg: int) -> int:
    return int(lib().tg_cfg_seed(cfg))


def jobs_per_trace(cfg: int) -> int:
    return int(lib().tg_cfg_jobs_per_trace(cfg))


def has_ext(cfg: int) -> bool:
    return bool(lib().tg_cfg_has_ext(cfg))


def generate_host(cfg: int, n_traces: int, trace_id0: int = 0, seed: int | None = None, out=None):
    """Generate traces [trace_id0, trace_id0+n) on the host. Returns (jobs[n*J,4] u32, ext or None, trace_off u64).

    ``out`` may supply preallocated (e.g. pinned) arrays (jobs, ext, trace_off)."""
    seed = seed_of(cfg) if seed is None else seed
    J = jobs_per_trace(cfg)
    if J == 0:
        raise ValueError(f"config {cfg} has no generator")
    if out is None:
        jobs = np.zeros((n_traces * J, 4), np.uint32)
        ext = np.zeros((n_traces * J, 4), np.uint32) if has_ext(cfg) else None
        off = np.zeros(n_traces + 1, np.uint64)
    else:
        jobs, ext, off = out
    rc = lib().tg_generate_host(cfg, seed, trace_id0, n_traces, jobs.ctypes.data_as(C.c_void_p),
                                None if ext is None else ext.ctypes.data_as(C.c_void_p),
                                off.ctypes.data_as(C.c_void_p))
    if rc != 0:
        raise RuntimeError(f"tg_generate_host failed ({rc})")
    return jobs, ext, off


def generate_device(cfg: int, n_traces: int, trace_id0: int = 0, seed: int | None = None, device=None,
                    stream=None):
    """Generate traces on the GPU into torch uint32/int64 tensors (jobs[n*J,4], ext[n*J,4] or None, off[n+1])."""
    import torch

    seed = seed_of(cfg) if seed is None else seed
    J = jobs_per_trace(cfg)
    dev = device or torch.device("cuda", torch.cuda.current_device())
    jobs = torch.empty((n_traces * J, 4), dtype=torch.int32, device=dev)
    ext = torch.empty((n_traces * J, 4), dtype=torch.int32, device=dev) if has_ext(cfg) else None
    off = torch.empty(n_traces + 1, dtype=torch.int64, device=dev)
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    rc = lib().tg_generate_device(cfg, seed, trace_id0, n_traces, C.c_void_p(jobs.data_ptr()),
                                  None if ext is None else C.c_void_p(ext.data_ptr()), C.c_void_p(off.data_ptr()),
                                  C.c_void_p(s.cuda_stream))
    if rc != 0:
        raise RuntimeError(f"tg_generate_device failed ({rc})")
    return jobs, ext, off


def dyn_samples(seed: int, trace_id: int, job_idx: int, job, ext, T: int, fast=False):
    """Per-iteration samples (y MiB, q Q16), i = 1..T, of one dynamic job record (fast: tg_dyn_sample_fast)."""
    job = np.ascontiguousarray(job, np.uint32)
    ext = np.ascontiguousarray(ext, np.uint32)
    y = np.zeros(T, np.uint32)
    q = np.zeros(T, np.uint32)
    fn = lib().tg_dyn_samples_host_fast if fast else lib().tg_dyn_samples_host
    fn(seed, trace_id, job_idx, job.ctypes.data_as(C.c_void_p),
                              ext.ctypes.data_as(C.c_void_p), T, y.ctypes.data_as(C.c_void_p),
                              q.ctypes.data_as(C.c_void_p))
    return y, q


def pack_job(x, y, iters, cls, ticks, ws=0, warps=0, slope_q8=0, sigma=0, qslope=0, xfer=0):
    """One job record + ext record in the tracegen.h format (for hand-written fixtures). xfer: PCIe transfer
    fraction of an iteration in 1/256 (record bits 24-31, reading R39)."""
    return ([x, y, (iters & 0xFFFF) | (cls << 16) | ((xfer & 0xFF) << 24), ticks],
            [ws, warps, slope_q8, (sigma & 0xFFFF) | (qslope << 16)])


def pack_traces(traces):
    """traces: list of lists of (job4, ext4) -> (jobs, ext, trace_off) numpy arrays."""
    jobs, ext, off = [], [], [0]
    for tr in traces:
        for j, e in tr:
            jobs.append(j)
            ext.append(e)
        off.append(len(jobs))
    J = np.array(jobs, np.uint32).reshape(-1, 4)
    E = np.array(ext, np.uint32).reshape(-1, 4)
    return J, E, np.array(off, np.uint64)


def explicit_samples(jobs, ext, trace_off, seed, trace_id0=0):
    """Materialise the per-iteration samples of every DYNAMIC job as a recorded series: (samples u32 [S, 2],
    sample_off u64 [n_jobs + 1]) aligned with the job records (non-dynamic jobs get none)."""
    n_traces = len(trace_off) - 1
    chunks, off = [], [0]
    for t in range(n_traces):
        for j in range(int(trace_off[t]), int(trace_off[t + 1])):
            cls = (int(jobs[j, 2]) >> 16) & 0xFF
            T = int(jobs[j, 2]) & 0xFFFF
            if cls == 2 and T > 0:
                y, q = dyn_samples(seed, trace_id0 + t, j - int(trace_off[t]), jobs[j], ext[j], T)
                chunks.append(np.stack([y, q], axis=1))
                off.append(off[-1] + T)
            else:
                off.append(off[-1])
    smp = np.concatenate(chunks).astype(np.uint32) if chunks else np.zeros((1, 2), np.uint32)
    return smp, np.array(off, np.uint64)
