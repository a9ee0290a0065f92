"""libmig.so without a GPU: it loads, exports every entry point include/mig.h declares, its host-side geometry
tables (Alg. 1 fcr by occupancy mask, Alg. 2 placement) agree with the oracle's literal instance-set enumeration,
geometry validation names the offending field, and device calls fail loudly (no CPU fallback)."""
import ctypes as C
import json

import numpy as np
import os
import re

import pytest
import torch

from conftest import ROOT, geom_path
from oracle import oracle as orc

import paper_2508_18556_b200 as mig

GEOMS = ["a30-24gb", "a100-40gb", "a100-40gb-1g10", "a100-80gb", "h100-80gb", "b200-180gb"]


def test_exports_every_declared_symbol():
    with open(os.path.join(ROOT, "include", "mig.h")) as f:
        hdr = f.read()
    names = set(re.findall(r"^\s*(?:mig_status|void|const char\*|uint32_t)\s+(mig_\w+)\s*\(", hdr, re.M))
    assert {"mig_geometry_load", "mig_estimate_memory", "mig_simulate", "mig_simulate_host"} <= names
    lib = C.CDLL(mig.LIB_PATH)
    for n in sorted(names):
        assert hasattr(lib, n), n


@pytest.mark.parametrize("name", GEOMS)
def test_geometry_tables_match_oracle(name):
    g = mig.mig_geometry_load(f"builtin:{name}")
    og = orc.Geometry(geom_path(name))
    nS, nF, nP = og.counts()
    info = g.info
    assert (info.n_states, info.n_finals, info.n_placements, info.fcr_s0) == (nS, nF, nP, nF)
    spec = json.load(open(geom_path(name)))
    masks = {}
    for inst, f, _ in og.states():
        m = 0
        for p, s in inst:
            m |= ((1 << spec["profiles"][p]["memory_slots"]) - 1) << s
        masks[m] = f
        # Alg. 2 on the same state: the library's mask-indexed placement equals the oracle's
        for prof in range(len(spec["profiles"])):
            assert mig.mig_geometry_place(g, m, prof) == og.allocate(inst, prof), (name, inst, prof)
    for m in range(1 << spec["total_memory_slots"]):
        assert mig.mig_geometry_fcr(g, m) == masks.get(m, 0)
    assert [p["mem_mib"] for p in g.profiles] == og.mem
    assert [p["compute"] for p in g.profiles] == og.compute


def test_geometry_validation_names_field(tmp_path):
    spec = json.load(open(geom_path("a100-40gb")))
    bad = json.loads(json.dumps(spec))
    bad["profiles"][1]["starts"] = [7]
    p = tmp_path / "bad.json"
    p.write_text(json.dumps(bad))
    with pytest.raises(mig.MigError, match=r"MIG_E_VALIDATION: profiles\[1\]\.starts\[0\]"):
        mig.mig_geometry_load(str(p))
    p.write_text("{\"total_memory_slots\": 8,")
    with pytest.raises(mig.MigError, match="MIG_E_PARSE"):
        mig.mig_geometry_load(str(p))
    with pytest.raises(mig.MigError, match="MIG_E_IO"):
        mig.mig_geometry_load(str(tmp_path / "missing.json"))
    unsorted = json.loads(json.dumps(spec))
    unsorted["profiles"][0], unsorted["profiles"][1] = unsorted["profiles"][1], unsorted["profiles"][0]
    p.write_text(json.dumps(unsorted))
    with pytest.raises(mig.MigError, match="sorted"):
        mig.mig_geometry_load(str(p))


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_device_calls_fail_loudly_without_gpu():
    g = mig.mig_geometry_load("builtin:a30-24gb")
    buf = (C.c_uint32 * 8)()
    off = (C.c_uint64 * 2)(0, 1)
    desc = mig.mig_traces(C.addressof(buf), None, C.addressof(off), 1, 0, 0, 1, 1, 0)
    pol = mig.policy(g)
    rc = mig._lib.mig_simulate(g.h, C.byref(desc), C.byref(pol), 1, None, None, None, None)
    assert rc == 6 and "no CUDA device" in mig._lib.mig_last_error().decode()
    y = (C.c_uint32 * 4)(1, 2, 3, 4)
    rc = mig._lib.mig_debug_phys_div(C.addressof(y), C.addressof(y), C.addressof(y), 4, None)
    assert rc == 6  # MIG_E_CUDA: the kernel cannot launch without a GPU (no host fallback)
    assert mig._lib.mig_debug_phys_div(None, None, None, 4, None) == 1  # MIG_E_INVALID_ARG


def test_workspace_parser_spec_examples():
    # PAPER.md:358-362 (CUBLAS_WORKSPACE_CONFIG); SPEC.md:234-236 worked values
    assert mig.mig_workspace_bytes(":4096:8", 1) == 33_554_432
    assert mig.mig_workspace_bytes("", 10) == 0
    assert mig.mig_workspace_bytes(":4096:2,:16:8", 3) == 3 * (4096 * 1024 * 2 + 16 * 1024 * 8) == 25_559_040
    for bad in [":4096", "4096:8", ":4096:8,", ":a:8", ":4096:8;"]:
        with pytest.raises(mig.MigError, match="MIG_E_PARSE"):
            mig.mig_workspace_bytes(bad, 1)


def test_timing_hook_without_launches():
    mig.mig_timing_enable(True)
    assert mig.mig_timing_query() == {}
    mig.mig_timing_enable(False)


@pytest.mark.parametrize("name", ["a30-24gb", "a100-40gb", "a100-40gb-1g10", "b200-180gb"])
def test_fusion_table_matches_literal_r8(name):
    """The slot-level fusion/fission answers the lane kernel reads (mig_geometry_fusion) against reading R8 evaluated
    literally on instance sets: for every valid state of the oracle's Alg. 1 enumeration, every
    set of busy instances (all subsets up to 5 instances, 24 seeded ones beyond) and every profile, the placements
    that overlap >= 1 instance and only idle ones; destroy the overlapped, create the placement; best by
    (fcr(result) from the oracle, -#destroyed, start)."""
    import numpy as np

    g = mig.mig_geometry_load(f"builtin:{name}")
    og = orc.Geometry(geom_path(name))
    spec = json.load(open(geom_path(name)))
    lens = [p["memory_slots"] for p in spec["profiles"]]
    starts = [p["starts"] for p in spec["profiles"]]
    rng = np.random.default_rng(11)
    n_checked = n_found = 0
    for inst, _, _ in og.states():
        masks = [((1 << lens[p]) - 1) << s for p, s in inst]
        occ = sum(masks)
        sm = sum(1 << s for _, s in inst)
        k = len(inst)
        subsets = range(1 << k) if k <= 5 else [int(x) for x in rng.integers(0, 1 << k, 24)]
        for bs in subsets:
            busy = sum(masks[i] for i in range(k) if (bs >> i) & 1)
            for p in range(len(lens)):
                best = None
                for s in starts[p]:
                    qm = ((1 << lens[p]) - 1) << s
                    over = [i for i in range(k) if masks[i] & qm]
                    if not over or any((bs >> i) & 1 for i in over):
                        continue
                    rest = [inst[i] for i in range(k) if i not in over] + [(p, s)]
                    key = (og.fcr(rest), -len(over), s)
                    if best is None or key > best[0]:
                        best = (key, sum(masks[i] for i in over))
                got = mig.mig_geometry_fusion(g, occ, sm, busy, p)
                want = (-1, 0) if best is None else (best[0][2], best[1])
                assert got == want, (inst, bs, p, got, want)
                n_checked += 1
                n_found += best is not None
    assert n_found > 0 and n_checked > 100


def test_scheme_a_rejects_arrival_streams():
    """Scheme A groups the whole queue at t = 0 (R38): with arrival ticks (R40) the call is an argument error."""
    from tracegen import tracegen as tg

    jobs, ext, off = tg.pack_traces([[tg.pack_job(4096, 4096, 1, 0, 10)]])
    g = mig.mig_geometry_load("builtin:a100-40gb")
    with pytest.raises(mig.MigError, match="INVALID_ARG"):
        mig.mig_simulate_host(g, jobs, ext, off, [mig.policy(g, kind=4)], arrival=np.zeros(1, np.uint32))


def _build_c_example(tmp_path):
    import subprocess

    exe = tmp_path / "c_api_example"
    lib_dir = os.path.dirname(mig.LIB_PATH)
    subprocess.run(["gcc", "-std=c11", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "c_api_example.c"), "-L", lib_dir, "-lmig",
                    f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    return subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)


def test_c_example_builds_against_the_header_and_library(tmp_path):
    """examples/c_api_example.c compiles with -Wall -Werror against include/mig.h and links libmig.so; without a
    GPU it fails loudly (MIG_E_CUDA, exit 2), never silently computing on the CPU."""
    r = _build_c_example(tmp_path)
    assert (r.returncode == 0 and "FUSION_FISSION" in r.stdout) or (r.returncode == 2 and "no CUDA device" in r.stderr)


@pytest.mark.gpu
def test_c_example_reproduces_example_w(tmp_path):
    """The plain-C caller gets example W's hand-derived results (tests/golden/config1_w.json)."""
    r = _build_c_example(tmp_path)
    assert r.returncode == 0, r.stderr
    got = {ln.split()[0]: ln.split() for ln in r.stdout.strip().splitlines()}
    assert got["BASELINE"][2] == "450" and got["STATIC"][2] == "210"
    assert got["DYNAMIC"][2] == "220" and got["FUSION_FISSION"][2] == "220"
    assert got["FUSION_FISSION"][12] == "27100" and got["BASELINE"][12] == "58500"


def test_samples_load_csv(tmp_path):
    # the recorded-trace loader (include/mig.h mig_samples_load_csv, SPEC.md S:260 format): bytes -> MiB rounded up,
    # reuse_ratio -> inverse reuse in Q16 (round(65536 / r)); iterations must be 1, 2, 3, ...
    import paper_2508_18556_b200 as mig

    p = tmp_path / "job.csv"
    p.write_text("iteration,requested_bytes,reuse_ratio\n1,1048576,1.0\n2,1048577,0.5\n3,3145728,0.8\n\n")
    s = mig.mig_samples_load_csv(str(p))
    assert s.tolist() == [[1, 65536], [2, 131072], [3, 81920]]
    for body, why in [("iteration,bytes,reuse_ratio\n1,1,1\n", "header"), ("iteration,requested_bytes,reuse_ratio\n2,1,1\n", "order"),
                      ("iteration,requested_bytes,reuse_ratio\n1,x,1\n", "requested_bytes"),
                      ("iteration,requested_bytes,reuse_ratio\n1,1,0\n", "reuse_ratio")]:
        p.write_text(body)
        with pytest.raises(mig.MigError, match="MIG_E_PARSE"):
            mig.mig_samples_load_csv(str(p))
    with pytest.raises(mig.MigError, match="MIG_E_IO"):
        mig.mig_samples_load_csv(str(tmp_path / "missing.csv"))
