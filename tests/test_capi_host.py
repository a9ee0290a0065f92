"""libmig.so without a GPU: it loads, exports every entry point include/mig.h declares, its host-side geometry
tables (Alg. 1 fcr by occupancy mask, Alg. 2 placement) agree with the oracle's literal instance-set enumeration,
geometry validation names the offending field, and device calls fail loudly (no CPU fallback)."""
import ctypes as C
import json
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
