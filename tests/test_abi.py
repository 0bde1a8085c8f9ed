"""The drop-in C-ABI library without a GPU: it builds, loads, exports every
symbol include/kcore_b200.h declares, validates arguments like the reference
(std::invalid_argument before any work, fastk.cpp:58-59) and never falls back
to a CPU path."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT, _has_gpu

HEADER = os.path.join(ROOT, "include", "kcore_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(kc_[a-z0-9_]+)\s*\(", text)) - {"kc_inspector_fn"})


def test_header_is_plain_c():
    # compiles as C99 with no C++/torch types in any signature
    r = subprocess.run(["gcc", "-std=c99", "-fsyntax-only", "-x", "c", HEADER],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "torch" not in open(HEADER).read().lower().replace("no torch", "")


def test_library_exports_every_declared_symbol(kc):
    lib = kc.library_path()
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (kc_\w+)", out))
    decl = declared_functions()
    assert decl, "no declarations parsed"
    missing = [f for f in decl if f not in exported]
    assert not missing, missing
    assert set(kc.api.ABI_SYMBOLS) == set(decl)


def test_library_targets_sm100a_only(kc):
    out = subprocess.run(["cuobjdump", "--list-elf", kc.library_path()], capture_output=True,
                         text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_status_strings_and_defaults(kc):
    L = kc.load_library()
    assert L.kc_abi_version() == 1
    for s in range(9):
        assert L.kc_status_str(s) and L.kc_status_str(s) != b"unknown status"
    o = kc.api._Options()
    L.kc_default_options(C.byref(o))
    # FastKOptions defaults, include/kcore/fastk.hpp:12-22
    assert (o.threads, o.batch, o.extended_notify, o.hybrid_tail) == (16, 256, 1, 1)
    d = kc.FastKOptions()
    assert (d.threads, d.batch, d.extended_notify, d.hybrid_tail) == (16, 256, True, True)


def test_invalid_options_rejected_before_any_work(kc):
    # tests/test_fastk.cpp:142-145: zero threads or batch -> invalid_argument
    g = kc.Graph.from_edges(3, [(0, 1), (1, 2), (0, 2)])
    with pytest.raises(ValueError):
        kc.fastk_run(g, kc.FastKOptions(threads=0))
    with pytest.raises(ValueError):
        kc.fastk_run(g, kc.FastKOptions(batch=0))
    L = kc.load_library()
    v = g._view()
    o = kc.api._Options()
    L.kc_default_options(C.byref(o))
    o.threads = 0
    out = np.zeros(3, np.uint32)
    st = kc.api._Stats()
    assert L.kc_fastk_run(C.byref(v), C.byref(o), out.ctypes.data, C.byref(st)) == 1


def test_bad_views_rejected(kc):
    L = kc.load_library()
    h = C.c_void_p()
    assert L.kc_graph_upload(None, 0, C.byref(h)) == 1
    assert L.kc_graph_upload_ex(None, 0, 0, 99, C.byref(h)) == 1


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device path")
def test_no_cpu_fallback_without_device(kc):
    g = kc.Graph.from_edges(3, [(0, 1), (1, 2), (0, 2)])
    with pytest.raises(kc.KCError) as e:
        kc.fastk_run(g)
    assert e.value.status == 2  # KC_ERR_NO_DEVICE
    with pytest.raises(kc.KCError):
        kc.gen_config(1, 100, 1000)
    with pytest.raises(kc.KCError) as e:  # the edge-list loader has no host path either
        kc.load_edge_list("1 2\n")
    assert e.value.status == 2
