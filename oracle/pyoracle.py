"""ctypes front-end for oracle/liboracle.so (our C restatement) and
oracle/_ref/libkcore_ref.so (the unmodified reference, compiled from
/root/reference by oracle/Makefile).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs.  The product never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libkcore_ref.so")
REF_SRC = "/root/reference/proj"

_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


def build(ref: bool = True) -> None:
    """Compile liboracle.so (and the reference when its sources are mounted)."""
    targets = ["oracle"]
    if ref and os.path.isdir(REF_SRC):
        targets += ["ref", "ref_nofastk"]
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


class Stats(C.Structure):
    """kco_stats (oracle/kc_oracle.c) — RunReport counters + work counters."""
    _fields_ = [(k, C.c_uint64) for k in (
        "iterations", "messages_sent", "messages_drained", "tail_pops",
        "e_scan", "notify_scan", "drops")]

    def as_dict(self) -> dict:
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


class RefStats(C.Structure):
    """RunReport counters from the reference (include/kcore/report.hpp:17-23)."""
    _fields_ = [(k, C.c_uint64) for k in (
        "iterations", "messages_sent", "messages_drained", "tail_pops")]

    def as_dict(self) -> dict:
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build(ref=False)
        L = C.CDLL(LIB_PATH)
        L.kco_rng_at.restype = C.c_uint64
        L.kco_rng_at.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.kco_perm_bits.restype = C.c_uint32
        L.kco_perm_bits.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64]
        L.kco_gen_er.argtypes = [C.c_uint32, C.c_uint64, C.c_uint64, _u32p]
        L.kco_gen_grid.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, _u32p]
        L.kco_gen_rmat.argtypes = [C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                   C.c_uint64, _u32p]
        L.kco_chunglu_weights.restype = C.c_double
        L.kco_chunglu_weights.argtypes = [C.c_uint32, C.c_double, C.c_double, C.c_double,
                                          C.c_uint64, _u64p]
        L.kco_gen_chunglu.argtypes = [C.c_uint32, _u64p, C.c_uint64, C.c_uint32, C.c_uint32,
                                      C.c_uint64, _u32p]
        L.kco_build_csr.restype = C.c_uint64
        L.kco_build_csr.argtypes = [C.c_uint32, _u32p, C.c_uint64, _u64p, _u32p]
        L.kco_compute_index.restype = C.c_uint32
        L.kco_compute_index.argtypes = [_u32p, C.c_uint64, C.c_uint32]
        L.kco_should_notify.restype = C.c_int
        L.kco_should_notify.argtypes = [C.c_uint32] * 3
        L.kco_peel.argtypes = [C.c_uint32, _u64p, _u32p, _u32p]
        L.kco_degree_hindex.restype = C.c_uint32
        L.kco_degree_hindex.argtypes = [C.c_uint32, _u64p]
        L.kco_jacobi.restype = C.c_int
        L.kco_jacobi.argtypes = [C.c_uint32, _u64p, _u32p, C.c_int, C.c_int, _u32p,
                                 C.POINTER(Stats), C.c_void_p, C.c_uint64, C.c_void_p,
                                 C.c_void_p, C.c_uint64]
        L.kco_sequential_tail.argtypes = [C.c_uint32, _u64p, _u32p, _u32p, _u8p, C.c_int,
                                          C.POINTER(Stats)]
        L.kco_fastk.restype = C.c_int
        L.kco_fastk.argtypes = [C.c_uint32, _u64p, _u32p, C.c_uint32, C.c_int, C.c_int, _u32p,
                                C.POINTER(Stats)]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_PATH):
            build(ref=True)
        L = C.CDLL(REF_PATH)
        L.ref_graph_from_csr.restype = C.c_void_p
        L.ref_graph_from_csr.argtypes = [C.c_uint32, _u64p, _u32p]
        L.ref_graph_from_edges.restype = C.c_void_p
        L.ref_graph_from_edges.argtypes = [C.c_uint32, _u32p, C.c_uint64]
        L.ref_graph_free.argtypes = [C.c_void_p]
        L.ref_load_edge_list.restype = C.c_void_p
        L.ref_load_edge_list.argtypes = [C.c_char_p, C.c_uint64, C.c_char_p, C.c_uint64,
                                         C.POINTER(C.c_uint64)]
        L.ref_graph_n.restype = C.c_uint32
        L.ref_graph_n.argtypes = [C.c_void_p]
        L.ref_graph_original_ids.argtypes = [C.c_void_p, _u64p]
        L.ref_graph_nnz.restype = C.c_uint64
        L.ref_graph_nnz.argtypes = [C.c_void_p]
        L.ref_graph_csr.argtypes = [C.c_void_p, _u64p, _u32p]
        L.ref_peel.restype = C.c_uint32
        L.ref_peel.argtypes = [C.c_void_p, _u32p, C.POINTER(C.c_double)]
        L.ref_fastk.restype = C.c_int
        L.ref_fastk.argtypes = [C.c_void_p, C.c_uint, C.c_uint32, C.c_int, C.c_int, _u32p,
                                C.POINTER(RefStats)]
        L.ref_fastk_observed.restype = C.c_uint64
        L.ref_fastk_observed.argtypes = [C.c_void_p, C.c_uint, C.c_uint32, C.c_int, C.c_int,
                                         _u32p, C.POINTER(RefStats), _u32p, _u64p, C.c_uint64]
        L.ref_fastk_trace.restype = C.c_uint64
        L.ref_fastk_trace.argtypes = [C.c_void_p, C.c_uint, C.c_uint32, C.c_int, C.c_int,
                                      np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS"),
                                      np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS"),
                                      C.c_uint64]
        L.ref_compute_index.restype = C.c_uint32
        L.ref_compute_index.argtypes = [_u32p, C.c_uint64, C.c_uint32]
        L.ref_should_notify.restype = C.c_int
        L.ref_should_notify.argtypes = [C.c_uint32] * 3
        L.ref_switch_condition.restype = C.c_int
        L.ref_switch_condition.argtypes = [C.c_uint64, C.c_uint32]
        L.ref_sequential_tail.argtypes = [C.c_void_p, _u32p, _u8p, C.c_int, C.POINTER(RefStats)]
        _ref = L
    return _ref


# --------------------------------------------------------------------------
# Graphs
# --------------------------------------------------------------------------
@dataclass
class CSR:
    n: int
    off: np.ndarray   # uint64[n+1]
    nbr: np.ndarray   # uint32[nnz]

    @property
    def nnz(self) -> int:
        return int(self.off[-1]) if self.n else 0

    def degrees(self) -> np.ndarray:
        return np.diff(self.off).astype(np.uint32)


def build_csr(n: int, pairs: np.ndarray) -> CSR:
    """graph.cpp:85-128 restated (parallel, same output)."""
    pairs = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1)
    m = pairs.size // 2
    off = np.zeros(n + 1, dtype=np.uint64)
    nbr = np.zeros(max(2 * m, 1), dtype=np.uint32)
    nnz = lib().kco_build_csr(n, pairs if pairs.size else np.zeros(2, np.uint32), m, off, nbr)
    return CSR(n, off, nbr[:nnz].copy())


def csr_from_edges(n: int, edges) -> CSR:
    pairs = np.asarray(list(edges), dtype=np.uint32).reshape(-1)
    return build_csr(n, pairs)


# -- kcgen v1 synthetic generators (BASELINE.json configs) --
Q32 = 1 << 32
P_KEEP = 3006477107      # floor(0.70 * 2^32)
P_DIAG = 214748364       # floor(0.05 * 2^32)
T_A = 2448131358         # floor(0.57 * 2^32)
T_AB = 3264175144        # floor(0.76 * 2^32)
T_ABC = 4080218931       # floor(0.95 * 2^32)


def gen_er(n: int, m: int, seed: int) -> np.ndarray:
    p = np.empty(2 * m, dtype=np.uint32)
    lib().kco_gen_er(n, m, seed, p)
    return p


def gen_grid(side: int, seed: int) -> np.ndarray:
    p = np.empty(6 * side * side, dtype=np.uint32)
    lib().kco_gen_grid(side, P_KEEP, P_DIAG, seed, p)
    return p


def gen_rmat(scale: int, edge_factor: int, seed: int) -> np.ndarray:
    m = edge_factor << scale
    p = np.empty(2 * m, dtype=np.uint32)
    lib().kco_gen_rmat(scale, m, T_A, T_AB, T_ABC, seed, p)
    return p


def chunglu_prefix(n: int, seed: int, gamma=2.1, mean=20.0, wmax=5e5):
    wq = np.empty(max(n, 1), dtype=np.uint64)
    lib().kco_chunglu_weights(n, gamma, mean, wmax, seed, wq)
    pre = np.zeros(n + 1, dtype=np.uint64)
    np.cumsum(wq[:n], out=pre[1:])
    m = int((int(pre[-1]) + 1024) // 2048)   # round(sum(w) / 2)
    return pre, m


def gen_chunglu(n: int, seed: int, cliques=200, csize=300, gamma=2.1, mean=20.0, wmax=5e5):
    pre, m = chunglu_prefix(n, seed, gamma, mean, wmax)
    total = m + cliques * csize * (csize - 1) // 2
    p = np.empty(2 * total, dtype=np.uint32)
    lib().kco_gen_chunglu(n, pre, m, cliques, csize, seed, p)
    return p


# --------------------------------------------------------------------------
# Algorithms
# --------------------------------------------------------------------------
def compute_index(est, cap: int) -> int:
    a = np.ascontiguousarray(est, dtype=np.uint32)
    if a.size == 0:
        a = np.zeros(1, np.uint32)
        return int(lib().kco_compute_index(a, 0, cap))
    return int(lib().kco_compute_index(a, a.size, cap))


def should_notify(nc: int, oc: int, ev: int) -> bool:
    return bool(lib().kco_should_notify(nc, oc, ev))


def peel(g: CSR) -> np.ndarray:
    core = np.zeros(max(g.n, 1), dtype=np.uint32)
    lib().kco_peel(g.n, g.off, _nbr(g), core)
    return core[: g.n]


def degree_hindex(g: CSR) -> int:
    return int(lib().kco_degree_hindex(g.n, g.off))


RULES = {"ref_ext": 0, "ref_plain": 1, "snap_plain": 2, "snap_ext": 3}


def jacobi(g: CSR, rule: str = "ref_ext", clamp: bool = False, snapshots: int = 0,
           record: int = 0):
    """Jacobi replay (shadow_run, tests/test_fastk.cpp:41-92) + counters."""
    est = np.zeros(max(g.n, 1), dtype=np.uint32)
    st = Stats()
    snap = np.zeros((snapshots, max(g.n, 1)), dtype=np.uint32) if snapshots else None
    act = np.zeros(record, dtype=np.uint64) if record else None
    scn = np.zeros(record, dtype=np.uint64) if record else None
    lib().kco_jacobi(g.n, g.off, _nbr(g), RULES[rule], int(clamp), est, C.byref(st),
                     snap.ctypes.data if snap is not None else None, snapshots,
                     act.ctypes.data if act is not None else None,
                     scn.ctypes.data if scn is not None else None, record)
    out = {"est": est[: g.n], "stats": st.as_dict()}
    it = st.iterations
    if snap is not None:
        out["snapshots"] = snap[: min(it + 1, snapshots), : g.n]
    if act is not None:
        out["active_counts"] = act[: min(it + 1, record)]
        out["scanned"] = scn[: min(it, record)]
    return out


def fastk(g: CSR, batch: int = 256, ext: bool = True, hybrid: bool = True):
    """fastk_run restated at T=1 (src/fastk.cpp:57-187)."""
    est = np.zeros(max(g.n, 1), dtype=np.uint32)
    st = Stats()
    rc = lib().kco_fastk(g.n, g.off, _nbr(g), batch, int(ext), int(hybrid), est, C.byref(st))
    if rc != 0:
        raise ValueError("fastk: batch must be >= 1")
    return est[: g.n], st.as_dict()


def sequential_tail(g: CSR, est, active, ext: bool = True):
    e = np.ascontiguousarray(est, dtype=np.uint32).copy()
    a = np.ascontiguousarray(active, dtype=np.uint8).copy()
    st = Stats()
    lib().kco_sequential_tail(g.n, g.off, _nbr(g), e, a, int(ext), C.byref(st))
    return e, a, st.as_dict()


def _nbr(g: CSR) -> np.ndarray:
    return g.nbr if g.nbr.size else np.zeros(1, np.uint32)


# --------------------------------------------------------------------------
# The reference itself (oracle/_ref/libkcore_ref.so)
# --------------------------------------------------------------------------
def ref_load_edge_list(text: bytes):
    """The reference's kcore::load_edge_list on `text` (test infrastructure):
    returns (CSR, original ids) or raises ValueError("line N: what", line)."""
    L = ref()
    err = C.create_string_buffer(512)
    line = C.c_uint64()
    h = L.ref_load_edge_list(text, len(text), err, 512, C.byref(line))
    if not h:
        e = ValueError(err.value.decode(errors="replace"))
        e.line = int(line.value)
        raise e
    try:
        n = L.ref_graph_n(h)
        nnz = L.ref_graph_nnz(h)
        off = np.zeros(n + 1, dtype=np.uint64)
        nbr = np.zeros(max(nnz, 1), dtype=np.uint32)
        L.ref_graph_csr(h, off, nbr)
        ids = np.zeros(max(n, 1), dtype=np.uint64)
        L.ref_graph_original_ids(h, ids)
        return CSR(n, off, nbr[:nnz]), ids[:n]
    finally:
        L.ref_graph_free(h)


class RefGraph:
    """A kcore::Graph owned by the reference library."""

    def __init__(self, g: CSR | None = None, *, n: int | None = None, pairs=None):
        L = ref()
        if g is not None:
            self.n = g.n
            self.h = L.ref_graph_from_csr(g.n, g.off, _nbr(g))
        else:
            p = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1)
            self.n = n
            self.h = L.ref_graph_from_edges(n, p if p.size else np.zeros(2, np.uint32), p.size // 2)

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_graph_free(self.h)
            self.h = None

    def csr(self) -> CSR:
        nnz = ref().ref_graph_nnz(self.h)
        off = np.zeros(self.n + 1, dtype=np.uint64)
        nbr = np.zeros(max(nnz, 1), dtype=np.uint32)
        ref().ref_graph_csr(self.h, off, nbr)
        return CSR(self.n, off, nbr[:nnz])

    def peel(self):
        core = np.zeros(max(self.n, 1), dtype=np.uint32)
        kavg = C.c_double()
        kmax = ref().ref_peel(self.h, core, C.byref(kavg))
        return core[: self.n], int(kmax), float(kavg.value)

    def fastk(self, threads=16, batch=256, ext=True, hybrid=True):
        core = np.zeros(max(self.n, 1), dtype=np.uint32)
        st = RefStats()
        rc = ref().ref_fastk(self.h, threads, batch, int(ext), int(hybrid), core, C.byref(st))
        if rc != 0:
            raise ValueError("fastk: invalid argument")
        return core[: self.n], st.as_dict()

    def fastk_observed(self, threads=2, batch=8, ext=True, hybrid=False, max_snap=4096):
        n = max(self.n, 1)
        core = np.zeros(n, dtype=np.uint32)
        st = RefStats()
        snaps = np.zeros(max_snap * n, dtype=np.uint32)
        acts = np.zeros(max_snap, dtype=np.uint64)
        k = ref().ref_fastk_observed(self.h, threads, batch, int(ext), int(hybrid), core,
                                     C.byref(st), snaps, acts, max_snap)
        k = min(k, max_snap)
        return (core[: self.n], st.as_dict(), snaps[: k * n].reshape(k, n)[:, : self.n],
                acts[:k])

    def fastk_trace(self, threads=4, batch=256, ext=True, hybrid=True, max_rows=4096):
        me = np.zeros(max_rows)
        af = np.zeros(max_rows)
        k = ref().ref_fastk_trace(self.h, threads, batch, int(ext), int(hybrid), me, af, max_rows)
        k = min(k, max_rows)
        return me[:k], af[:k]

    def sequential_tail(self, est, active, ext=True):
        e = np.ascontiguousarray(est, dtype=np.uint32).copy()
        a = np.ascontiguousarray(active, dtype=np.uint8).copy()
        st = RefStats()
        ref().ref_sequential_tail(self.h, e, a, int(ext), C.byref(st))
        return e, a, st.as_dict()


def ref_compute_index(est, cap: int) -> int:
    a = np.ascontiguousarray(est, dtype=np.uint32)
    return int(ref().ref_compute_index(a if a.size else np.zeros(1, np.uint32), a.size, cap))


def physical_cores() -> int:
    """Physical cores as counted by tests/acceptance.cpp:555-581."""
    cores = set()
    phys = core = -1
    try:
        with open("/proc/cpuinfo") as f:
            for line in f.read().split("\n") + [""]:
                if not line.strip():
                    if phys >= 0 and core >= 0:
                        cores.add((phys, core))
                    phys = core = -1
                    continue
                if ":" not in line:
                    continue
                key = line.split("\t")[0]
                val = line.split(":", 1)[1].strip()
                if key == "physical id":
                    phys = int(val)
                elif key == "core id":
                    core = int(val)
    except OSError:
        pass
    return len(cores) if cores else (os.cpu_count() or 1)
