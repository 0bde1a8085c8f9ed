"""ctypes binding of include/kcore_b200.h and the reference-shaped Python API.

Names, argument meaning and error behaviour mirror the reference C++ API
(/root/reference/proj/include/kcore/*.hpp) so tests read like the
reference's own (tests/test_fastk.cpp, tests/test_oracle.cpp).
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Callable, Iterable, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# KC_LIB_PATH overrides the library (development: A/B builds); default in-tree.
_LIB_PATH = os.environ.get("KC_LIB_PATH") or os.path.join(_HERE, "libkcore_b200.so")

_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")


# --------------------------------------------------------------------------
# C structs (include/kcore_b200.h)
# --------------------------------------------------------------------------
class _Options(C.Structure):
    _fields_ = [("threads", C.c_uint32), ("batch", C.c_uint32),
                ("extended_notify", C.c_int32), ("hybrid_tail", C.c_int32),
                ("rule", C.c_int32), ("max_rounds", C.c_uint32),
                ("smem_cache", C.c_uint32), ("reserved", C.c_uint32 * 8)]


class _Stats(C.Structure):
    _fields_ = [("iterations", C.c_uint64), ("messages_sent", C.c_uint64),
                ("messages_drained", C.c_uint64), ("tail_pops", C.c_uint64),
                ("e_scan", C.c_uint64), ("v_eval", C.c_uint64), ("drops", C.c_uint64),
                ("tail_rounds", C.c_uint64), ("k_max", C.c_uint32), ("h_graph", C.c_uint32),
                ("k_avg", C.c_double), ("t_upload_ms", C.c_float), ("t_prep_ms", C.c_float),
                ("t_solve_ms", C.c_float), ("t_download_ms", C.c_float),
                ("kernel_launches", C.c_uint32), ("pad0", C.c_uint32),
                ("scan_evaluate", C.c_uint64), ("scan_notify", C.c_uint64),
                ("reserved", C.c_uint32 * 2)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_ if k not in ("reserved", "pad0")}


class _CSRView(C.Structure):
    _fields_ = [("n", C.c_uint32), ("nnz", C.c_uint64),
                ("offsets", C.c_void_p), ("neighbors", C.c_void_p)]


class _CSRDev(C.Structure):
    _fields_ = [("view", _CSRView), ("device", C.c_int), ("original_ids", C.c_void_p)]


class _ParseError(C.Structure):
    _fields_ = [("line", C.c_uint64), ("what", C.c_char * 160)]


_INSPECTOR = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint32), C.c_uint32,
                         C.c_uint64)

# every symbol include/kcore_b200.h declares (checked by tests/test_abi.py)
ABI_SYMBOLS = (
    "kc_status_str", "kc_abi_version", "kc_default_options", "kc_last_error",
    "kc_graph_upload", "kc_graph_upload_device", "kc_graph_free", "kc_graph_n",
    "kc_graph_nnz", "kc_graph_timings", "kc_solve", "kc_solve_device",
    "kc_solve_observed", "kc_fastk_run", "kc_graph_stream", "kc_gen_config",
    "kc_csr_dev_free", "kc_csr_dev_download", "kc_debug_phase_times", "kc_graph_upload_ex",
    "kc_debug_round_stats", "kc_debug_gather_probe", "kc_solve_traced", "kc_peel", "kc_verify", "kc_load_edge_list",
    "kc_load_edge_list_file", "kc_csr_dev_original_ids", "kc_sequential_tail",
    "kc_debug_layout", "kc_trim_memory", "kc_debug_host_copy",
)
KC_DEBUG_PHASE_TIMES = 1
KC_DEBUG_LEGACY_COUNT = 2
KC_DEBUG_VERIFY_PERTURB = 4
KC_DEBUG_NO_PULL = 8
KC_UPLOAD_FORCE_OFF64 = 1
KC_UPLOAD_FORCE_EST32 = 2
KC_UPLOAD_UNSORTED_ROWS = 4

_lib = None


def library_path() -> str:
    return _LIB_PATH


def load_library():
    """Load libkcore_b200.so.  Raises (no fallback) when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise RuntimeError(
            f"{_LIB_PATH} is not built; run `python -m paper_2512_00233_b200.build` "
            "(there is no CPU fallback for this path)")
    L = C.CDLL(_LIB_PATH)
    L.kc_status_str.restype = C.c_char_p
    L.kc_status_str.argtypes = [C.c_int]
    L.kc_last_error.restype = C.c_char_p
    L.kc_abi_version.restype = C.c_int
    L.kc_default_options.argtypes = [C.POINTER(_Options)]
    L.kc_graph_upload.restype = C.c_int
    L.kc_graph_upload.argtypes = [C.POINTER(_CSRView), C.c_int, C.POINTER(C.c_void_p)]
    L.kc_graph_upload_device.restype = C.c_int
    L.kc_graph_upload_device.argtypes = [C.POINTER(_CSRView), C.c_int, C.POINTER(C.c_void_p)]
    L.kc_graph_upload_ex.restype = C.c_int
    L.kc_graph_upload_ex.argtypes = [C.POINTER(_CSRView), C.c_int, C.c_int, C.c_uint32,
                                     C.POINTER(C.c_void_p)]
    L.kc_graph_free.argtypes = [C.c_void_p]
    L.kc_graph_n.restype = C.c_uint32
    L.kc_graph_n.argtypes = [C.c_void_p]
    L.kc_graph_nnz.restype = C.c_uint64
    L.kc_graph_nnz.argtypes = [C.c_void_p]
    L.kc_graph_timings.restype = C.c_int
    L.kc_graph_timings.argtypes = [C.c_void_p, C.POINTER(C.c_float), C.POINTER(C.c_float)]
    L.kc_graph_stream.restype = C.c_void_p
    L.kc_graph_stream.argtypes = [C.c_void_p]
    L.kc_solve.restype = C.c_int
    L.kc_solve.argtypes = [C.c_void_p, C.POINTER(_Options), C.c_void_p, C.POINTER(_Stats)]
    L.kc_solve_device.restype = C.c_int
    L.kc_solve_device.argtypes = [C.c_void_p, C.POINTER(_Options), C.c_void_p, C.POINTER(_Stats)]
    L.kc_solve_observed.restype = C.c_int
    L.kc_solve_observed.argtypes = [C.c_void_p, C.POINTER(_Options), _INSPECTOR, C.c_void_p,
                                    C.c_void_p, C.POINTER(_Stats)]
    L.kc_solve_traced.restype = C.c_int
    L.kc_solve_traced.argtypes = [C.c_void_p, C.POINTER(_Options), C.c_void_p, C.c_void_p,
                                  C.c_uint64, C.POINTER(C.c_uint64), C.c_void_p,
                                  C.POINTER(_Stats)]
    L.kc_load_edge_list.restype = C.c_int
    L.kc_load_edge_list.argtypes = [C.c_char_p, C.c_uint64, C.c_int, C.POINTER(C.POINTER(_CSRDev)),
                                    C.POINTER(_ParseError)]
    L.kc_load_edge_list_file.restype = C.c_int
    L.kc_load_edge_list_file.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.POINTER(_CSRDev)),
                                         C.POINTER(_ParseError)]
    L.kc_csr_dev_original_ids.restype = C.c_int
    L.kc_csr_dev_original_ids.argtypes = [C.POINTER(_CSRDev), C.c_void_p]
    L.kc_sequential_tail.restype = C.c_int
    L.kc_sequential_tail.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.POINTER(_Stats)]
    L.kc_peel.restype = C.c_int
    L.kc_peel.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(_Stats)]
    L.kc_verify.restype = C.c_int
    L.kc_verify.argtypes = [C.c_void_p, C.POINTER(_Options), C.c_void_p, C.c_uint64,
                            C.POINTER(C.c_uint64)]
    L.kc_fastk_run.restype = C.c_int
    L.kc_fastk_run.argtypes = [C.POINTER(_CSRView), C.POINTER(_Options), C.c_void_p,
                               C.POINTER(_Stats)]
    L.kc_gen_config.restype = C.c_int
    L.kc_gen_config.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                                C.POINTER(C.POINTER(_CSRDev))]
    L.kc_csr_dev_free.argtypes = [C.POINTER(_CSRDev)]
    L.kc_debug_phase_times.restype = C.c_int
    L.kc_debug_phase_times.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64,
                                       C.POINTER(C.c_uint32)]
    L.kc_debug_round_stats.restype = C.c_int
    L.kc_debug_round_stats.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32]
    L.kc_debug_gather_probe.restype = C.c_int
    L.kc_debug_gather_probe.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_float)]
    L.kc_debug_host_copy.restype = None
    L.kc_debug_host_copy.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64]
    L.kc_trim_memory.restype = C.c_int
    L.kc_trim_memory.argtypes = []
    L.kc_debug_layout.restype = C.c_int
    L.kc_debug_layout.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.POINTER(C.c_uint32), C.POINTER(C.c_int)]
    L.kc_csr_dev_download.restype = C.c_int
    L.kc_csr_dev_download.argtypes = [C.POINTER(_CSRDev), C.c_void_p, C.c_void_p]
    _lib = L
    return L


class KCError(RuntimeError):
    def __init__(self, status: int, where: str = ""):
        L = load_library()
        msg = L.kc_status_str(status).decode()
        detail = L.kc_last_error().decode()
        super().__init__(f"{where}: {msg}" + (f" ({detail})" if detail else ""))
        self.status = status


def _check(status: int, where: str) -> None:
    if status == 0:
        return
    if status == 1:  # KC_ERR_INVALID_ARGUMENT  ~ std::invalid_argument
        raise ValueError(load_library().kc_last_error().decode() or "invalid argument")
    raise KCError(status, where)


# --------------------------------------------------------------------------
# Reference types
# --------------------------------------------------------------------------
class Rule(enum.IntEnum):
    REFERENCE = 0   # notify on settled values, re-evaluate notified (fastk.cpp:156-163)
    COUNTING = 1    # support counters: only vertices that will drop are evaluated
    AUTO = 2


@dataclass
class FastKOptions:
    """include/kcore/fastk.hpp:12-22 (+ GPU knobs)."""
    threads: int = 16
    batch: int = 256
    extended_notify: bool = True
    hybrid_tail: bool = True
    rule: Rule = Rule.AUTO
    max_rounds: int = 0
    smem_cache: int = 0
    debug_flags: int = 0

    def _c(self) -> _Options:
        o = _Options()
        o.threads = max(0, int(self.threads))
        o.batch = max(0, int(self.batch))
        o.extended_notify = int(bool(self.extended_notify))
        o.hybrid_tail = int(bool(self.hybrid_tail))
        o.rule = int(self.rule)
        o.max_rounds = int(self.max_rounds)
        o.smem_cache = int(self.smem_cache) & 0xffffffff
        o.reserved[0] = int(self.debug_flags)
        return o


@dataclass
class IterationStat:
    """report.hpp:12-15"""
    mean_error: float
    active_fraction: float


@dataclass
class RunReport:
    """report.hpp:17-23 (+ GPU work counters and timings in `gpu`)."""
    iterations: int = 0
    messages_sent: int = 0
    messages_drained: int = 0
    tail_pops: int = 0
    trace: list = field(default_factory=list)
    gpu: dict = field(default_factory=dict)


@dataclass
class CorenessResult:
    """oracle.hpp:10-14"""
    coreness: np.ndarray
    k_max: int = 0
    k_avg: float = 0.0


@dataclass
class EngineResult:
    """report.hpp:25-28"""
    result: CorenessResult
    report: RunReport


@dataclass
class Instrumentation:
    """report.hpp:33-39: hooks at iteration boundaries (iteration 0 = degrees)."""
    truth: Optional[CorenessResult] = None
    trace_convergence: bool = False
    inspector: Optional[Callable[[int, np.ndarray, int], None]] = None


def make_coreness_result(coreness) -> CorenessResult:
    """oracle.cpp:8-19"""
    c = np.ascontiguousarray(coreness, dtype=np.uint32)
    if c.size == 0:
        return CorenessResult(c, 0, 0.0)
    return CorenessResult(c, int(c.max()), float(c.astype(np.float64).sum() / c.size))


def should_notify(new_core: int, old_core: int, est_v: int) -> bool:
    """fastk.hpp:25-27"""
    return new_core < est_v and old_core >= est_v


def switch_condition(active_count: int, batch: int) -> bool:
    """fastk.hpp:29-31"""
    return active_count < batch


class Graph:
    """Immutable simple undirected CSR (graph.hpp:37-75)."""

    def __init__(self, offsets=None, neighbors=None):
        if offsets is None:
            offsets = np.zeros(1, dtype=np.uint64)
        self._off = np.ascontiguousarray(offsets, dtype=np.uint64)
        self._nbr = np.ascontiguousarray(
            neighbors if neighbors is not None else np.zeros(0, np.uint32), dtype=np.uint32)
        if self._off.size < 1 or int(self._off[0]) != 0 or int(self._off[-1]) != self._nbr.size:
            raise ValueError("offsets must start at 0 and end at len(neighbors)")
        # the reference's Graph cannot hold anything else (graph.hpp:37-75); the
        # C-ABI re-checks on the device (KC_ERR_INVALID_ARGUMENT)
        if self._off.size > 1 and bool(np.any(self._off[1:] < self._off[:-1])):
            raise ValueError("offsets must be non-decreasing")
        if self._nbr.size and int(self._nbr.max()) >= self._off.size - 1:
            raise ValueError("neighbour id out of range")

    @classmethod
    def from_edges(cls, node_count: int, edges) -> "Graph":
        """Graph::from_edges (graph.hpp:43-44; build_csr graph.cpp:85-128):
        self-loops dropped, parallel edges collapse, rows strictly increasing."""
        e = np.asarray(edges, dtype=np.int64).reshape(-1, 2) if len(edges) else \
            np.zeros((0, 2), np.int64)
        if e.size and (e.min() < 0 or e.max() >= node_count):
            raise ValueError("edge endpoint out of range")
        e = e[e[:, 0] != e[:, 1]]
        both = np.concatenate([e, e[:, ::-1]]) if e.size else e
        key = np.unique(both[:, 0] * np.int64(node_count) + both[:, 1]) if both.size else \
            np.zeros(0, np.int64)
        src = key // max(node_count, 1)
        dst = (key % max(node_count, 1)).astype(np.uint32)
        off = np.zeros(node_count + 1, dtype=np.uint64)
        np.cumsum(np.bincount(src, minlength=node_count), out=off[1:])
        return cls(off, dst)

    def node_count(self) -> int:
        return self._off.size - 1

    def edge_count(self) -> int:
        return self._nbr.size // 2

    def degree(self, u: int) -> int:
        return int(self._off[u + 1] - self._off[u])

    def neighbors(self, u: int) -> np.ndarray:
        return self._nbr[int(self._off[u]):int(self._off[u + 1])]

    def offsets(self) -> np.ndarray:
        return self._off

    def neighbor_array(self) -> np.ndarray:
        return self._nbr

    def degrees(self) -> np.ndarray:
        return np.diff(self._off).astype(np.uint32)

    def _view(self) -> _CSRView:
        v = _CSRView()
        v.n = self.node_count()
        v.nnz = self._nbr.size
        v.offsets = self._off.ctypes.data
        v.neighbors = self._nbr.ctypes.data if self._nbr.size else None
        return v


class ParseError(ValueError):
    """kcore::ParseError (graph.hpp:13-23): malformed edge list, 1-based line."""

    def __init__(self, line: int, what: str):
        super().__init__(f"line {line}: {what}")
        self.line = line
        self.what = what


class IoError(RuntimeError):
    """kcore::IoError (graph.hpp:25-28)."""


class DeviceCSR:
    """A CSR in HBM: built by kc_gen_config (synthetic configs, kcgen v1) or
    loaded from a text edge list (kc_load_edge_list)."""

    def __init__(self, ptr):
        self._p = ptr

    @property
    def n(self) -> int:
        return self._p.contents.view.n

    @property
    def nnz(self) -> int:
        return self._p.contents.view.nnz

    def view(self) -> _CSRView:
        return self._p.contents.view

    def download(self) -> Graph:
        off = np.zeros(self.n + 1, dtype=np.uint64)
        nbr = np.zeros(max(self.nnz, 1), dtype=np.uint32)
        _check(load_library().kc_csr_dev_download(self._p, off.ctypes.data, nbr.ctypes.data),
               "kc_csr_dev_download")
        return Graph(off, nbr[: self.nnz])

    def original_ids(self) -> np.ndarray:
        """Graph::original_id for every dense id (graph.hpp:57)."""
        ids = np.zeros(max(self.n, 1), dtype=np.uint64)
        _check(load_library().kc_csr_dev_original_ids(self._p, ids.ctypes.data),
               "kc_csr_dev_original_ids")
        return ids[: self.n]

    def free(self) -> None:
        if self._p:
            load_library().kc_csr_dev_free(self._p)
            self._p = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def load_edge_list(text, device: int = 0) -> DeviceCSR:
    """kcore::load_edge_list (graph.hpp:76-81) parsed and densified on the
    device.  `text`: bytes or str.  Raises ParseError like the reference."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    p = C.POINTER(_CSRDev)()
    err = _ParseError()
    st = load_library().kc_load_edge_list(data, len(data), device, C.byref(p), C.byref(err))
    if st == 7:  # KC_ERR_PARSE
        raise ParseError(int(err.line), err.what.decode(errors="replace"))
    _check(st, "kc_load_edge_list")
    return DeviceCSR(p)


def load_edge_list_file(path: str, device: int = 0) -> DeviceCSR:
    """kcore::load_edge_list_file (graph.hpp:84) for plain-text files."""
    p = C.POINTER(_CSRDev)()
    err = _ParseError()
    st = load_library().kc_load_edge_list_file(path.encode(), device, C.byref(p), C.byref(err))
    if st == 7:
        raise ParseError(int(err.line), err.what.decode(errors="replace"))
    if st == 8:  # KC_ERR_IO
        raise IoError(err.what.decode(errors="replace"))
    _check(st, "kc_load_edge_list_file")
    return DeviceCSR(p)


def trim_memory() -> None:
    """Hand the device memory the library keeps between calls back to the driver."""
    _check(load_library().kc_trim_memory(), "kc_trim_memory")


def gen_config(cfg: int, p0: int, p1: int = 0, p2: int = 0, seed: int = 1,
               device: int = 0) -> DeviceCSR:
    """Build BASELINE.json config `cfg` (or a scaled variant) on the device."""
    p = C.POINTER(_CSRDev)()
    _check(load_library().kc_gen_config(cfg, p0, p1, p2, seed, device, C.byref(p)),
           "kc_gen_config")
    return DeviceCSR(p)


class GpuGraph:
    """An uploaded, laid-out graph handle (kc_graph)."""

    def __init__(self, g, device: int = 0, flags: int = 0):
        L = load_library()
        self._h = C.c_void_p()
        if isinstance(g, DeviceCSR):
            v = g.view()
            _check(L.kc_graph_upload_ex(C.byref(v), device, 1, flags, C.byref(self._h)),
                   "kc_graph_upload_ex")
        else:
            self._keep = g
            v = g._view()
            _check(L.kc_graph_upload_ex(C.byref(v), device, 0, flags, C.byref(self._h)),
                   "kc_graph_upload_ex")
        self.n = L.kc_graph_n(self._h)
        self.nnz = L.kc_graph_nnz(self._h)

    def timings(self):
        tu, tp = C.c_float(), C.c_float()
        load_library().kc_graph_timings(self._h, C.byref(tu), C.byref(tp))
        return tu.value, tp.value

    def stream(self) -> int:
        return load_library().kc_graph_stream(self._h) or 0

    def solve(self, options: FastKOptions | None = None, out: np.ndarray | None = None):
        o = (options or FastKOptions())._c()
        st = _Stats()
        if out is None:
            out = np.zeros(max(self.n, 1), dtype=np.uint32)
        _check(load_library().kc_solve(self._h, C.byref(o), out.ctypes.data, C.byref(st)),
               "kc_solve")
        return out[: self.n], st.as_dict()

    def solve_device(self, out_ptr: int, options: FastKOptions | None = None):
        o = (options or FastKOptions())._c()
        st = _Stats()
        _check(load_library().kc_solve_device(self._h, C.byref(o), C.c_void_p(out_ptr),
                                              C.byref(st)), "kc_solve_device")
        return st.as_dict()

    def solve_observed(self, options: FastKOptions | None,
                       fn: Callable[[int, np.ndarray, int], None]):
        o = (options or FastKOptions())._c()
        st = _Stats()
        out = np.zeros(max(self.n, 1), dtype=np.uint32)
        err = []

        def cb(user, it, est, n, active):
            try:
                arr = np.ctypeslib.as_array(est, shape=(n,)).copy() if n else \
                    np.zeros(0, np.uint32)
                fn(int(it), arr, int(active))
                return 0
            except Exception as e:  # propagate after the call returns
                err.append(e)
                return 1

        cfn = _INSPECTOR(cb)
        status = load_library().kc_solve_observed(self._h, C.byref(o), cfn, None,
                                                  out.ctypes.data, C.byref(st))
        if err:
            raise err[0]
        _check(status, "kc_solve_observed")
        return out[: self.n], st.as_dict()

    def solve_traced(self, options: FastKOptions | None, truth):
        """Convergence trace on the device (kc_solve_traced; record_iteration,
        report.cpp:7-18): returns (coreness, stats, [IterationStat])."""
        o = (options or FastKOptions())._c()
        st = _Stats()
        out = np.zeros(max(self.n, 1), dtype=np.uint32)
        tr = np.ascontiguousarray(truth, dtype=np.uint32)
        if tr.size != self.n:
            raise ValueError("truth must hold one coreness per vertex")
        cap = 4096
        rows = np.zeros((cap, 2), dtype=np.float64)
        nrows = C.c_uint64()
        _check(load_library().kc_solve_traced(self._h, C.byref(o), tr.ctypes.data, rows.ctypes.data,
                                              cap, C.byref(nrows), out.ctypes.data, C.byref(st)),
               "kc_solve_traced")
        if nrows.value > cap:  # long runs: once more with room for every row
            cap = int(nrows.value)
            rows = np.zeros((cap, 2), dtype=np.float64)
            _check(load_library().kc_solve_traced(self._h, C.byref(o), tr.ctypes.data,
                                                  rows.ctypes.data, cap, C.byref(nrows),
                                                  out.ctypes.data, C.byref(st)),
                   "kc_solve_traced")
        trace = [IterationStat(float(a), float(b)) for a, b in rows[: nrows.value]]
        return out[: self.n], st.as_dict(), trace

    def sequential_tail(self, est, active, extended_notify: bool = True):
        """kcore::sequential_tail (fastk.hpp:38-39) on the device: returns
        (estimates, active flags, stats) — the caller's arrays are not
        modified."""
        e = np.ascontiguousarray(est, dtype=np.uint32).copy()
        a = np.ascontiguousarray(active, dtype=np.uint8).copy()
        if e.size != self.n or a.size != self.n:
            raise ValueError("est and active need one entry per vertex")
        st = _Stats()
        _check(load_library().kc_sequential_tail(self._h, e.ctypes.data, a.ctypes.data,
                                                 int(bool(extended_notify)), C.byref(st)),
               "kc_sequential_tail")
        return e, a, st.as_dict()

    def peel(self):
        """kcore::peel_coreness (oracle.cpp:21-66) as an independent device
        algorithm (kc_peel): returns (coreness, stats; iterations = levels)."""
        st = _Stats()
        out = np.zeros(max(self.n, 1), dtype=np.uint32)
        _check(load_library().kc_peel(self._h, out.ctypes.data, C.byref(st)), "kc_peel")
        return out[: self.n], st.as_dict()

    def verify(self, options: FastKOptions | None = None, cap: int = 1024):
        """kcore::verify (oracle.cpp:68-75) on the device: FastK vs the device
        peel.  Returns (mismatch count, [(node, candidate, truth)] ascending,
        at most `cap`)."""
        o = (options or FastKOptions())._c()
        out = np.zeros((max(cap, 1), 3), dtype=np.uint32)
        cnt = C.c_uint64()
        _check(load_library().kc_verify(self._h, C.byref(o), out.ctypes.data, cap, C.byref(cnt)),
               "kc_verify")
        m = min(cap, cnt.value)
        return int(cnt.value), [tuple(int(x) for x in r) for r in out[:m]]

    def phase_times(self) -> np.ndarray:
        """[256 rounds, grid, 8] %globaltimer stamps (debug; KC_DEBUG_PHASE_TIMES)."""
        grid = C.c_uint32()
        buf = np.zeros(256 * 1024 * 8, dtype=np.uint64)
        _check(load_library().kc_debug_phase_times(self._h, buf.ctypes.data, buf.size,
                                                   C.byref(grid)), "kc_debug_phase_times")
        return buf[: 256 * grid.value * 8].reshape(256, grid.value, 8)

    def gather_probe(self, reps: int = 3) -> float:
        """ms per pass of the solver's inner operation alone (id stream + one
        estimate gather per adjacency entry; kc_debug_gather_probe)."""
        ms = C.c_float()
        _check(load_library().kc_debug_gather_probe(self._h, reps, C.byref(ms)),
               "kc_debug_gather_probe")
        return ms.value

    def layout(self):
        """(offsets [n_nz + 1], neighbours [nnz], perm [n], rows_sorted): the
        handle's relabelled CSR on the host (debug; kc_debug_layout)."""
        L = load_library()
        n_nz, srt = C.c_uint32(), C.c_int()
        _check(L.kc_debug_layout(self._h, None, None, None, C.byref(n_nz), C.byref(srt)),
               "kc_debug_layout")
        off = np.zeros(n_nz.value + 1, dtype=np.uint64)
        adj = np.zeros(max(int(L.kc_graph_nnz(self._h)), 1), dtype=np.uint32)
        perm = np.zeros(max(int(L.kc_graph_n(self._h)), 1), dtype=np.uint32)
        _check(L.kc_debug_layout(self._h, off.ctypes.data, adj.ctypes.data, perm.ctypes.data,
                                 None, None), "kc_debug_layout")
        return off, adj[: int(L.kc_graph_nnz(self._h))], perm[: int(L.kc_graph_n(self._h))], bool(srt.value)

    def round_stats(self, rounds: int) -> np.ndarray:
        """[rounds, 9] per-round counters of the last solve (debug): evals,
        escan (sum of degrees), drops, fires, nscan, ascan (entries streamed by
        evaluate), HUGE|BIG<<32, WARP|SUB<<32, THREAD."""
        buf = np.zeros((rounds, 9), dtype=np.uint64)
        _check(load_library().kc_debug_round_stats(self._h, buf.ctypes.data, rounds),
               "kc_debug_round_stats")
        return buf

    def free(self) -> None:
        if getattr(self, "_h", None):
            load_library().kc_graph_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _report(st: dict, trace=None) -> RunReport:
    return RunReport(iterations=int(st["iterations"]), messages_sent=int(st["messages_sent"]),
                     messages_drained=int(st["messages_drained"]),
                     tail_pops=int(st["tail_pops"]), trace=trace or [], gpu=st)


def fastk_run_abi(g: Graph, options: FastKOptions | None = None,
                  out: np.ndarray | None = None):
    """The one-shot C-ABI drop-in, kc_fastk_run: host CSR in (upload, layout,
    solve, download, free in one call), coreness written to `out` (host).
    Returns (coreness, stats dict)."""
    o = (options or FastKOptions())._c()
    st = _Stats()
    n = g.node_count()
    if out is None:
        out = np.zeros(max(n, 1), dtype=np.uint32)
    v = g._view()
    _check(load_library().kc_fastk_run(C.byref(v), C.byref(o), out.ctypes.data, C.byref(st)),
           "kc_fastk_run")
    return out[:n], st.as_dict()


def fastk_run(g: Graph, options: FastKOptions | None = None,
              instr: Instrumentation | None = None, device: int = 0) -> EngineResult:
    """kcore::fastk_run (fastk.hpp:46-47) on the B200.

    ValueError for zero threads/batch before any work (fastk.cpp:58-59)."""
    options = options or FastKOptions()
    if int(options.threads) == 0:
        raise ValueError("fastk: threads must be >= 1")
    if int(options.batch) == 0:
        raise ValueError("fastk: batch must be >= 1")
    gg = GpuGraph(g, device, flags=KC_UPLOAD_UNSORTED_ROWS)  # one solve: no row sort
    try:
        if instr is None or (not instr.trace_convergence and instr.inspector is None):
            core, st = gg.solve(options)
            return EngineResult(CorenessResult(core, int(st["k_max"]), float(st["k_avg"])),
                                _report(st))
        trace = []
        n = g.node_count()
        truth = None
        if instr.trace_convergence:
            if instr.truth is None:
                raise ValueError("trace_convergence requires truth")
            truth = np.asarray(instr.truth.coreness, dtype=np.float64)
            if instr.inspector is None:  # trace only: reductions on the device
                core, st, trace = gg.solve_traced(options, instr.truth.coreness)
                return EngineResult(CorenessResult(core, int(st["k_max"]), float(st["k_avg"])),
                                    _report(st, trace))

        def hook(it, est, active):
            if truth is not None:  # record_iteration, report.cpp:7-18
                gap = float((est.astype(np.float64) - truth).sum()) if n else 0.0
                trace.append(IterationStat(gap / n if n else 0.0, active / n if n else 0.0))
            if instr.inspector is not None:
                instr.inspector(it, est, active)

        core, st = gg.solve_observed(options, hook)
        return EngineResult(CorenessResult(core, int(st["k_max"]), float(st["k_avg"])),
                            _report(st, trace))
    finally:
        gg.free()
