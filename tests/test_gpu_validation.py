"""Malformed CSR through the raw C-ABI (no Python-side checks): the upload
fails with KC_ERR_INVALID_ARGUMENT (device-side checks in kc_prep.cu) instead
of reading or writing out of bounds."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _upload_raw(kc, off, nbr, flags=0, on_device=False):
    L = kc.load_library()
    off = np.ascontiguousarray(off, np.uint64)
    nbr = np.ascontiguousarray(nbr, np.uint32)
    v = kc.api._CSRView()
    v.n = off.size - 1
    v.nnz = nbr.size
    v.offsets = off.ctypes.data
    v.neighbors = nbr.ctypes.data if nbr.size else None
    h = C.c_void_p()
    st = L.kc_graph_upload_ex(C.byref(v), 0, 0, flags, C.byref(h))
    if st == 0:
        L.kc_graph_free(h)
    return st


@pytest.mark.parametrize("flags", [0, 4])  # sorted rows / KC_UPLOAD_UNSORTED_ROWS
def test_upload_rejects_malformed_csr(gpu, flags):
    KC_ERR_INVALID_ARGUMENT = 1
    good_off = np.array([0, 2, 4, 6], np.uint64)
    good_nbr = np.array([1, 2, 0, 2, 0, 1], np.uint32)
    assert _upload_raw(gpu, good_off, good_nbr, flags) == 0
    # a neighbour id >= n (would index perm/inv/E out of bounds)
    assert _upload_raw(gpu, good_off, np.array([1, 2, 0, 9, 0, 1], np.uint32), flags) == \
        KC_ERR_INVALID_ARGUMENT
    big = np.array([1, 2, 0, 0xFFFFFFFF, 0, 1], np.uint32)
    assert _upload_raw(gpu, good_off, big, flags) == KC_ERR_INVALID_ARGUMENT
    # non-monotone offsets (offsets[0] and offsets[n] still consistent)
    assert _upload_raw(gpu, np.array([0, 4, 2, 6], np.uint64), good_nbr, flags) == \
        KC_ERR_INVALID_ARGUMENT
    # the library stays usable afterwards
    g = gpu.Graph(good_off, good_nbr)
    core, _ = gpu.GpuGraph(g).solve()
    assert list(core) == [2, 2, 2]


def test_library_leaves_process_state_alone(gpu):
    """The library allocates from its own memory pool (the device's default
    pool keeps its release threshold for co-resident libraries) and restores
    the caller's current device."""
    from cuda.bindings import runtime as rt
    import torch
    torch.cuda.set_device(0)
    err, pool = rt.cudaDeviceGetDefaultMemPool(0)
    assert err == rt.cudaError_t.cudaSuccess
    err, before = rt.cudaMemPoolGetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrReleaseThreshold)
    g = gpu.Graph.from_edges(4, [(0, 1), (1, 2), (2, 0), (2, 3)])
    core, _ = gpu.GpuGraph(g).solve()
    assert list(core) == [2, 2, 2, 1]
    err, after = rt.cudaMemPoolGetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrReleaseThreshold)
    assert int(after) == int(before)
    assert torch.cuda.current_device() == 0
