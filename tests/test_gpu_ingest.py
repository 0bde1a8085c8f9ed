"""Edge-list ingest on the device (kc_ingest.cu) vs the reference's
kcore::load_edge_list (src/graph.cpp:22-80, 141-199): the golden fixtures
written from the reference (tests/golden/edge_lists.json) and, where the
compiled reference is present, live comparisons on larger random texts."""
import os

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def check_graph(d, want):
    assert d.n == want["n"]
    host = d.download()
    assert host.offsets().tolist() == want["offsets"]
    assert host.neighbor_array().tolist() == want["neighbors"]
    assert [str(int(x)) for x in d.original_ids()] == want["original_ids"]


def test_golden_edge_lists(gpu):
    cases = golden("edge_lists.json")
    assert len(cases) >= 15
    for name, want in cases.items():
        if "error" in want:
            with pytest.raises(gpu.ParseError) as e:
                gpu.load_edge_list(want["text"])
            assert e.value.line == want["error_line"], name
            assert str(e.value) == want["error"], name
        else:
            check_graph(gpu.load_edge_list(want["text"]), want)


def test_loaded_graph_solves_like_the_reference(gpu, oracle):
    want = golden("edge_lists.json")["random_3000"]
    d = gpu.load_edge_list(want["text"])
    core, _ = gpu.GpuGraph(d).solve()
    off = np.array(want["offsets"], np.uint64)
    nbr = np.array(want["neighbors"], np.uint32)
    assert np.array_equal(core, oracle.peel(oracle.CSR(want["n"], off, nbr)))


def _random_text(rng, m, id_hi):
    u = rng.integers(0, id_hi, m, dtype=np.uint64)
    v = rng.integers(0, id_hi, m, dtype=np.uint64)
    seps = np.array([" ", "\t", "  "])[rng.integers(0, 3, m)]
    lines = [f"{a}{s}{b}" for a, s, b in zip(u.tolist(), seps.tolist(), v.tolist())]
    lines.insert(0, "# generated")
    return ("\n".join(lines) + "\n").encode()


@pytest.mark.parametrize("id_hi", [1 << 12, 1 << 40])
def test_large_random_vs_reference(gpu, ref, id_hi):
    """200 K edges, dense (table path of densify) and sparse (sort path) ids."""
    rng = np.random.default_rng(id_hi % 997)
    text = _random_text(rng, 200_000, id_hi)
    g, ids = ref.ref_load_edge_list(text)
    d = gpu.load_edge_list(text)
    assert d.n == g.n and d.nnz == g.nnz
    host = d.download()
    assert np.array_equal(host.offsets(), g.off)
    assert np.array_equal(host.neighbor_array(), g.nbr)
    assert np.array_equal(d.original_ids(), ids)


def test_file_and_io_error(gpu, tmp_path):
    want = golden("edge_lists.json")["basic"]
    p = tmp_path / "g.txt"
    p.write_text(want["text"])
    check_graph(gpu.load_edge_list_file(str(p)), want)
    with pytest.raises(gpu.IoError):
        gpu.load_edge_list_file(str(tmp_path / "missing.txt"))


def test_gzip_file_like_the_reference(gpu, tmp_path):
    """load_edge_list_file reads gzip input transparently (graph.cpp:200-226):
    the same CSR and original ids as the plain text, for every golden case;
    malformed compressed input raises ParseError / IoError like the text."""
    import gzip
    cases = golden("edge_lists.json")
    for name, want in cases.items():
        p = tmp_path / f"{name}.txt.gz"
        with gzip.open(p, "wb") as f:
            f.write(want["text"].encode())
        if "error" in want:
            with pytest.raises(gpu.ParseError) as e:
                gpu.load_edge_list_file(str(p))
            assert e.value.line == want["error_line"]
        else:
            check_graph(gpu.load_edge_list_file(str(p)), want)
    bad = tmp_path / "truncated.gz"
    data = gzip.compress(cases["random_3000"]["text"].encode())
    bad.write_bytes(data[: len(data) // 2])
    with pytest.raises((gpu.IoError, gpu.ParseError)):
        gpu.load_edge_list_file(str(bad))
