"""The HBM generator + on-device CSR construction (kc_gen_config; the GPU
form of build_csr, src/graph.cpp:85-128) equal the CPU generator + the
reference's CSR construction on the same kcgen v1 inputs."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [
    (1, (5000, 40000, 0), 11),
    (1, (100000, 1000000, 0), 1),
    (2, (300, 0, 0), 2),
    (3, (12, 16, 0), 3),
    (3, (17, 16, 0), 3),
    (5, (14, 8, 0), 5),
    (4, (30000, 4, 40), 4),
    (4, (200000, 10, 100), 9),
]


def cpu_csr(oracle, cfg, p, seed):
    if cfg == 1:
        return oracle.build_csr(p[0], oracle.gen_er(p[0], p[1], seed))
    if cfg == 2:
        return oracle.build_csr(p[0] * p[0], oracle.gen_grid(p[0], seed))
    if cfg in (3, 5):
        return oracle.build_csr(1 << p[0], oracle.gen_rmat(p[0], p[1], seed))
    return oracle.build_csr(p[0], oracle.gen_chunglu(p[0], seed, cliques=p[1], csize=p[2]))


@pytest.mark.parametrize("cfg,p,seed", CASES)
def test_gpu_generator_equals_cpu(gpu, oracle, cfg, p, seed):
    want = cpu_csr(oracle, cfg, p, seed)
    d = gpu.gen_config(cfg, p[0], p[1], p[2], seed=seed)
    got = d.download()
    assert got.node_count() == want.n
    assert np.array_equal(got.offsets(), want.off)
    assert np.array_equal(got.neighbor_array(), want.nbr)


def test_gpu_csr_equals_reference_builder(gpu, ref):
    """Against the reference's own Graph::from_edges on the same pairs."""
    pairs = ref.gen_rmat(11, 16, 21)
    want = ref.RefGraph(n=1 << 11, pairs=pairs).csr()
    got = gpu.gen_config(3, 11, 16, 0, seed=21).download()
    assert np.array_equal(got.offsets(), want.off)
    assert np.array_equal(got.neighbor_array(), want.nbr)


def test_device_upload_path_solves(gpu, oracle):
    """kc_graph_upload_device: the graph never leaves HBM."""
    d = gpu.gen_config(3, 16, 16, 0, seed=3)
    gg = gpu.GpuGraph(d)
    core, st = gg.solve(gpu.FastKOptions())
    truth = oracle.peel(cpu_csr(oracle, 3, (16, 16, 0), 3))
    assert np.array_equal(core, truth)
