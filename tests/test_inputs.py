"""Pins for the seeded input generator (xmgn_inputs) -- CPU only."""
import json
import os

import numpy as np
import pytest
import torch

from xmgn_inputs import configs, geometry, graph, partition, tensors

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_knn_collinear_tie():
    g = GOLD["knn_collinear_tie"]
    nb = graph.knn(np.array(g["positions"], np.float32), g["k"])
    assert nb[1, 0] == g["in_neighbour_of_1"]
    assert (graph.knn_brute(np.array(g["positions"], np.float32), 1) == nb).all()


def test_knn_complete():
    g = GOLD["knn_complete"]
    pos = geometry.sphere_points(g["n"], seed=3)[0]
    nb = graph.knn(pos, g["k"])
    for i in range(g["n"]):
        assert sorted(nb[i]) == [j for j in range(g["n"]) if j != i]


@pytest.mark.parametrize("n,k", [(500, 6), (2000, 12), (300, 1)])
def test_knn_equals_brute_force(n, k):
    pos = geometry.car_points(n, seed=7)[0]
    assert (graph.knn(pos, k) == graph.knn_brute(pos, k)).all()


def test_knn_ties_on_lattice():
    # integer lattice: massive exact distance ties, resolved by index
    g = np.stack(np.meshgrid(np.arange(6), np.arange(6), np.arange(3), indexing="ij"), -1)
    pos = g.reshape(-1, 3).astype(np.float32)
    assert (graph.knn(pos, 6) == graph.knn_brute(pos, 6)).all()


def test_symmetrize_examples():
    s, d = graph.symmetrize(np.array([0]), np.array([1]))
    off, src = graph.to_csr(s, d, 2)
    got = sorted((int(src[k]), int(i)) for i in range(2) for k in range(off[i], off[i + 1]))
    assert got == [tuple(x) for x in GOLD["symmetrize_single"]["expected"]]
    g = GOLD["symmetrize_knn1_collinear"]
    s, d = graph.knn_edges(np.array(g["positions"], np.float32), g["k"])
    s, d = graph.symmetrize(s, d)
    off, src = graph.to_csr(s, d, 3)
    assert off[-1] == g["n_edges"]


def test_prefix_nesting_and_degree():
    counts = [200, 500, 1200]
    pos, _ = geometry.nested_levels(counts, "car", seed=5)
    for c in counts[:-1]:
        p2, _ = geometry.nested_levels([x for x in counts if x <= c], "car", seed=5)
        assert np.array_equal(p2, pos[:c])
    off, src = graph.multiscale_graph(pos, counts, 6)
    deg = np.diff(off)
    assert deg.min() >= 6
    assert off[-1] <= sum(2 * 6 * c for c in counts)        # union bound
    # CSR invariants: strictly ascending sources per row, no self loops, symmetric
    dst = np.repeat(np.arange(len(pos)), deg)
    assert (src != dst).all()
    for i in range(0, len(pos), 97):
        r = src[off[i]:off[i + 1]]
        assert (np.diff(r) > 0).all()
    fwd = set(zip(src.tolist(), dst.tolist()))
    assert all((d, s) in fwd for s, d in fwd)


def test_graph_deterministic():
    a = configs.custom((100, 400), P=2, halo=2)
    b = configs.custom((100, 400), P=2, halo=2)
    assert configs.checksum(a) == configs.checksum(b)


def _path_graph():
    s = np.array([0, 1, 1, 2, 2, 3, 3, 4])
    d = np.array([1, 0, 2, 1, 3, 2, 4, 3])
    return graph.to_csr(s, d, 5)


@pytest.mark.parametrize("L", [1, 2])
def test_path_graph_halo(L):
    g = GOLD["path_graph_halo"]
    off, src = _path_graph()
    owner = np.array(g["owner"])
    ps = partition.partition_set(off, src, owner, 2, L)
    ho = ps["halo_offsets"]
    for p in range(2):
        assert sorted(ps["halo"][ho[p]:ho[p + 1]].tolist()) == g[f"L{L}"][f"halo_p{p}"]
    if L == 1:
        repl = (len(ps["owned"]) + len(ps["halo"])) / 5
        assert repl == pytest.approx(GOLD["path_graph_replication"]["value"])


def test_halo_zero_and_saturation():
    off, src = _path_graph()
    owner = np.array([0, 0, 1, 1, 1])
    assert len(partition.partition_set(off, src, owner, 2, 0)["halo"]) == 0
    ps = partition.partition_set(off, src, owner, 2, 10)
    assert len(ps["halo"]) == 5


def test_rcb_cube():
    pos = np.array(GOLD["rcb_cube_corners"]["positions"], np.float32)
    owner = partition.rcb(pos, 2)
    assert sorted(np.nonzero(owner == 0)[0].tolist()) == [0, 2, 4, 6]


def test_rcb_balance_and_coverage():
    b = configs.custom((500, 3000), P=8, halo=3)
    cnt = np.diff(b["owned_offsets"])
    assert cnt.max() - cnt.min() <= 1
    assert np.array_equal(np.sort(b["owned"]), np.arange(3000))


def test_tensors_bf16_exact_and_device_free():
    v = tensors.sym_uniform(7, 3, np.arange(1000), 64, 1.7)
    assert torch.equal(v, v.to(torch.bfloat16).float())
    # rows hashed by global id: a subset equals the corresponding rows
    sub = tensors.sym_uniform(7, 3, np.array([5, 999, 17]), 64, 1.7)
    assert torch.equal(sub, v[[5, 999, 17]])
    u = tensors.uniform(1, 2, np.arange(20000), 8)
    assert 0.0 < float(u.min()) and float(u.max()) < 1.0
    assert abs(float(u.mean()) - 0.5) < 0.01


def test_param_layout_count():
    for H, L, m in [(8, 3, 2), (128, 15, 2), (512, 15, 2), (16, 2, 1)]:
        lay, n = tensors.param_layout(H, L, m)
        assert n == tensors.param_count(H, L, m) == L * ((5 + 2 * m) * H * H + (2 * m + 6) * H)
    p = tensors.params(8, 2)
    lay, _ = tensors.param_layout(8, 2)
    for name, l, blk, slot, off, shape, fan in lay:
        v = p[off:off + int(np.prod(shape))]
        if name == "gamma":
            assert float((v - 1).abs().max()) <= 0.1 * 3 ** 0.5 + 1e-3
        elif name.startswith("W"):
            assert float(v.abs().max()) <= fan ** -0.5 + 1e-3
