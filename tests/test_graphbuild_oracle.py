"""Pins of the NEXT-4 graph-construction oracle (oracle/graphbuild.py): SPEC.md's hand
examples, exact ties on a lattice, structural invariants, and agreement with the input
generator's independent construction (KD-tree candidates + exact selection, sparse-matrix
BFS; itself pinned against brute force in tests/test_inputs.py).  CPU only."""
import numpy as np
import pytest

from oracle import graphbuild as G
from xmgn_inputs import configs, geometry, graph, partition


def test_knn_tie_rule_and_complete_neighbourhoods():
    # x = 0, 1, 2 with k = 1 -> node 1's in-neighbour is node 0 (tie by index)
    pos = np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0]], np.float32)
    assert list(G.knn(pos, 1)[:, 0]) == [1, 0, 1]
    # n = 5, k = 4 -> every other node
    p5 = geometry.sphere_points(5, seed=2)[0]
    nb = G.knn(p5, 4)
    for i in range(5):
        assert sorted(nb[i]) == [j for j in range(5) if j != i]
    # k = 1 on the 3 collinear points -> 4 directed edges after symmetrisation
    off, src = G.multiscale_csr(pos, [3], 1)
    assert len(src) == 4


def test_lattice_ties_match_generator():
    """A 6 x 6 x 2 integer lattice: every node has many equal-distance neighbours."""
    g = np.stack(np.meshgrid(np.arange(6), np.arange(6), np.arange(2), indexing="ij"), -1).reshape(-1, 3)
    pos = g.astype(np.float32)
    assert np.array_equal(G.knn(pos, 6), graph.knn_brute(pos, 6))
    off, src = G.multiscale_csr(pos, [20, len(pos)], 6)
    o2, s2 = graph.multiscale_graph(pos, [20, len(pos)], 6)
    assert np.array_equal(off, o2) and np.array_equal(src, s2)


def test_path_graph_halo_spec_example():
    # path 0-1-2-3-4, owner {0,1} -> p0, {2,3,4} -> p1
    off = np.array([0, 1, 3, 5, 7, 8])
    src = np.array([1, 0, 2, 1, 3, 2, 4, 3])
    owner = np.array([0, 0, 1, 1, 1])
    ps = G.partitions(off, src, owner, 2, 1)
    assert list(ps["halo"]) == [2, 1] and list(ps["halo_offsets"]) == [0, 1, 2]
    ps = G.partitions(off, src, owner, 2, 2)
    assert list(ps["halo"][:2]) == [2, 3] and list(ps["halo"][2:]) == [1, 0]   # (ring, id) order
    assert list(ps["halo_ring"]) == [1, 2, 1, 2]
    # replication factor (3 + 4) / 5 = 1.4 at L = 1
    ps = G.partitions(off, src, owner, 2, 1)
    assert (5 + len(ps["halo"])) / 5 == 1.4


def test_rcb_cube_corners_and_balance():
    # 8 unit-cube corners, P = 2 -> the two x-median halves (x is the first widest axis)
    c = np.array([[x, y, z] for x in (0, 1) for y in (0, 1) for z in (0, 1)], np.float32)
    owner = G.rcb(c, 2)
    assert np.array_equal(owner, (c[:, 0] > 0).astype(np.int64))
    pos = geometry.car_points(1000, seed=3)[0]
    for P in (3, 7, 8):
        cnt = np.bincount(G.rcb(pos, P), minlength=P)
        assert cnt.sum() == 1000 and cnt.max() - cnt.min() <= int(np.ceil(np.log2(P)))   # +-1/2 per split level


@pytest.mark.parametrize("shape,levels,P,depth", [("sphere", (60, 250), 4, 3), ("car", (100, 300, 700), 5, 4)])
def test_oracle_matches_generator(shape, levels, P, depth):
    """The generator (configs.build) constructs the same graph and partitions."""
    pos = geometry.nested_levels(list(levels), shape=shape, seed=4)[0]
    ref = G.build(pos, list(levels), 6, P, depth)
    b = configs.build(shape, list(levels), 6, P, depth, seed=4)
    for key in ("offsets", "sources", "owner", "owned_offsets", "owned", "halo_offsets", "halo", "halo_ring"):
        assert np.array_equal(ref[key], b[key]), key


def test_halo_invariants():
    pos = geometry.sphere_points(300, seed=5)[0]
    off, src = G.multiscale_csr(pos, [300], 6)
    owner = G.rcb(pos, 4)
    prev = None
    for L in (1, 2, 3):
        ps = G.partitions(off, src, owner, 4, L)
        sets = [set(ps["halo"][ps["halo_offsets"][p]:ps["halo_offsets"][p + 1]]) for p in range(4)]
        if prev is not None:
            assert all(a <= b for a, b in zip(prev, sets))        # monotone in L
        prev = sets
    assert sorted(np.concatenate([np.flatnonzero(owner == p) for p in range(4)])) == list(range(300))
    # saturation: depth >= diameter -> owned + halo = everything
    ps = G.partitions(off, src, owner, 4, 300)
    for p in range(4):
        assert (owner == p).sum() + ps["halo_offsets"][p + 1] - ps["halo_offsets"][p] == 300
    # halo rings equal the generator's sparse-matrix BFS
    r = G.halo_rings(off, src, np.flatnonzero(owner == 1), 3)
    r2 = partition.halo_rings(off, src, owner == 1, 3)
    assert np.array_equal(r, r2)
