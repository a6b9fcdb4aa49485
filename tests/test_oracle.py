"""Pins for the FP64 oracle (oracle/oracle.cpp), each against something other
than itself: a dense autograd brute force, finite differences, closed forms,
graph-theoretic invariants and the paper's central equivalence (PAPER.md:157,
172-176).  CPU only."""
import numpy as np
import pytest
import torch

import oracle
from oracle import brute
from xmgn_inputs import configs, geometry, graph, partition, tensors


def small_graph(n=24, k=4, seed=11, isolated=True):
    pos = geometry.sphere_points(n, seed=seed)[0]
    s, d = graph.knn_edges(pos, k)
    s, d = graph.symmetrize(s, d)
    nn = n + 1 if isolated else n          # node n has no edges
    return graph.to_csr(s, d, nn)


def rnd(shape, seed, scale=1.0):
    return np.random.default_rng(seed).uniform(-scale, scale, shape)


def make_params(H, L, m, seed=0):
    return tensors.params(H, L, m).double().numpy() if seed == 0 else \
        rnd(oracle.param_count(H, L, m), seed, 0.3)


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("m,H,L", [(2, 8, 3), (1, 4, 2)])
def test_oracle_matches_dense_bruteforce(m, H, L):
    off, src = small_graph()
    N, E = len(off) - 1, len(src)
    P = make_params(H, L, m, seed=3)
    h0, e0, g = rnd((N, H), 1, 1.5), rnd((E, H), 2, 1.5), rnd((N, H), 4)
    f = oracle.forward(off, src, P, h0, e0, H, L, m)
    b = oracle.backward(off, src, P, f, g, H, L, m)
    ref = brute.run(off, src, P, h0, e0, g, H, L, m)
    assert rel(f["h"], ref["h"]) < 1e-12
    assert rel(b["params"], ref["params"]) < 1e-12
    assert rel(b["h0"], ref["h0"]) < 1e-12
    assert rel(b["e0"], ref["e0"]) < 1e-12
    # the isolated node aggregates nothing: its a^l rows are 0
    assert np.all(f["a"][:, N - 1] == 0.0)


def test_oracle_finite_differences():
    off, src = small_graph(16, 3, isolated=False)
    N, E, H, L, m = len(off) - 1, len(src), 4, 2, 2
    P = make_params(H, L, m, seed=5)
    h0, e0, g = rnd((N, H), 6), rnd((E, H), 7), rnd((N, H), 8)
    f = oracle.forward(off, src, P, h0, e0, H, L, m)
    b = oracle.backward(off, src, P, f, g, H, L, m)
    loss = lambda P_, h_, e_: float((g * oracle.forward(off, src, P_, h_, e_, H, L, m)["h"][-1]).sum())  # noqa
    rng = np.random.default_rng(0)
    step = 1e-6
    for idx in rng.choice(P.size, 12, replace=False):
        Pp, Pm = P.copy(), P.copy()
        Pp[idx] += step; Pm[idx] -= step
        fd = (loss(Pp, h0, e0) - loss(Pm, h0, e0)) / (2 * step)
        assert abs(fd - b["params"][idx]) <= 1e-6 * max(1.0, abs(fd))
    for arr, key in ((h0, "h0"), (e0, "e0")):
        for flat in rng.choice(arr.size, 5, replace=False):
            i = np.unravel_index(flat, arr.shape)
            ap, am = arr.copy(), arr.copy()
            ap[i] += step; am[i] -= step
            args_p = (P, ap, e0) if key == "h0" else (P, h0, ap)
            args_m = (P, am, e0) if key == "h0" else (P, h0, am)
            fd = (loss(*args_p) - loss(*args_m)) / (2 * step)
            assert abs(fd - b[key][i]) <= 1e-6 * max(1.0, abs(fd))


def test_closed_form_zero_last_linear():
    """W_{m+1} = 0 in every block => each block outputs the constant LN(b_{m+1});
    h^L = h^0 + sum_l c_n^l and e^L = e^0 + sum_l c_e^l exactly (up to FP64
    rounding), and dW_j, db_j for j <= m vanish."""
    off, src = small_graph(40, 5)
    N, E, H, L, m = len(off) - 1, len(src), 8, 3, 2
    P = make_params(H, L, m, seed=9)
    lay, _ = tensors.param_layout(H, L, m)
    c = {0: np.zeros(H), 1: np.zeros(H)}
    for name, l, blk, slot, offp, shape, fan in lay:
        if name == f"W{m+1}":
            P[offp:offp + shape[0] * shape[1]] = 0.0
    for l in range(L):
        for blk in (0, 1):
            ent = {name: (offp, shape) for name, ll, bb, s, offp, shape, fan in lay if ll == l and bb == blk}
            sl = lambda nm: torch.tensor(P[ent[nm][0]:ent[nm][0] + H])  # noqa
            c[blk] += torch.nn.functional.layer_norm(sl(f"b{m+1}")[None], (H,), sl("gamma"), sl("beta"), 1e-5)[0].numpy()
    h0, e0, g = rnd((N, H), 1), rnd((E, H), 2), rnd((N, H), 3)
    f = oracle.forward(off, src, P, h0, e0, H, L, m)
    assert np.abs(f["h"][-1] - (h0 + c[1])).max() < 1e-13
    assert np.abs(f["e"][-1] - (e0 + c[0])).max() < 1e-13
    b = oracle.backward(off, src, P, f, g, H, L, m)
    for name, l, blk, slot, offp, shape, fan in lay:
        if name in [f"W{j}" for j in range(1, m + 1)] + [f"b{j}" for j in range(1, m + 1)]:
            assert np.all(b["params"][offp:offp + int(np.prod(shape))] == 0.0)


def test_degree_classes_bitwise():
    """e^0 = 0 and h^0 = one constant row: layer-1 rows depend only on in-degree
    (the aggregation multiplicity, Eq. 2): equal degree => bitwise equal."""
    b = configs.custom((400,), P=1, halo=0)
    off, src = b["offsets"], b["sources"]
    N, E, H, L = len(off) - 1, len(src), 8, 1
    P = make_params(H, L, 2, seed=13)
    h0 = np.tile(rnd((1, H), 5), (N, 1))
    f = oracle.forward(off, src, P, h0, np.zeros((E, H)), H, L)
    deg = np.diff(off)
    classes = np.unique(deg)
    assert len(classes) >= 3
    reps = []
    for d in classes:
        rows = f["h"][1][deg == d]
        assert (rows == rows[0]).all()
        reps.append(rows[0])
    reps = np.array(reps)
    assert len(np.unique(reps, axis=0)) == len(classes)


@pytest.fixture(scope="module")
def two_level():
    return configs.custom((300, 1500), k=6, P=4, halo=3)


def _partitioned(b, H, L, P, depth, g_full, params):
    off, src = b["offsets"], b["sources"]
    N = len(off) - 1
    oo = b["owned_offsets"]
    res = []
    for p in range(len(oo) - 1):
        owned = b["owned"][oo[p]:oo[p + 1]]
        lg = oracle.local_graph(off, src, owned, depth)
        h0 = tensors.node_features(lg["gid"], H).double().numpy()
        e0 = tensors.edge_features(lg["edge_gid"], H).double().numpy()
        f = oracle.forward(lg["offsets"], lg["sources"], params, h0, e0, H, L)
        g = np.zeros((len(lg["gid"]), H))
        g[:lg["n_owned"]] = g_full[lg["gid"][:lg["n_owned"]]]
        bk = oracle.backward(lg["offsets"], lg["sources"], params, f, g, H, L)
        res.append((lg, f, bk))
    return res


def test_partitioned_equals_full(two_level):
    """halo = L => owned rows of the partitioned forward equal
    the full graph (bitwise under the in-edge-order rule) and the sum
    of per-partition gradients equals the full-graph gradient."""
    b = two_level
    off, src = b["offsets"], b["sources"]
    N, E, H, L = len(off) - 1, len(src), 8, 3
    params = make_params(H, L, 2)
    h0 = tensors.node_features(np.arange(N), H).double().numpy()
    e0 = tensors.edge_features(np.arange(E), H).double().numpy()
    g = tensors.upstream_grad(np.arange(N), H).double().numpy()
    f = oracle.forward(off, src, params, h0, e0, H, L)
    bk = oracle.backward(off, src, params, f, g, H, L)
    Gp = np.zeros_like(bk["params"]); gh = np.zeros_like(bk["h0"]); ge = np.zeros_like(bk["e0"])
    for lg, fp, bp in _partitioned(b, H, L, 4, L, g, params):
        no = lg["n_owned"]
        assert np.array_equal(fp["h"][-1][:no], f["h"][-1][lg["gid"][:no]])     # bitwise
        Gp += bp["params"]
        np.add.at(gh, lg["gid"], bp["h0"])
        np.add.at(ge, lg["edge_gid"], bp["e0"])
    assert rel(Gp, bk["params"]) < 1e-12
    assert rel(gh, bk["h0"]) < 1e-12
    assert rel(ge, bk["e0"]) < 1e-12


def test_halo_too_small_is_detected(two_level):
    """Negative control: halo = L-1 breaks equality."""
    b = two_level
    off, src = b["offsets"], b["sources"]
    N, E, H, L = len(off) - 1, len(src), 8, 3
    params = make_params(H, L, 2)
    h0 = tensors.node_features(np.arange(N), H).double().numpy()
    e0 = tensors.edge_features(np.arange(E), H).double().numpy()
    f = oracle.forward(off, src, params, h0, e0, H, L)
    worst = 0.0
    for lg, fp, _ in _partitioned(b, H, L, 4, L - 1, np.zeros((N, H)), params):
        no = lg["n_owned"]
        worst = max(worst, np.abs(fp["h"][-1][:no] - f["h"][-1][lg["gid"][:no]]).max())
    assert worst > 1e-6


def test_local_graph_matches_generator_halo(two_level):
    b = two_level
    oo, ho = b["owned_offsets"], b["halo_offsets"]
    for p in range(len(oo) - 1):
        lg = oracle.local_graph(b["offsets"], b["sources"], b["owned"][oo[p]:oo[p + 1]], 3)
        no = lg["n_owned"]
        assert np.array_equal(lg["gid"][:no], b["owned"][oo[p]:oo[p + 1]])
        assert np.array_equal(lg["gid"][no:], b["halo"][ho[p]:ho[p + 1]])
        assert np.array_equal(lg["ring"][no:], b["halo_ring"][ho[p]:ho[p + 1]])
        rev = lg["rev"]
        assert (rev >= 0).all() and np.array_equal(rev[rev], np.arange(len(rev)))


def test_locality_probe():
    """after L layers a node depends only on its L-hop ball."""
    b = configs.custom((600,), P=1, halo=0)
    off, src = b["offsets"], b["sources"]
    N, E, H, L = len(off) - 1, len(src), 8, 2
    params = make_params(H, L, 2)
    ring = partition.halo_rings(off, src, np.arange(N) == 0, L + 1)
    far = np.nonzero(ring < 0)[0][0]
    h0 = tensors.node_features(np.arange(N), H).double().numpy()
    e0 = tensors.edge_features(np.arange(E), H).double().numpy()
    f1 = oracle.forward(off, src, params, h0, e0, H, L)
    h0[far] += 1.0
    f2 = oracle.forward(off, src, params, h0, e0, H, L)
    assert np.array_equal(f1["h"][-1][0], f2["h"][-1][0])
    assert not np.array_equal(f1["h"][-1][far], f2["h"][-1][far])


def test_permutation_equivariance():
    off, src = small_graph(30, 5, isolated=False)
    N, E, H, L = len(off) - 1, len(src), 8, 2
    params = make_params(H, L, 2, seed=4)
    h0, e0 = rnd((N, H), 1), rnd((E, H), 2)
    f = oracle.forward(off, src, params, h0, e0, H, L)
    perm = np.random.default_rng(1).permutation(N)          # new id of old node
    dst = np.repeat(np.arange(N), np.diff(off))
    key = perm[dst] * N + perm[src]
    order = np.argsort(key)
    off2, src2 = graph.to_csr(perm[src], perm[dst], N)
    h02 = np.empty_like(h0); h02[perm] = h0
    f2 = oracle.forward(off2, src2, params, h02, e0[order], H, L)
    assert np.abs(f2["h"][-1][perm] - f["h"][-1]).max() < 1e-12
