"""Pins for the NEXT-1 oracle (oracle/model.py): encoder -> processor -> decoder ->
owned-row MSE, each against something other than itself -- the dense PyTorch-FP64
autograd statement (oracle/brute.run_model), SPEC.md's worked feature examples,
SSE additivity over halo partitions, finite differences and a
closed form.  CPU only."""
import math

import numpy as np
import pytest

import oracle
from oracle import brute
from oracle import model as M
from xmgn_inputs import geometry, graph, tensors


def small(n=20, k=4, seed=3):
    pos, nrm = geometry.sphere_points(n, seed=seed)
    s, d = graph.knn_edges(pos, k)
    s, d = graph.symmetrize(s, d)
    off, src = graph.to_csr(s, d, n)
    return pos.astype(np.float64), nrm.astype(np.float64), off, src


def rnd(shape, seed, scale=1.0):
    return np.random.default_rng(seed).uniform(-scale, scale, shape)


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def setup(H, L, m, n=20, seed=3):
    pos, nrm, off, src = small(n, seed=seed)
    P = rnd(oracle.param_count(H, L, m), 11, 0.3)
    io = rnd(M.io_param_count(H, m), 12, 0.4)
    stats = M.feature_stats(pos, nrm, off, src)
    t = rnd((len(off) - 1, 4), 13, 1.5)
    return pos, nrm, off, src, P, io, stats, t


@pytest.mark.parametrize("m,H,L", [(2, 8, 2), (1, 6, 1)])
def test_model_oracle_matches_dense_autograd(m, H, L):
    pos, nrm, off, src, P, io, stats, t = setup(H, L, m)
    fw = M.forward(off, src, pos, nrm, P, io, stats, H, L, m, targets=t)
    bw = M.backward(off, src, P, io, fw, H, L, m)
    ref = brute.run_model(off, src, pos, nrm, P, io, stats, t, H, L, m)
    assert rel(fw["y"], ref["y"]) < 1e-12
    assert abs(fw["loss"] - ref["loss"]) <= 1e-12 * abs(ref["loss"])
    assert rel(bw["params"], ref["params"]) < 1e-11
    assert rel(bw["io"], ref["io"]) < 1e-11


def test_feature_examples_spec():
    # origin -> sin columns 0, cos columns 1; width 24 with position + normal
    X = M.node_inputs(np.zeros((1, 3)), np.array([[0.0, 0.0, 1.0]]))
    assert X.shape == (1, 24)
    four = X[0, 6:].reshape(3, 3, 2)           # [freq][coord][sin, cos]
    assert np.all(four[..., 0] == 0.0) and np.all(four[..., 1] == 1.0)
    # (0.25, 0, 0), f = 2 pi: sin = 1, cos = 0 within 1e-12 (quarter period)
    X = M.node_inputs(np.array([[0.25, 0.0, 0.0]]), np.zeros((1, 3)))
    assert abs(X[0, 6] - 1.0) < 1e-12 and abs(X[0, 7]) < 1e-12
    # f = 4 pi at x = 0.25: sin(pi) = 0, cos(pi) = -1 (freq-major order: columns 12, 13)
    assert abs(X[0, 12]) < 1e-12 and abs(X[0, 13] + 1.0) < 1e-12
    # receiver i = (0,0,0), sender j = (1,0,0) -> (1,0,0,1); swap negates
    pos = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0]])
    off, src = np.array([0, 1, 2]), np.array([1, 0])          # edge 1->0, edge 0->1
    Xe = M.edge_inputs(pos, off, src)
    assert np.array_equal(Xe[0], [1.0, 0.0, 0.0, 1.0])
    assert np.array_equal(Xe[1], [-1.0, 0.0, 0.0, 1.0])
    # coincident points -> zeros
    assert np.array_equal(M.edge_inputs(np.zeros((2, 3)), off, src), np.zeros((2, 4)))


def test_zscore_stats():
    pos, nrm, off, src = small(40)
    mean, std = M.feature_stats(pos, nrm, off, src)
    Xn = M.zscore(M.node_inputs(pos, nrm), mean[:24], std[:24])
    Xe = M.zscore(M.edge_inputs(pos, off, src), mean[24:], std[24:])
    assert np.abs(Xn.mean(0)).max() < 1e-12 and np.abs(Xe.mean(0)).max() < 1e-12
    assert np.abs(Xn.std(0) - 1).max() < 1e-12 and np.abs(Xe.std(0) - 1).max() < 1e-12


def test_partitioned_sse_and_gradients_sum_to_full():
    """Sum over halo partitions of the owned-row SSE / (N d) equals the full-graph MSE and
    the summed gradients equal the full graph's."""
    from xmgn_inputs import partition
    H, L, m = 6, 2, 2
    pos, nrm, off, src, P, io, stats, t = setup(H, L, m, n=48, seed=5)
    N = len(off) - 1
    full = M.forward(off, src, pos, nrm, P, io, stats, H, L, m, targets=t)
    gfull = M.backward(off, src, P, io, full, H, L, m)
    owner = partition.rcb(pos.astype(np.float32), 3)
    loss, gp, gi = 0.0, 0.0, 0.0
    for p in range(3):
        lg = oracle.local_graph(off, src, np.flatnonzero(owner == p), L)
        gid = lg["gid"]
        fw = M.forward(lg["offsets"], lg["sources"], pos[gid], nrm[gid], P, io, stats, H, L, m, targets=t[gid],
                       n_owned=lg["n_owned"], n_global=N)
        bw = M.backward(lg["offsets"], lg["sources"], P, io, fw, H, L, m)
        assert rel(fw["y"][:lg["n_owned"]], full["y"][gid[:lg["n_owned"]]]) < 1e-12
        loss += fw["loss"]; gp = gp + bw["params"]; gi = gi + bw["io"]
    assert abs(loss - full["loss"]) <= 1e-12 * full["loss"]
    assert rel(gp, gfull["params"]) < 1e-10
    assert rel(gi, gfull["io"]) < 1e-10


def test_io_finite_differences():
    H, L, m = 4, 1, 2
    pos, nrm, off, src, P, io, stats, t = setup(H, L, m, n=14, seed=7)
    fw = M.forward(off, src, pos, nrm, P, io, stats, H, L, m, targets=t)
    bw = M.backward(off, src, P, io, fw, H, L, m)
    f = lambda x: M.forward(off, src, pos, nrm, P, x, stats, H, L, m, targets=t)["loss"]  # noqa: E731
    rng = np.random.default_rng(1)
    for i in rng.choice(io.size, 24, replace=False):
        d = np.zeros_like(io); d[i] = 1e-5
        fd = (f(io + d) - f(io - d)) / 2e-5
        assert abs(fd - bw["io"][i]) <= 1e-6 * max(1.0, abs(fd)), (i, fd, bw["io"][i])


def test_decoder_closed_form():
    """W_{m+1} = 0 in the decoder: y = b_{m+1} on every row whatever the graph, and the
    loss is the closed-form mean of (b - t)^2."""
    H, L, m = 6, 2, 2
    pos, nrm, off, src, P, io, stats, t = setup(H, L, m)
    lay, _ = M.io_layout(H, m)
    name, o, s = lay["dec"][-2]
    io = io.copy(); io[o:o + s[0] * s[1]] = 0.0
    b = io[lay["dec"][-1][1]:lay["dec"][-1][1] + 4]
    fw = M.forward(off, src, pos, nrm, P, io, stats, H, L, m, targets=t)
    assert np.abs(fw["y"] - b).max() < 1e-15
    assert abs(fw["loss"] - ((b - t) ** 2).mean()) < 1e-14
    # and the processor gradient vanishes (nothing flows through a zero output layer)
    bw = M.backward(off, src, P, io, fw, H, L, m)
    assert np.abs(bw["params"]).max() == 0.0


def test_io_param_count_matches_generator():
    for H, m in ((8, 2), (128, 1), (512, 2)):
        assert tensors.io_param_layout(H, m)[1] == M.io_param_count(H, m)
    # (F_n + F_e) H + 2 m (H^2 + H) + 4 H (encoders) + decoder
    H, m = 512, 2
    enc = (24 + 4) * H + 2 * H + 2 * m * (H * H + H) + 4 * H
    dec = m * (H * H + H) + H * 4 + 4
    assert M.io_param_count(H, m) == enc + dec
    assert math.isclose(M.FREQS[2], 8 * math.pi)
