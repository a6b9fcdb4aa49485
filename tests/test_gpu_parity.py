"""GPU parity: the CUDA path through the C-ABI vs the FP64 oracle.

Tolerances (north_star): forward max|dh| <= tau * RMS(h_oracle)
at the last layer, tau = 1e-4 in the FP32 check mode and 2e-2 for 16-bit
operand modes; parameter gradients per tensor relative Frobenius <= tau."""
import numpy as np
import pytest
import torch

from xmgn_inputs import configs, geometry, graph, partition
from gpu_util import (max_over_rms, oracle_full, oracle_probe, per_tensor_rel, rel_fro, run_gpu)

pytestmark = pytest.mark.gpu

FP32, BF16, FP16 = 1, 0, 2
TAU = {FP32: 1e-4, BF16: 2e-2, FP16: 2e-2}


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2411_17164_b200 import xmgn  # noqa: F401  (fails loudly if libxmgn.so is missing)


def _check(res, ref, H, L, tau, m=2, inputs=True):
    f = max_over_rms(res["h"], ref["h"])
    gw, name = per_tensor_rel(res["params"], ref["params"], H, L, m)
    assert f <= tau, f"forward max/RMS {f:.3e} > {tau}"
    assert gw <= tau, f"gradient {name} rel Frobenius {gw:.3e} > {tau}"
    if inputs:
        assert rel_fro(res["h0"], ref["h0"]) <= tau
        assert rel_fro(res["e0"], ref["e0"]) <= tau
    return f, gw


@pytest.mark.parametrize("N", [64, 128, 256])
@pytest.mark.parametrize("amn,bmn", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_selftest_gemm(N, amn, bmn):
    from paper_2411_17164_b200 import xmgn
    M, K = 384, 192
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(N, K, device="cuda").bfloat16()
    C = torch.zeros(M, N, device="cuda")
    xmgn.selftest_gemm(A.t().contiguous() if amn else A, B.t().contiguous() if bmn else B, C, amn, bmn, M, N, K)
    torch.cuda.synchronize()
    ref = A.double() @ B.double().t()
    assert (C.double() - ref).abs().max().item() < 1e-3


def test_cfg1_fp32_check_mode():
    """CFG1: 2,000-point sphere, k=6, H=128, L=2, one partition, FP32 check mode."""
    b = configs.load("cfg1")
    res = run_gpu(b, 128, 2, FP32)
    ref = oracle_full(b, 128, 2)
    _check(res, ref, 128, 2, TAU[FP32])


@pytest.mark.parametrize("prec", [FP32, FP16, BF16])
def test_multiscale_partitioned_all_modes(prec):
    """2-level nested cloud, 4 RCB partitions with halo 3, L=3, H=128 (ragged tiles)."""
    b = configs.custom((300, 1500), k=6, P=4, halo=3)
    res = run_gpu(b, 128, 3, prec)
    ref = oracle_full(b, 128, 3)
    _check(res, ref, 128, 3, TAU[prec])


@pytest.mark.parametrize("H", [256, 512])
@pytest.mark.parametrize("prec", [FP16, BF16])
def test_wide_hidden(H, prec):
    b = configs.custom((200, 900), k=6, P=2, halo=2, shape="car")
    res = run_gpu(b, H, 2, prec)
    ref = oracle_full(b, H, 2)
    _check(res, ref, H, 2, TAU[prec])


def test_mlp_one_hidden_layer():
    b = configs.custom((500,), k=6, P=2, halo=2)
    res = run_gpu(b, 128, 2, FP32, m=1)
    ref = oracle_full(b, 128, 2, m=1)
    _check(res, ref, 128, 2, TAU[FP32], m=1)


def test_isolated_node_and_single_edge():
    """an isolated node aggregates 0; a node with one in-edge
    aggregates exactly that edge."""
    pos = geometry.sphere_points(300, seed=2)[0]
    s, d = graph.symmetrize(*graph.knn_edges(pos, 4))
    s = np.concatenate([s, [300, 301]]); d = np.concatenate([d, [301, 300]])  # 300-301 pair
    off, src = graph.to_csr(s, d, 303)                                          # 302 isolated
    owner = np.zeros(303, np.int64)
    b = dict(offsets=off, sources=src, **partition.partition_set(off, src, owner, 1, 2))
    res = run_gpu(b, 128, 2, FP32)
    ref = oracle_full(b, 128, 2)
    _check(res, ref, 128, 2, TAU[FP32])


@pytest.mark.parametrize("prec,gtol", [(FP32, 1e-5), (FP16, 2e-3)])
def test_partitioned_forward_bitwise_and_grad_sum(prec, gtol):
    """PAPER.md:172-176 on the GPU: owned rows of P=4 equal P=1 bitwise (local
    in-edge order = global order, identical per-row arithmetic); summed
    gradients agree to the operand rounding (per-partition dZ rows of halo
    nodes are rounded separately: ~2^-11 relative in FP16, ~2^-17 in check mode)."""
    b1 = configs.custom((300, 1500), k=6, P=1, halo=3)
    b4 = configs.custom((300, 1500), k=6, P=4, halo=3)
    r1 = run_gpu(b1, 128, 3, prec)
    r4 = run_gpu(b4, 128, 3, prec)
    assert np.array_equal(r1["h"], r4["h"])
    assert rel_fro(r4["params"], r1["params"]) < gtol
    assert rel_fro(r4["h0"], r1["h0"]) < gtol


def test_deterministic_bitwise():
    b = configs.custom((300, 1500), k=6, P=4, halo=3)
    a = run_gpu(b, 128, 3, FP16)
    c = run_gpu(b, 128, 3, FP16)
    for k in ("h", "params", "h0", "e0"):
        assert np.array_equal(a[k], c[k]), k


def test_check_finite_and_state_errors():
    from paper_2411_17164_b200 import xmgn
    from paper_2411_17164_b200.processor import Processor
    t = torch.ones(1000, device="cuda")
    xmgn.check_finite(t)
    t[777] = float("nan")
    with pytest.raises(xmgn.XmgnError, match="ENONFINITE"):
        xmgn.check_finite(t)
    b = configs.custom((400,), k=6, P=2, halo=2)
    pr = Processor(b, 128, 2, precision=FP16)
    params = pr.make_params()
    gp = torch.zeros(pr.n_params, device="cuda")
    h0, e0, g = pr.make_inputs(1)
    with pytest.raises(xmgn.XmgnError, match="ESTATE"):
        pr.backward(1, params, g, gp)
    pr.forward(1, params, h0, e0)
    with pytest.raises(xmgn.XmgnError, match="ESTATE"):
        pr.backward(0, params, g, gp)
    pr.backward(1, params, g, gp)
    with pytest.raises(xmgn.XmgnError, match="EHALO"):
        xmgn.Workspace(pr.graph, xmgn.model_cfg(128, 3))
    with pytest.raises(xmgn.XmgnError, match="EUNSUPPORTED"):
        xmgn.Workspace(pr.graph, xmgn.model_cfg(96, 2))
    pr.close()


@pytest.mark.slow
def test_cfg2_full_forward_fp16():
    """CFG2 at full size (100k points, 15 layers, H=128): every output row vs the oracle."""
    b = configs.load("cfg2")
    res = run_gpu(b, 128, 15, FP16, want_inputs=False)
    import oracle
    from xmgn_inputs import tensors
    off, src = b["offsets"], b["sources"]
    N, E = len(off) - 1, len(src)
    f = oracle.forward(off, src, tensors.params(128, 15).double().numpy(),
                       tensors.node_features(np.arange(N), 128).double().numpy(),
                       tensors.edge_features(np.arange(E), 128).double().numpy(), 128, 15)
    err = max_over_rms(res["h"], f["h"][-1])
    assert err <= TAU[FP16], err


@pytest.mark.slow
def test_cfg2_probe_gradients():
    """CFG2 full-size gradients: with dL/dh^L non-zero only on probe rows, the
    full-graph gradient is the sum of each probe's L-hop-ball gradient (locality,
    PAPER.md:157), which the oracle computes ball by ball."""
    b = configs.load("cfg2")
    N = len(b["offsets"]) - 1
    probes = np.random.default_rng(0).choice(N, 6, replace=False)
    mask = np.zeros(N)
    mask[probes] = 1.0
    res = run_gpu(b, 128, 15, FP16, g_rows=mask)
    Gp = None
    for pnode in probes:
        o = oracle_probe(b, int(pnode), 128, 15)
        Gp = o["params"] if Gp is None else Gp + o["params"]
        assert np.abs(res["h"][pnode] - o["h"]).max() <= TAU[FP16] * np.sqrt((res["h"] ** 2).mean())
    gw, name = per_tensor_rel(res["params"], Gp, 128, 15)
    assert gw <= TAU[FP16], (gw, name)


@pytest.mark.slow
def test_cfg4_probe_forward():
    """CFG4 (the bench workload: 2M-point 3-level cloud, 8 partitions, H=512,
    L=15): one owned probe row per partition pair vs the oracle's 15-hop ball."""
    b = configs.load("cfg4")
    res = run_gpu(b, 512, 15, FP16, want_inputs=False)
    rms = np.sqrt((res["h"][b["owned"][:10000]] ** 2).mean())
    N = len(b["offsets"]) - 1
    for pnode in np.random.default_rng(1).choice(N, 1, replace=False):
        o = oracle_probe(b, int(pnode), 512, 15, with_grad=False)
        assert np.abs(res["h"][pnode] - o["h"]).max() <= TAU[FP16] * rms


def _hand_bundle(offsets, sources, owner, P, halo):
    from xmgn_inputs import partition as part
    offsets = np.asarray(offsets, np.int64)
    sources = np.asarray(sources, np.int64)
    return dict(offsets=offsets, sources=sources, owner=np.asarray(owner),
                **part.partition_set(offsets, sources, np.asarray(owner), P, halo))


@pytest.mark.parametrize("prec", [FP32, FP16])
def test_degenerate_graphs(prec):
    """Degenerate inputs: isolated nodes (empty in-neighbourhood: agg = 0),
    fewer edges than one 128-row tile, and partitions whose halo-shrunk top layers have
    no edges at all.  Path 0-1-2-3-4 plus isolated nodes 5 and 6, split into 3 partitions."""
    # CSR by destination, sources ascending, symmetric
    nbr = {0: [1], 1: [0, 2], 2: [1, 3], 3: [2, 4], 4: [3], 5: [], 6: []}
    offsets = np.cumsum([0] + [len(nbr[i]) for i in range(7)])
    sources = np.concatenate([nbr[i] for i in range(7)]).astype(np.int64)
    b = _hand_bundle(offsets, sources, [0, 0, 1, 1, 2, 2, 2], 3, 2)
    res = run_gpu(b, 128, 2, prec)
    ref = oracle_full(b, 128, 2)
    _check(res, ref, 128, 2, TAU[prec])


def test_single_partial_tile_many_partitions():
    """Every partition smaller than one CTA pair tile (256 rows), ragged everywhere."""
    b = configs.custom((60, 180), k=4, P=6, halo=3)
    res = run_gpu(b, 256, 3, FP16)
    ref = oracle_full(b, 256, 3)
    _check(res, ref, 256, 3, TAU[FP16])


@pytest.mark.slow
def test_cfg4_probe_gradients():
    """CFG4 at the bench's full size and launch configuration (8 halo partitions,
    H=512, L=15, FP16): with dL/dh^L non-zero on one probe row only, the parameter
    gradient summed over the 8 partitions equals the probe's 15-hop-ball gradient,
    which the FP64 oracle computes (partitioned = full graph)."""
    b = configs.load("cfg4")
    N = len(b["offsets"]) - 1
    probe = int(np.random.default_rng(2).choice(N, 1)[0])
    mask = np.zeros(N)
    mask[probe] = 1.0
    res = run_gpu(b, 512, 15, FP16, g_rows=mask, want_inputs=False)
    o = oracle_probe(b, probe, 512, 15)
    rms = np.sqrt((res["h"][b["owned"][:10000]] ** 2).mean())
    assert np.abs(res["h"][probe] - o["h"]).max() <= TAU[FP16] * rms
    gw, name = per_tensor_rel(res["params"], o["params"], 512, 15)
    assert gw <= TAU[FP16], (gw, name)


def test_z1_checkpoint_mode(monkeypatch):
    """Opt-in XMGN_Z1=1: the forward keeps z_1 and the backward replaces the first edge
    GEMM's recompute by a K = 0 step that reloads it; same parity bound as the default."""
    monkeypatch.setenv("XMGN_Z1", "1")
    b = configs.custom((300, 1500), k=6, P=4, halo=3)
    res = run_gpu(b, 512, 3, FP16)
    ref = oracle_full(b, 512, 3)
    _check(res, ref, 512, 3, TAU[FP16])
