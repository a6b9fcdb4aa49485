"""GPU graph construction (NEXT-4, xmgn_build_graph) vs the oracle (oracle/graphbuild.py) and
the input generator (KD-tree + exact selection, pinned against brute force): every array of the
multi-scale kNN CSR, the RCB owner array and the (ring, id)-ordered halo lists bit-exact."""
import numpy as np
import pytest
import torch

from oracle import graphbuild as G
from xmgn_inputs import configs, geometry

pytestmark = pytest.mark.gpu
KEYS = ("offsets", "sources", "owner", "owned_offsets", "owned", "halo_offsets", "halo", "halo_ring")


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2411_17164_b200 import xmgn  # noqa: F401


def gpu_build(pos, levels, k, P, depth):
    from paper_2411_17164_b200 import xmgn
    t = torch.as_tensor(np.ascontiguousarray(pos, np.float32), device="cuda")
    return xmgn.build_graph(t, levels, k, P, depth)


def same(a, b):
    for key in KEYS:
        assert np.array_equal(np.asarray(a[key]), np.asarray(b[key])), key


@pytest.mark.parametrize("shape,levels,k,P,depth", [("sphere", (60, 250), 6, 4, 3), ("car", (100, 300, 700), 6, 5, 4),
                                                    ("sphere", (40, 400), 12, 3, 2), ("car", (500,), 1, 1, 2)])
def test_build_matches_oracle(shape, levels, k, P, depth):
    pos = geometry.nested_levels(list(levels), shape=shape, seed=4)[0]
    same(gpu_build(pos, levels, k, P, depth), G.build(pos, list(levels), k, P, depth))


def test_build_lattice_ties():
    """Integer lattice: exact equal distances everywhere, so the (d2, index) tie rule decides."""
    g = np.stack(np.meshgrid(np.arange(9), np.arange(7), np.arange(3), indexing="ij"), -1).reshape(-1, 3)
    pos = g.astype(np.float32) * 0.5
    perm = np.random.default_rng(0).permutation(len(pos))
    pos = pos[perm]
    same(gpu_build(pos, (50, len(pos)), 6, 4, 3), G.build(pos, [50, len(pos)], 6, 4, 3))


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_build_matches_generator_at_scale(name):
    c = configs.CONFIGS[name]
    b = configs.load(name)
    out = gpu_build(b["positions"], c["levels"], c["k"], c["P"], c["L"])
    same(out, b)


def test_built_graph_runs_the_processor():
    """The built graph loads (xmgn_load_graph) and the processor forward on it equals the one on
    the generator's bundle bitwise."""
    from paper_2411_17164_b200.processor import Processor
    b = configs.custom((300, 1500), k=6, P=3, halo=2)
    out = gpu_build(b["positions"], (300, 1500), 6, 3, 2)
    out["positions"], out["normals"] = b["positions"], b["normals"]
    res = []
    for bundle in (b, out):
        pr = Processor(bundle, 128, 2)
        params = pr.make_params()
        h0, e0, _ = pr.make_inputs(1)
        res.append(pr.forward(1, params, h0, e0).cpu().numpy())
        pr.close()
    assert np.array_equal(res[0], res[1])


def test_build_errors():
    from paper_2411_17164_b200 import xmgn
    pos = geometry.sphere_points(100, seed=1)[0]
    with pytest.raises(xmgn.XmgnError, match="EINVAL"):
        gpu_build(pos, (50, 90), 6, 2, 2)          # levels must end at n
    with pytest.raises(xmgn.XmgnError, match="EUNSUPPORTED"):
        gpu_build(pos, (100,), 17, 2, 2)
