"""The five BASELINE.json configurations as seeded graph recipes, with a disk cache.

CFG1  sphere, 2,000 points, k=6, H=128, L=2, P=1, FP32 check mode
CFG2  car proxy, 100k points, k=6, H=128, L=15, P=1
CFG3  car proxy, levels 50k/200k/800k, k=6, H=512, L=15, P=8, halo 15
CFG4  car proxy, levels 500k/1M/2M, k=6, H=512, L=15, P=8, halo 15
CFG5  car proxy, levels 2.5M/5M/10M, k=6, H=512, L=15, P=32, halo 15

Geometry seed 0.  Small test graphs use ``custom``.
"""
import hashlib
import os
import numpy as np

from . import geometry, graph, partition

CONFIGS = {
    "cfg1": dict(shape="sphere", levels=[2000], k=6, H=128, L=2, P=1, prec="fp32check"),
    "cfg2": dict(shape="car", levels=[100_000], k=6, H=128, L=15, P=1, prec="bf16"),
    "cfg3": dict(shape="car", levels=[50_000, 200_000, 800_000], k=6, H=512, L=15, P=8, prec="bf16"),
    "cfg4": dict(shape="car", levels=[500_000, 1_000_000, 2_000_000], k=6, H=512, L=15, P=8, prec="bf16"),
    "cfg5": dict(shape="car", levels=[2_500_000, 5_000_000, 10_000_000], k=6, H=512, L=15, P=32, prec="bf16"),
}

# Outside the repo so it never travels with a gpurun snapshot; only a cache
# (missing entries are regenerated deterministically).
CACHE = os.environ.get("XMGN_CACHE", os.path.join(os.path.expanduser("~"), ".cache", "xmgn_graphs"))


def build(shape, levels, k, P, halo, seed=0):
    pos, nrm = geometry.nested_levels(levels, shape=shape, seed=seed)
    offsets, sources = graph.multiscale_graph(pos, levels, k)
    owner = partition.rcb(pos, P)
    ps = partition.partition_set(offsets, sources, owner, P, halo)
    return dict(positions=pos, normals=nrm, offsets=offsets, sources=sources, owner=owner, **ps)


def checksum(bundle):
    h = hashlib.sha256()
    for key in sorted(bundle):
        a = np.ascontiguousarray(bundle[key])
        h.update(key.encode())
        h.update(a.tobytes())
    return h.hexdigest()


def load(name, halo=None, P=None, cache=True):
    """Graph + partition bundle for a named config (cached as .npz)."""
    c = CONFIGS[name]
    halo = c["L"] if halo is None else halo
    P = c["P"] if P is None else P
    tag = f"{name}_P{P}_h{halo}"
    path = os.path.join(CACHE, tag + ".npz")
    if cache and os.path.exists(path):
        with np.load(path) as z:
            return {k: z[k] for k in z.files}
    b = build(c["shape"], c["levels"], c["k"], P, halo)
    if cache:
        os.makedirs(CACHE, exist_ok=True)
        tmp = path + f".tmp{os.getpid()}.npz"
        np.savez(tmp, **b)
        os.replace(tmp, path)
    return b


def custom(n_levels=(300, 1500), k=6, P=4, halo=3, shape="sphere", seed=0):
    return build(shape, list(n_levels), k, P, halo, seed)
