"""Synthetic surface point clouds (untimed tooling).

* Unit sphere (CFG1): x = g/|g|, g ~ N(0, I3) from PCG64(seed).
* Car proxy (CFG2-5): a closed superellipsoid with semi-axes (2.30, 0.95, 0.70) m,
  tessellated and sampled area-uniformly with the sqrt-barycentric map
  (SPEC.md:58-61).  The paper samples the DrivAerML STL surface (PAPER.md:217,
  231); we have no dataset, so this is a shape-alike with the same point counts.
* Levels are prefix-nested: level i's points are the first n_i points of level
  i+1 ("The points from the initial point cloud serve as a subset
  of the finer point cloud").  Each level appends fresh samples
  drawn from its own sub-seed.
"""
import numpy as np


def _rng(seed, sub):
    return np.random.Generator(np.random.PCG64([int(seed), int(sub)]))


def sphere_points(n, seed=0, sub=0):
    g = _rng(seed, sub).standard_normal((n, 3))
    x = g / np.linalg.norm(g, axis=1, keepdims=True)
    return x.astype(np.float32), x.astype(np.float32)  # positions, normals


def _superellipsoid_mesh(axes=(2.30, 0.95, 0.70), e=0.45, nu=256, nv=128):
    a, b, c = axes
    u = np.linspace(0.0, 2.0 * np.pi, nu, endpoint=False)
    v = np.linspace(-0.5 * np.pi, 0.5 * np.pi, nv + 1)
    f = lambda w, p: np.sign(w) * np.abs(w) ** p  # noqa: E731
    cv, sv = np.cos(v)[:, None], np.sin(v)[:, None]
    cu, su = np.cos(u)[None, :], np.sin(u)[None, :]
    x = a * f(cv, e) * f(cu, e)
    y = b * f(cv, e) * f(su, e)
    z = c * f(sv, e) * np.ones_like(cu)
    verts = np.stack([x, y, z], -1).reshape(-1, 3)
    tris = []
    for i in range(nv):
        for j in range(nu):
            p00 = i * nu + j
            p01 = i * nu + (j + 1) % nu
            p10 = (i + 1) * nu + j
            p11 = (i + 1) * nu + (j + 1) % nu
            tris.append((p00, p10, p11))
            tris.append((p00, p11, p01))
    tris = np.asarray(tris, dtype=np.int64)
    A, B, C = verts[tris[:, 0]], verts[tris[:, 1]], verts[tris[:, 2]]
    cr = np.cross(B - A, C - A)
    area = 0.5 * np.linalg.norm(cr, axis=1)
    keep = area > 1e-14
    A, B, C, cr, area = A[keep], B[keep], C[keep], cr[keep], area[keep]
    nrm = cr / np.linalg.norm(cr, axis=1, keepdims=True)
    return A, B, C, nrm, area


_MESH = None


def car_points(n, seed=0, sub=0):
    """Area-uniform samples on the car-proxy surface (sqrt-barycentric map)."""
    global _MESH
    if _MESH is None:
        _MESH = _superellipsoid_mesh()
    A, B, C, nrm, area = _MESH
    rng = _rng(seed, sub)
    cdf = np.cumsum(area)
    cdf /= cdf[-1]
    t = np.searchsorted(cdf, rng.random(n), side="right")
    t = np.minimum(t, len(area) - 1)
    r1, r2 = rng.random(n), rng.random(n)
    s = np.sqrt(r1)[:, None]
    r2 = r2[:, None]
    p = (1.0 - s) * A[t] + s * (1.0 - r2) * B[t] + s * r2 * C[t]
    return p.astype(np.float32), nrm[t].astype(np.float32)


def nested_levels(counts, shape="car", seed=0):
    """Prefix-nested multi-level cloud: returns positions/normals of the finest
    level (n_{S-1} points); level i is the prefix [0, counts[i])."""
    counts = [int(c) for c in counts]
    if any(b <= a for a, b in zip(counts, counts[1:])) or counts[0] <= 0:
        raise ValueError("level counts must be positive and strictly increasing")
    gen = car_points if shape == "car" else sphere_points
    pos, nrm = [], []
    prev = 0
    for i, c in enumerate(counts):
        p, q = gen(c - prev, seed=seed, sub=i)
        pos.append(p)
        nrm.append(q)
        prev = c
    return np.concatenate(pos), np.concatenate(nrm)
