"""kNN connectivity, symmetrisation, multi-scale union and CSR by destination.

* kNN (Sec. III-B; k=6 per PAPER.md:231): for node i, edges
  (j -> i) for the k nearest distinct j.  Squared distances are evaluated in
  FP64 from FP32 positions as ((dx*dx)+(dy*dy))+(dz*dz); ties are broken by the
  smaller index.  A kd-tree proposes candidates; the (d2, index)
  re-sort makes the result equal to brute force.
* Symmetrise so halo hops are undirected hops.
* Multi-scale: kNN per prefix level, symmetrised, union of all
  levels, deduplicated; node set = finest level.
* CSR by destination: ``offsets`` i64[N+1], ``sources`` i64[E] strictly
  ascending within a row.
"""
import numpy as np
from scipy.spatial import cKDTree


def _d2(pos, i, j):
    p = pos.astype(np.float64)
    d = p[j] - p[i]
    return (d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2]


def knn_brute(pos, k):
    """O(n^2) reference: in-neighbours (n, k) of every node under the tie rule."""
    n = len(pos)
    k = min(k, n - 1)
    out = np.empty((n, k), dtype=np.int64)
    idx = np.arange(n)
    for i in range(n):
        d2 = _d2(pos, np.full(n, i), idx)
        d2[i] = np.inf
        order = np.lexsort((idx, d2))
        out[i] = order[:k]
    return out


def knn(pos, k, workers=-1):
    """kd-tree candidates + exact (d2, index) selection (equals ``knn_brute``)."""
    n = len(pos)
    k = min(k, n - 1)
    tree = cKDTree(pos.astype(np.float64))
    q = min(n, k + 5)
    out = np.empty((n, k), dtype=np.int64)
    todo = np.arange(n)
    while len(todo):
        _, cand = tree.query(pos[todo].astype(np.float64), k=q, workers=workers)
        cand = np.asarray(cand, dtype=np.int64).reshape(len(todo), q)
        d2 = _d2(pos, todo[:, None], cand)
        worst = d2.max(1)                           # farthest proposed candidate
        d2[cand == todo[:, None]] = np.inf          # drop self
        order = np.lexsort((cand, d2), axis=1)
        cs = np.take_along_axis(cand, order, 1)
        ds = np.take_along_axis(d2, order, 1)
        # exact iff the k-th kept distance is strictly below the worst candidate
        # (otherwise an equal-distance point with a smaller index may be missing)
        ok = (ds[:, k - 1] < worst) | (q >= n)
        out[todo[ok]] = cs[ok, :k]
        todo = todo[~ok]
        q = min(n, 2 * q)
    return out


def knn_edges(pos, k, **kw):
    """Directed edges (src=j, dst=i) for j in kNN(i)."""
    nb = knn(pos, k, **kw)
    dst = np.repeat(np.arange(len(pos), dtype=np.int64), nb.shape[1])
    return nb.reshape(-1), dst


def symmetrize(src, dst):
    s = np.concatenate([src, dst])
    d = np.concatenate([dst, src])
    return s, d


def to_csr(src, dst, n):
    """Deduplicate, drop self-loops and sort by (dst, src)."""
    keep = src != dst
    key = np.unique(dst[keep].astype(np.int64) * n + src[keep].astype(np.int64))
    d = key // n
    s = key - d * n
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.add.at(offsets, d + 1, 1)
    np.cumsum(offsets, out=offsets)
    return offsets, s.astype(np.int64)


def multiscale_graph(pos, counts, k, **kw):
    """Union of per-level symmetrised kNN graphs over prefix-nested levels."""
    n = len(pos)
    S, D = [], []
    for c in counts:
        s, d = knn_edges(pos[:c], k, **kw)
        s, d = symmetrize(s, d)
        S.append(s)
        D.append(d)
    return to_csr(np.concatenate(S), np.concatenate(D), n)
