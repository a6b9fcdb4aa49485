"""Plain oracle of the graph construction (NEXT-4) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/`` may import this module.  Each function is the definition written
out, in the paper's order (Sec. III-B/C; PAPER.md:231 k = 6,
halo 15), with the readings of SURVEY §8(c):

* kNN ("connecting each point to its k-nearest neighbors"): for node i
  the k = min(k, n - 1) nodes j != i with the smallest (d2(i, j), j), d2 evaluated
  in FP64 from the FP32 positions as ((dx dx) + (dy dy)) + dz dz (P12: ties by the
  smaller index).  Brute force over all pairs.
* symmetrise (P10) and multi-scale union (P11; "the point cloud
  from the previous scale is a subset of the point cloud at the next finer scale.
  Edge connectivity is determined at each scale"): per prefix level, edges (j -> i)
  and (i -> j) for j in kNN(i); the union over levels, deduplicated; CSR by
  destination with ascending sources.
* recursive coordinate bisection (the METIS stand-in): split the node
  set along the axis of largest extent (first such axis) at position
  round_half_even(n p_left / p), nodes ordered by (coordinate, id).
* halo rings ("the size of the halo region is set to be equal to the
  number of message passing layers"): ring(v) = undirected hop distance to the owned
  set when <= depth, by breadth-first search.

Pins: tests/test_graphbuild_oracle.py (hand-made examples from SPEC.md, a lattice with
exact ties, and agreement with the input generator's independent KD-tree / sparse-
matrix construction, itself pinned against brute force in tests/test_inputs.py).
"""
from collections import deque

import numpy as np


def d2(pos, i, j):
    p = np.asarray(pos, np.float32).astype(np.float64)
    dx, dy, dz = (p[j, c] - p[i, c] for c in range(3))
    return (dx * dx + dy * dy) + dz * dz


def knn(pos, k, block=512):
    """[n, k'] neighbours of every node, k' = min(k, n - 1), ordered by (d2, index)."""
    n = len(pos)
    kk = min(k, n - 1)
    p = np.asarray(pos, np.float32).astype(np.float64)
    out = np.empty((n, kk), np.int64)
    idx = np.arange(n)
    for a in range(0, n, block):
        q = np.arange(a, min(n, a + block))
        d = p[None, :, :] - p[q, None, :]
        dd = (d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2]
        dd[np.arange(len(q)), q] = np.inf
        for r, i in enumerate(q):
            out[i] = np.lexsort((idx, dd[r]))[:kk]
    return out


def multiscale_csr(pos, counts, k):
    """Union over prefix levels of the symmetrised kNN edges -> (offsets, sources)."""
    n = len(pos)
    edges = set()
    for c in counts:
        nb = knn(pos[:c], k)
        for i in range(c):
            for j in nb[i]:
                edges.add((i, int(j)))   # (dst, src): j -> i
                edges.add((int(j), i))   # and i -> j
    E = sorted(edges)
    offsets = np.zeros(n + 1, np.int64)
    for d, _ in E:
        offsets[d + 1] += 1
    return np.cumsum(offsets), np.array([s for _, s in E], np.int64)


def round_half_even(x):
    return int(np.round(x))   # numpy rounds halves to even, as Python's round()


def rcb(pos, P):
    """owner[n]: partition ids in recursion order (left = lower ids)."""
    p = np.asarray(pos, np.float32).astype(np.float64)
    owner = np.empty(len(p), np.int64)

    def rec(nodes, p0, np_):
        if np_ == 1:
            owner[nodes] = p0
            return
        pl = np_ // 2
        ext = [p[nodes, c].max() - p[nodes, c].min() for c in range(3)]
        ax = ext.index(max(ext))
        order = sorted(nodes, key=lambda v: (p[v, ax], v))
        nl = round_half_even(len(nodes) * pl / np_)
        rec(np.array(order[:nl], np.int64), p0, pl)
        rec(np.array(order[nl:], np.int64), p0 + pl, np_ - pl)

    rec(np.arange(len(p), dtype=np.int64), 0, P)
    return owner


def halo_rings(offsets, sources, owned, depth):
    """ring[v] (-1 beyond depth) by breadth-first search from the owned set."""
    n = len(offsets) - 1
    ring = np.full(n, -1, np.int64)
    dq = deque()
    for v in owned:
        ring[v] = 0
        dq.append(v)
    while dq:
        v = dq.popleft()
        if ring[v] == depth:
            continue
        for j in sources[offsets[v]:offsets[v + 1]]:   # symmetric graph: in = out neighbours
            if ring[j] < 0:
                ring[j] = ring[v] + 1
                dq.append(j)
    return ring


def partitions(offsets, sources, owner, P, depth):
    """owned / halo lists in the C-ABI layout (halo ordered by (ring, id))."""
    owned, halo, hring = [], [], []
    for p in range(P):
        ow = np.flatnonzero(owner == p)
        ring = halo_rings(offsets, sources, ow, depth)
        hv = [v for v in range(len(ring)) if ring[v] > 0]
        hv.sort(key=lambda v: (ring[v], v))
        owned.append(ow)
        halo.append(np.array(hv, np.int64))
        hring.append(ring[hv].astype(np.int32) if hv else np.zeros(0, np.int32))
    off = lambda L: np.concatenate([[0], np.cumsum([len(x) for x in L])]).astype(np.int64)  # noqa: E731
    return dict(owned_offsets=off(owned), owned=np.concatenate(owned), halo_offsets=off(halo),
                halo=np.concatenate(halo), halo_ring=np.concatenate(hring))


def build(pos, counts, k, P, depth):
    off, src = multiscale_csr(pos, counts, k)
    owner = rcb(pos, P)
    return dict(offsets=off, sources=src, owner=owner, **partitions(off, src, owner, P, depth))
