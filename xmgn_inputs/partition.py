"""Balanced partitioning and halo rings (untimed tooling).

* Recursive coordinate bisection (RCB) on the finest positions stands in for
  METIS (PAPER.md:172 uses METIS; SPEC.md:286 allows coordinate bisection): split
  along the widest axis at the (weighted) median, ties by node index.
* Halo of partition p at depth L = {v not owned by p : undirected hop distance
  (v, owned_p) <= L} ("The size of the halo region is set to be
  equal to the number of message passing layers").  Returned
  ordered by (ring, id) together with the ring of each halo node.
"""
import numpy as np
import scipy.sparse as sp


def rcb(pos, P):
    """Owner array (int64[n]); partition ids follow the recursion order."""
    n = len(pos)
    if not 1 <= P <= n:
        raise ValueError("need 1 <= P <= n")
    owner = np.empty(n, dtype=np.int64)

    def rec(idx, p0, np_):
        if np_ == 1:
            owner[idx] = p0
            return
        pl = np_ // 2
        sub = pos[idx].astype(np.float64)
        ax = int(np.argmax(sub.max(0) - sub.min(0)))
        order = np.lexsort((idx, sub[:, ax]))
        nl = int(round(len(idx) * pl / np_))
        rec(idx[order[:nl]], p0, pl)
        rec(idx[order[nl:]], p0 + pl, np_ - pl)

    rec(np.arange(n, dtype=np.int64), 0, P)
    return owner


def adjacency(offsets, sources):
    n = len(offsets) - 1
    data = np.ones(len(sources), dtype=np.float32)
    return sp.csr_matrix((data, sources, offsets), shape=(n, n))


def halo_rings(offsets, sources, owned_mask, depth, A=None):
    """ring[v] = hop distance to the owned set if <= depth, else -1."""
    if A is None:
        A = adjacency(offsets, sources)
    ring = np.full(len(owned_mask), -1, dtype=np.int32)
    ring[owned_mask] = 0
    frontier = owned_mask.astype(np.float32)
    for r in range(1, depth + 1):
        reach = (A @ frontier) > 0
        new = reach & (ring < 0)
        if not new.any():
            break
        ring[new] = r
        frontier = new.astype(np.float32)
    return ring


def partition_set(offsets, sources, owner, P, depth):
    """Concatenated owned/halo lists in the C-ABI layout."""
    A = adjacency(offsets, sources)
    owned, halo, hring = [], [], []
    for p in range(P):
        mask = owner == p
        ring = halo_rings(offsets, sources, mask, depth, A)
        owned.append(np.nonzero(mask)[0].astype(np.int64))
        hv = np.nonzero(ring > 0)[0]
        order = np.lexsort((hv, ring[hv]))
        halo.append(hv[order].astype(np.int64))
        hring.append(ring[hv[order]].astype(np.int32))
    off = lambda L: np.concatenate([[0], np.cumsum([len(x) for x in L])]).astype(np.int64)  # noqa: E731
    return dict(owned_offsets=off(owned), owned=np.concatenate(owned),
                halo_offsets=off(halo), halo=np.concatenate(halo) if halo else np.zeros(0, np.int64),
                halo_ring=np.concatenate(hring) if hring else np.zeros(0, np.int32))
