// xmgn_load_graph: validation and per-partition staging.
//
// Staging follows PAPER.md:170-174 (Sec. III-A): each partition is its owned set
// plus the halo of nodes within halo_depth undirected hops, and is processed as
// an independent graph.  Local numbering is ring-major (owned, then ring 1..d,
// ascending global id inside a ring) so that
//   * the owned rows are the prefix [0, n_owned)  -> loss mask is implicit
//     (PAPER.md:197), and
//   * the destinations that layer l must still update (ring <= L-l) are a prefix
//     of the nodes AND of the dst-sorted edges (halo shrinking).
// Local in-edges keep the global CSR order (edges whose source is not local are
// dropped), which makes the partitioned aggregation sum in exactly
// the full graph's order.  rev[k] indexes the reverse edge (the graph is
// symmetric), used for the deterministic source-side gradient sums.
#include <algorithm>
#include <cstring>
#include <vector>
#include <omp.h>
#include "graph.h"

namespace xmgn {

static xmgn_status validate_csr(const xmgn_graph_desc* d) {
  const int64_t N = d->n_nodes, E = d->n_edges;
  const int64_t* off = d->csr_offsets;
  const int64_t* src = d->csr_sources;
  if (N <= 0 || E < 0 || !off || (!src && E > 0))
    return set_error(XMGN_EINVAL, "xmgn_load_graph: n_nodes=%lld n_edges=%lld or null CSR arrays", (long long)N,
                     (long long)E);
  if (off[0] != 0) return set_error(XMGN_EINVAL, "xmgn_load_graph: csr_offsets[0]=%lld != 0", (long long)off[0]);
  if (off[N] != E)
    return set_error(XMGN_EINVAL, "xmgn_load_graph: csr_offsets[%lld]=%lld != n_edges=%lld", (long long)N,
                     (long long)off[N], (long long)E);
  for (int64_t i = 0; i < N; ++i)
    if (off[i + 1] < off[i])
      return set_error(XMGN_EINVAL, "xmgn_load_graph: csr_offsets not monotone at index %lld", (long long)i);
  for (int64_t i = 0; i < N; ++i) {
    for (int64_t k = off[i]; k < off[i + 1]; ++k) {
      int64_t j = src[k];
      if (j < 0 || j >= N)
        return set_error(XMGN_EINVAL, "xmgn_load_graph: csr_sources[%lld]=%lld out of range [0,%lld)",
                         (long long)k, (long long)j, (long long)N);
      if (j == i) return set_error(XMGN_EINVAL, "xmgn_load_graph: self-loop at csr_sources[%lld] (node %lld)",
                                   (long long)k, (long long)i);
      if (k > off[i] && src[k - 1] >= j)
        return set_error(XMGN_EINVAL,
                         "xmgn_load_graph: csr_sources not strictly ascending in row %lld at index %lld "
                         "(duplicate or unsorted)",
                         (long long)i, (long long)k);
    }
  }
  // symmetry: (j -> i) present  =>  (i -> j) present
  int64_t bad = -1;
#pragma omp parallel for schedule(static) reduction(max : bad)
  for (int64_t i = 0; i < N; ++i)
    for (int64_t k = off[i]; k < off[i + 1]; ++k) {
      int64_t j = src[k];
      if (!std::binary_search(src + off[j], src + off[j + 1], i)) bad = std::max(bad, k);
    }
  if (bad >= 0)
    return set_error(XMGN_EINVAL, "xmgn_load_graph: graph not symmetric: reverse of edge csr_sources[%lld] missing",
                     (long long)bad);
  return XMGN_OK;
}

static xmgn_status validate_parts(const xmgn_graph_desc* d) {
  const int64_t N = d->n_nodes;
  const int P = d->n_parts;
  if (P <= 0 || d->halo_depth < 0 || d->halo_depth > 63 || !d->owned_offsets || !d->owned || !d->halo_offsets)
    return set_error(XMGN_EINVAL, "xmgn_load_graph: n_parts=%d halo_depth=%d (0..63) or null partition arrays", P,
                     d->halo_depth);
  if (d->owned_offsets[0] != 0 || d->owned_offsets[P] != N)
    return set_error(XMGN_EINVAL, "xmgn_load_graph: owned_offsets must span [0, n_nodes]");
  std::vector<int32_t> owner(N, -1);
  for (int p = 0; p < P; ++p) {
    int64_t a = d->owned_offsets[p], b = d->owned_offsets[p + 1];
    if (b <= a) return set_error(XMGN_EINVAL, "xmgn_load_graph: owned_offsets: partition %d is empty", p);
    for (int64_t t = a; t < b; ++t) {
      int64_t v = d->owned[t];
      if (v < 0 || v >= N) return set_error(XMGN_EINVAL, "xmgn_load_graph: owned[%lld]=%lld out of range", (long long)t, (long long)v);
      if (t > a && d->owned[t - 1] >= v)
        return set_error(XMGN_EINVAL, "xmgn_load_graph: owned list of partition %d not ascending at owned[%lld]", p,
                         (long long)t);
      if (owner[v] >= 0)
        return set_error(XMGN_EINVAL, "xmgn_load_graph: node %lld owned by partitions %d and %d", (long long)v,
                         owner[v], p);
      owner[v] = p;
    }
  }
  if (d->halo_offsets[0] != 0) return set_error(XMGN_EINVAL, "xmgn_load_graph: halo_offsets[0] != 0");
  for (int p = 0; p < P; ++p) {
    int64_t a = d->halo_offsets[p], b = d->halo_offsets[p + 1];
    if (b < a) return set_error(XMGN_EINVAL, "xmgn_load_graph: halo_offsets not monotone at %d", p);
    for (int64_t t = a; t < b; ++t) {
      int64_t v = d->halo[t];
      int32_t r = d->halo_ring[t];
      if (v < 0 || v >= N) return set_error(XMGN_EINVAL, "xmgn_load_graph: halo[%lld]=%lld out of range", (long long)t, (long long)v);
      if (r < 1 || r > d->halo_depth)
        return set_error(XMGN_EINVAL, "xmgn_load_graph: halo_ring[%lld]=%d outside 1..%d", (long long)t, r,
                         d->halo_depth);
      if (owner[v] == p)
        return set_error(XMGN_EINVAL, "xmgn_load_graph: halo[%lld]=%lld is owned by its own partition %d",
                         (long long)t, (long long)v, p);
      if (t > a) {
        int32_t rp = d->halo_ring[t - 1];
        if (rp > r || (rp == r && d->halo[t - 1] >= v))
          return set_error(XMGN_EINVAL, "xmgn_load_graph: halo of partition %d not ordered by (ring, id) at halo[%lld]",
                           p, (long long)t);
      }
    }
  }
  return XMGN_OK;
}

// Independent BFS (undirected = in-neighbours on a symmetric graph): the halo
// lists must be exactly the rings 1..depth.
static xmgn_status check_halo_bfs(const xmgn_graph_desc* d) {
  const int64_t N = d->n_nodes;
  const int P = d->n_parts;
  std::vector<int> bad(P, 0);
  std::vector<int64_t> bad_node(P, -1);
#pragma omp parallel
  {
    std::vector<int32_t> dist(N, -1);
    std::vector<int64_t> frontier, next, touched;
#pragma omp for schedule(dynamic, 1)
    for (int p = 0; p < P; ++p) {
      touched.clear();
      frontier.assign(d->owned + d->owned_offsets[p], d->owned + d->owned_offsets[p + 1]);
      for (int64_t v : frontier) { dist[v] = 0; touched.push_back(v); }
      for (int r = 1; r <= d->halo_depth; ++r) {
        next.clear();
        for (int64_t v : frontier)
          for (int64_t k = d->csr_offsets[v]; k < d->csr_offsets[v + 1]; ++k) {
            int64_t u = d->csr_sources[k];
            if (dist[u] < 0) { dist[u] = r; next.push_back(u); touched.push_back(u); }
          }
        frontier.swap(next);
      }
      int64_t nh = (int64_t)touched.size() - (d->owned_offsets[p + 1] - d->owned_offsets[p]);
      if (nh != d->halo_offsets[p + 1] - d->halo_offsets[p]) { bad[p] = 1; }
      for (int64_t t = d->halo_offsets[p]; t < d->halo_offsets[p + 1] && !bad[p]; ++t)
        if (dist[d->halo[t]] != d->halo_ring[t]) { bad[p] = 2; bad_node[p] = d->halo[t]; }
      for (int64_t v : touched) dist[v] = -1;
    }
  }
  for (int p = 0; p < P; ++p)
    if (bad[p])
      return set_error(XMGN_EHALO,
                       "xmgn_load_graph: halo of partition %d is not the %d-hop BFS ring set (%s, node %lld)", p,
                       d->halo_depth, bad[p] == 1 ? "size differs" : "ring differs", (long long)bad_node[p]);
  return XMGN_OK;
}

static void stage_partition(const xmgn_graph_desc* d, int p, Part& P, std::vector<int32_t>& lid) {
  const int64_t* off = d->csr_offsets;
  const int64_t* src = d->csr_sources;
  const int64_t no = d->owned_offsets[p + 1] - d->owned_offsets[p];
  const int64_t nh = d->halo_offsets[p + 1] - d->halo_offsets[p];
  const int64_t nl = no + nh;
  P.n_owned = no;
  P.n_local = nl;
  P.depth = d->halo_depth;
  P.gid.resize(nl);
  P.ring.resize(nl);
  for (int64_t t = 0; t < no; ++t) { P.gid[t] = d->owned[d->owned_offsets[p] + t]; P.ring[t] = 0; }
  for (int64_t t = 0; t < nh; ++t) {
    P.gid[no + t] = d->halo[d->halo_offsets[p] + t];
    P.ring[no + t] = d->halo_ring[d->halo_offsets[p] + t];
  }
  for (int64_t t = 0; t < nl; ++t) lid[P.gid[t]] = (int32_t)t;
  P.offsets.assign(nl + 1, 0);
  P.src.clear();
  P.edge_gid.clear();
  for (int64_t t = 0; t < nl; ++t) {
    int64_t v = P.gid[t];
    for (int64_t k = off[v]; k < off[v + 1]; ++k) {
      int32_t j = lid[src[k]];
      if (j >= 0) { P.src.push_back(j); P.edge_gid.push_back(k); }
    }
    P.offsets[t + 1] = (int64_t)P.src.size();
  }
  const int64_t el = (int64_t)P.src.size();
  P.e_local = el;
  P.dst.resize(el);
  for (int64_t t = 0; t < nl; ++t)
    for (int64_t k = P.offsets[t]; k < P.offsets[t + 1]; ++k) P.dst[k] = (int32_t)t;
  // reverse edge: (j -> i) at k  <->  (i -> j) in row j; row j is ordered by
  // ascending GLOBAL source id, so binary-search on global ids.
  P.rev.assign(el, -1);
  for (int64_t k = 0; k < el; ++k) {
    int32_t i = P.dst[k], j = P.src[k];
    int64_t gi = P.gid[i];
    int64_t lo = P.offsets[j], hi = P.offsets[j + 1];
    while (lo < hi) {
      int64_t mid = (lo + hi) / 2;
      if (P.gid[P.src[mid]] < gi) lo = mid + 1; else hi = mid;
    }
    if (lo < P.offsets[j + 1] && P.src[lo] == i) P.rev[k] = (int32_t)lo;
  }
  for (int r = 0; r <= P.depth + 1; ++r) {
    int64_t n = 0;
    while (n < nl && P.ring[n] < r) ++n;
    P.ring_nodes[r] = n;
    P.ring_edges[r] = P.offsets[n];
  }
  for (int64_t t = 0; t < nl; ++t) lid[P.gid[t]] = -1;
}

}  // namespace xmgn

using namespace xmgn;

extern "C" xmgn_status xmgn_load_graph(const xmgn_graph_desc* desc, int cuda_device, xmgn_graph** out) {
  return guarded("xmgn_load_graph", [&]() -> xmgn_status {
    if (!desc || !out) return set_error(XMGN_EINVAL, "xmgn_load_graph: null argument");
    *out = nullptr;
    xmgn_status s;
    if ((s = validate_csr(desc)) != XMGN_OK) return s;
    if ((s = validate_parts(desc)) != XMGN_OK) return s;
    if ((s = check_halo_bfs(desc)) != XMGN_OK) return s;
    auto* g = new xmgn_graph();
    g->device = cuda_device;
    g->n_nodes = desc->n_nodes;
    g->n_edges = desc->n_edges;
    g->depth = desc->halo_depth;
    g->parts.resize(desc->n_parts);
    std::vector<int32_t> lid(desc->n_nodes, -1);
    for (int p = 0; p < desc->n_parts; ++p) stage_partition(desc, p, g->parts[p], lid);
    for (auto& P : g->parts)
      for (int64_t k = 0; k < P.e_local; ++k)
        if (P.rev[k] < 0) {
          int64_t e = P.e_local;
          delete g;
          return set_error(XMGN_EINVAL, "xmgn_load_graph: reverse of local edge %lld missing (e_local=%lld)",
                           (long long)k, (long long)e);
        }
    *out = g;
    return XMGN_OK;
  });
}

extern "C" xmgn_status xmgn_part_info_get(const xmgn_graph* g, int part, xmgn_part_info* out) {
  if (!g || !out || part < 0 || part >= (int)g->parts.size())
    return set_error(XMGN_EINVAL, "xmgn_part_info_get: bad handle or part %d", part);
  const Part& P = g->parts[part];
  std::memset(out, 0, sizeof(*out));
  out->n_owned = P.n_owned;
  out->n_local = P.n_local;
  out->e_local = P.e_local;
  out->depth = P.depth;
  for (int r = 0; r <= P.depth + 1; ++r) { out->ring_nodes[r] = P.ring_nodes[r]; out->ring_edges[r] = P.ring_edges[r]; }
  return XMGN_OK;
}

extern "C" xmgn_status xmgn_export_part(const xmgn_graph* g, int part, int64_t* gid, int64_t* loff, int64_t* lsrc,
                                        int64_t* legid, int64_t* rev) {
  if (!g || part < 0 || part >= (int)g->parts.size())
    return set_error(XMGN_EINVAL, "xmgn_export_part: bad handle or part %d", part);
  const Part& P = g->parts[part];
  for (int64_t t = 0; t < P.n_local; ++t) {
    if (gid) gid[t] = P.gid[t];
  }
  if (loff)
    for (int64_t t = 0; t <= P.n_local; ++t) loff[t] = P.offsets[t];
  for (int64_t k = 0; k < P.e_local; ++k) {
    if (lsrc) lsrc[k] = P.src[k];
    if (legid) legid[k] = P.edge_gid[k];
    if (rev) rev[k] = P.rev[k];
  }
  return XMGN_OK;
}

extern "C" void xmgn_free_graph(xmgn_graph* g) { delete g; }
