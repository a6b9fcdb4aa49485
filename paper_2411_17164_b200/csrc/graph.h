// Host-side graph handle: per-partition local arrays (ring-major numbering).
#pragma once
#include <cstdint>
#include <vector>
#include "xmgn_internal.h"

namespace xmgn {

struct Part {
  int64_t n_owned = 0, n_local = 0, e_local = 0;
  int32_t depth = 0;
  std::vector<int64_t> gid;       // local -> global node id
  std::vector<int32_t> ring;      // ring of each local node
  std::vector<int64_t> offsets;   // local CSR by destination [n_local+1]
  std::vector<int32_t> src, dst;  // local endpoints of each local edge
  std::vector<int64_t> edge_gid;  // local -> global edge index (global CSR position)
  std::vector<int32_t> rev;       // reverse local edge
  int64_t ring_nodes[65] = {0}, ring_edges[65] = {0};
};

}  // namespace xmgn

struct xmgn_graph {
  int device = 0;
  int64_t n_nodes = 0, n_edges = 0;
  int32_t depth = 0;
  std::vector<xmgn::Part> parts;
};
