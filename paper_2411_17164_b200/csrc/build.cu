// Graph construction on the GPU (NEXT-4; Sec. III-B/C,
// PAPER.md:231 "3-level graph ... Each node is connected to its 6 nearest neighbors ... halo
// size of 15"), read per SURVEY §8(c) P10-P14:
//   * kNN per prefix level, exact under the tie rule: d2 in FP64 from the FP32 positions as
//     ((dx dx) + (dy dy)) + dz dz (no contraction), ties by the smaller index (P12).  Points are
//     binned in a uniform cell grid (one 64-bit key radix sort); a query visits cubic shells of
//     cells until its k-th distance is strictly below the distance to any unvisited cell;
//   * symmetrise + union over levels + CSR by destination (P10, P11): one radix sort of 64-bit
//     (dst, src) keys and a unique pass;
//   * recursive coordinate bisection (the METIS stand-in): per segment the axis of
//     largest extent, a radix sort of (coordinate, id) keys, the split at round-half-even(n p_l/p);
//   * halo rings: level-synchronous BFS (pull form, deterministic) from each owned set, then the
//     (ring, id)-ordered halo lists by stable selection.
// Sorting / selection use CUB (the CUDA toolkit's device primitives); everything else is here.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <cuda_runtime.h>
#include <cfloat>
#include <cmath>
#include <cstring>
#include <vector>
#include "xmgn_internal.h"
#include "kernels_launch.h"

struct xmgn_built_graph {
  int64_t n = 0, E = 0;
  int P = 0, depth = 0;
  std::vector<int64_t> offsets, sources, owner, owned_offsets, owned, halo_offsets, halo;
  std::vector<int32_t> halo_ring;
};

namespace xmgn {
namespace {

template <class T>
struct DBuf {   // device buffer (RAII)
  T* p = nullptr;
  size_t n = 0;
  explicit DBuf(size_t count = 0) { alloc(count); }
  void alloc(size_t count) {
    free();
    n = count;
    if (count) XMGN_CUDA(cudaMalloc(&p, count * sizeof(T)), "xmgn_build_graph: cudaMalloc");
  }
  void free() {
    if (p) cudaFree(p);
    p = nullptr;
  }
  ~DBuf() { free(); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
};

struct Temp {   // CUB temporary storage, grown on demand
  DBuf<uint8_t> b;
  void* get(size_t bytes) {
    if (bytes > b.n) b.alloc(bytes);
    return b.p;
  }
};

struct Grid {
  float lo[3];
  float inv_h;
  double h;
  int nc[3];
};

__device__ __forceinline__ int cell_of(float x, float lo, float inv_h, int nc) {
  int c = (int)floorf((x - lo) * inv_h);
  return c < 0 ? 0 : (c >= nc ? nc - 1 : c);
}
__device__ __forceinline__ uint64_t cell_key(int cx, int cy, int cz, const Grid& g) {
  return ((uint64_t)cx * (uint64_t)g.nc[1] + (uint64_t)cy) * (uint64_t)g.nc[2] + (uint64_t)cz;
}

// key = cell << 32 | id, so one sort gives the cell-major point order
__global__ void k_cell_keys(const float* __restrict__ pos, int c, Grid g, uint64_t* __restrict__ keys) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < c; i += gridDim.x * blockDim.x) {
    const int cx = cell_of(pos[3 * i], g.lo[0], g.inv_h, g.nc[0]);
    const int cy = cell_of(pos[3 * i + 1], g.lo[1], g.inv_h, g.nc[1]);
    const int cz = cell_of(pos[3 * i + 2], g.lo[2], g.inv_h, g.nc[2]);
    keys[i] = (cell_key(cx, cy, cz, g) << 32) | (uint32_t)i;
  }
}

// sorted keys -> point order, sorted positions, and the cell key of each sorted slot
__global__ void k_split_keys(const uint64_t* __restrict__ sk, const float* __restrict__ pos, int c,
                             int* __restrict__ order, float* __restrict__ spos, uint64_t* __restrict__ cells) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < c; t += gridDim.x * blockDim.x) {
    const int i = (int)(uint32_t)sk[t];
    order[t] = i;
    spos[3 * t] = pos[3 * i];
    spos[3 * t + 1] = pos[3 * i + 1];
    spos[3 * t + 2] = pos[3 * i + 2];
    cells[t] = sk[t] >> 32;
  }
}

__device__ __forceinline__ int lower_bound_u64(const uint64_t* a, int n, uint64_t x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

constexpr int K_MAX = 16;

// one thread per query (queries taken in cell order for locality); exact k nearest under the
// (d2, index) order.  After shells 0..r every unvisited point is at distance >= r h (up to the
// rounding of the cell assignment, covered by `slack`), so the search stops once the k-th d2 is
// strictly below (r h - slack)^2.
__global__ void __launch_bounds__(128) k_knn(const float* __restrict__ spos, const int* __restrict__ order,
                                             const uint64_t* __restrict__ ucell, const int* __restrict__ ustart,
                                             int nu, int c, int k, Grid g, double slack, int rmax,
                                             int* __restrict__ nb) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= c) return;
  const int i = order[t];
  const float px = spos[3 * t], py = spos[3 * t + 1], pz = spos[3 * t + 2];
  const double qx = px, qy = py, qz = pz;
  const int cx = cell_of(px, g.lo[0], g.inv_h, g.nc[0]);
  const int cy = cell_of(py, g.lo[1], g.inv_h, g.nc[1]);
  const int cz = cell_of(pz, g.lo[2], g.inv_h, g.nc[2]);
  double bd[K_MAX];
  int bj[K_MAX];
  int cnt = 0;
  for (int r = 0; r <= rmax; ++r) {
    for (int dx = -r; dx <= r; ++dx) {
      const int x = cx + dx;
      if (x < 0 || x >= g.nc[0]) continue;
      for (int dy = -r; dy <= r; ++dy) {
        const int y = cy + dy;
        if (y < 0 || y >= g.nc[1]) continue;
        const bool edge_xy = dx == -r || dx == r || dy == -r || dy == r;
        for (int dz = -r; dz <= r; dz += (edge_xy ? 1 : (r > 0 ? 2 * r : 1))) {
          const int z = cz + dz;
          if (z < 0 || z >= g.nc[2]) continue;
          const uint64_t key = cell_key(x, y, z, g);
          const int u = lower_bound_u64(ucell, nu, key);
          if (u >= nu || ucell[u] != key) continue;
          for (int s = ustart[u]; s < ustart[u + 1]; ++s) {
            const int j = order[s];
            if (j == i) continue;
            const double ex = __dsub_rn((double)spos[3 * s], qx);
            const double ey = __dsub_rn((double)spos[3 * s + 1], qy);
            const double ez = __dsub_rn((double)spos[3 * s + 2], qz);
            const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey)), __dmul_rn(ez, ez));
            if (cnt == k && (d2 > bd[k - 1] || (d2 == bd[k - 1] && j > bj[k - 1]))) continue;
            int q = cnt < k ? cnt++ : k - 1;   // insertion position from the back
            while (q > 0 && (bd[q - 1] > d2 || (bd[q - 1] == d2 && bj[q - 1] > j))) {
              bd[q] = bd[q - 1];
              bj[q] = bj[q - 1];
              --q;
            }
            bd[q] = d2;
            bj[q] = j;
          }
        }
      }
    }
    if (cnt == k) {
      const double b = r * g.h - slack;
      if (b > 0 && bd[k - 1] < b * b) break;
    }
  }
  for (int q = 0; q < k; ++q) nb[(size_t)i * k + q] = bj[q];
}

// both directions of every kNN edge of a level: key = dst * n + src
__global__ void k_edge_keys(const int* __restrict__ nb, int c, int k, uint64_t n, uint64_t* __restrict__ keys) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)c * k;
       t += (long long)gridDim.x * blockDim.x) {
    const uint64_t i = (uint64_t)(t / k), j = (uint64_t)nb[t];
    keys[2 * t] = i * n + j;       // j -> i
    keys[2 * t + 1] = j * n + i;   // i -> j
  }
}

__global__ void k_csr(const uint64_t* __restrict__ keys, long long E, uint64_t n, int64_t* __restrict__ offsets,
                      int64_t* __restrict__ sources) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < E; e += (long long)gridDim.x * blockDim.x)
    sources[e] = (int64_t)(keys[e] % n);
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v <= (long long)n;
       v += (long long)gridDim.x * blockDim.x) {
    long long lo = 0, hi = E;
    const uint64_t x = (uint64_t)v * n;
    while (lo < hi) {
      const long long mid = (lo + hi) >> 1;
      if (keys[mid] < x) lo = mid + 1;
      else hi = mid;
    }
    offsets[v] = lo;
  }
}

__device__ __forceinline__ uint32_t orderable(float f) {
  if (f == 0.0f) f = 0.0f;   // -0 == +0 in the oracle's comparison
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// RCB: coordinate `ax` of the segment's nodes -> (coordinate, id) keys
__global__ void k_rcb_keys(const float* __restrict__ pos, const int* __restrict__ perm, int len, int ax,
                           uint64_t* __restrict__ keys) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < len; t += gridDim.x * blockDim.x) {
    const int v = perm[t];
    keys[t] = ((uint64_t)orderable(pos[3 * (size_t)v + ax]) << 32) | (uint32_t)v;
  }
}
__global__ void k_rcb_unkey(const uint64_t* __restrict__ keys, int len, int* __restrict__ perm) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < len; t += gridDim.x * blockDim.x)
    perm[t] = (int)(uint32_t)keys[t];
}
// per-segment bounding box: block-local min / max, then a fixed-order second pass
__global__ void k_bbox(const float* __restrict__ pos, const int* __restrict__ perm, int len, float* __restrict__ part) {
  float mn[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, mx[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < len; t += gridDim.x * blockDim.x) {
    const int v = perm ? perm[t] : t;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float x = pos[3 * (size_t)v + c];
      mn[c] = fminf(mn[c], x);
      mx[c] = fmaxf(mx[c], x);
    }
  }
  __shared__ float s[6][256];
#pragma unroll
  for (int c = 0; c < 3; ++c) { s[c][threadIdx.x] = mn[c]; s[3 + c][threadIdx.x] = mx[c]; }
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        s[c][threadIdx.x] = fminf(s[c][threadIdx.x], s[c][threadIdx.x + w]);
        s[3 + c][threadIdx.x] = fmaxf(s[3 + c][threadIdx.x], s[3 + c][threadIdx.x + w]);
      }
    __syncthreads();
  }
  if (threadIdx.x < 6) part[blockIdx.x * 6 + threadIdx.x] = s[threadIdx.x][0];
}
__global__ void k_set_owner(const int* __restrict__ perm, int len, int p, int64_t* __restrict__ owner) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < len; t += gridDim.x * blockDim.x) owner[perm[t]] = p;
}

// BFS (pull): v joins ring r if any in-neighbour (= neighbour, symmetric graph) is in ring r - 1
__global__ void k_ring_init(const int64_t* __restrict__ owner, int n, int p, int* __restrict__ ring) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    ring[v] = owner[v] == p ? 0 : -1;
}
__global__ void k_ring_step(const int64_t* __restrict__ off, const int64_t* __restrict__ src, int n, int r,
                            int* __restrict__ ring) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    if (ring[v] != -1) continue;
    for (int64_t e = off[v]; e < off[v + 1]; ++e)
      if (ring[src[e]] == r - 1) { ring[v] = r; break; }
  }
}
struct OwnedBy {
  const int64_t* owner;
  int p;
  __device__ bool operator()(int v) const { return owner[v] == p; }
};
struct InRing {
  const int* ring;
  int r;
  __device__ bool operator()(int v) const { return ring[v] == r; }
};
__global__ void k_iota(int* __restrict__ a, int n) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) a[t] = t;
}
__global__ void k_i32_to_i64(const int* __restrict__ a, int n, int64_t* __restrict__ b) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) b[t] = a[t];
}

inline int blocks_for(long long n, int threads = 256) {
  return (int)std::max<long long>(1, std::min<long long>((n + threads - 1) / threads, 148LL * 32));
}

}  // namespace
}  // namespace xmgn

using namespace xmgn;

extern "C" xmgn_status xmgn_build_graph(const float* pos, int64_t n_nodes, const int64_t* level_counts,
                                        int n_levels, int k, int n_parts, int halo_depth, int cuda_device,
                                        void* stream, xmgn_built_graph** out) {
  return guarded("xmgn_build_graph", [&]() -> xmgn_status {
    if (!pos || !level_counts || !out) return set_error(XMGN_EINVAL, "xmgn_build_graph: null argument");
    *out = nullptr;
    const int64_t n = n_nodes;
    if (n < 2 || n >= (1LL << 31)) return set_error(XMGN_EINVAL, "xmgn_build_graph: n_nodes=%lld", (long long)n);
    if (n_levels < 1 || level_counts[n_levels - 1] != n)
      return set_error(XMGN_EINVAL, "xmgn_build_graph: level_counts must end at n_nodes=%lld", (long long)n);
    for (int l = 0; l < n_levels; ++l)
      if (level_counts[l] < 2 || (l > 0 && level_counts[l] <= level_counts[l - 1]))
        return set_error(XMGN_EINVAL, "xmgn_build_graph: level_counts[%d]=%lld not increasing (>= 2)", l,
                         (long long)level_counts[l]);
    if (k < 1 || k > K_MAX) return set_error(XMGN_EUNSUPPORTED, "xmgn_build_graph: k=%d (1..%d)", k, K_MAX);
    if (n_parts < 1 || n_parts > n) return set_error(XMGN_EINVAL, "xmgn_build_graph: n_parts=%d", n_parts);
    if (halo_depth < 0 || halo_depth > 63) return set_error(XMGN_EINVAL, "xmgn_build_graph: halo_depth=%d", halo_depth);
    XMGN_CUDA(cudaSetDevice(cuda_device), "xmgn_build_graph: cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    Temp tmp;
    size_t tb = 0;
    const int N = (int)n;
    // ---- bounding box of all points
    DBuf<float> bpart(blocks_for(n) * 6);
    k_bbox<<<blocks_for(n), 256, 0, st>>>(pos, nullptr, N, bpart.p);
    std::vector<float> hb(bpart.n);
    XMGN_CUDA(cudaMemcpyAsync(hb.data(), bpart.p, hb.size() * 4, cudaMemcpyDeviceToHost, st), "bbox");
    XMGN_CUDA(cudaStreamSynchronize(st), "bbox");
    float lo[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, hi[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
    for (size_t b = 0; b < hb.size() / 6; ++b)
      for (int c = 0; c < 3; ++c) { lo[c] = std::min(lo[c], hb[6 * b + c]); hi[c] = std::max(hi[c], hb[6 * b + 3 + c]); }
    double ext[3], emax = 0, amax = 0;
    for (int c = 0; c < 3; ++c) {
      ext[c] = (double)hi[c] - (double)lo[c];
      emax = std::max(emax, ext[c]);
      amax = std::max({amax, std::fabs((double)lo[c]), std::fabs((double)hi[c])});
    }
    if (emax <= 0) return set_error(XMGN_EINVAL, "xmgn_build_graph: all points coincide");
    // ---- per level: exact kNN, then both edge directions as (dst, src) keys
    std::vector<int64_t> kk(n_levels);
    int64_t nkeys = 0;
    for (int l = 0; l < n_levels; ++l) {
      kk[l] = std::min<int64_t>(k, level_counts[l] - 1);
      nkeys += 2 * level_counts[l] * kk[l];
    }
    DBuf<uint64_t> ekeys(nkeys);
    int64_t kbase = 0;
    {
      DBuf<uint64_t> ck(n), cks(n), cells(n), ucell(n);
      DBuf<int> order(n), ustart(n + 1), nu_d(1), nb(n * k);
      DBuf<float> spos(3 * n);
      for (int l = 0; l < n_levels; ++l) {
        const int c = (int)level_counts[l], kl = (int)kk[l];
        Grid g;
        double vol = 1;
        for (int d = 0; d < 3; ++d) vol *= std::max(ext[d], 1e-6 * emax);
        g.h = std::cbrt(vol / c);
        for (int d = 0; d < 3; ++d) {
          g.lo[d] = lo[d];
          g.nc[d] = (int)std::min(1.0 + std::floor(ext[d] / g.h), 1048576.0);
        }
        g.inv_h = (float)(1.0 / g.h);
        const double slack = 1e-5 * g.h + 1e-6 * (amax + g.h);
        const int rmax = std::max({g.nc[0], g.nc[1], g.nc[2]});
        k_cell_keys<<<blocks_for(c), 256, 0, st>>>(pos, c, g, ck.p);
        cub::DeviceRadixSort::SortKeys(nullptr, tb, ck.p, cks.p, c, 0, 64, st);
        cub::DeviceRadixSort::SortKeys(tmp.get(tb), tb, ck.p, cks.p, c, 0, 64, st);
        k_split_keys<<<blocks_for(c), 256, 0, st>>>(cks.p, pos, c, order.p, spos.p, cells.p);
        // unique cells and their first slots
        DBuf<int> counts(c);
        cub::DeviceRunLengthEncode::Encode(nullptr, tb, cells.p, ucell.p, counts.p, nu_d.p, c, st);
        cub::DeviceRunLengthEncode::Encode(tmp.get(tb), tb, cells.p, ucell.p, counts.p, nu_d.p, c, st);
        int nu = 0;
        XMGN_CUDA(cudaMemcpyAsync(&nu, nu_d.p, 4, cudaMemcpyDeviceToHost, st), "cells");
        XMGN_CUDA(cudaStreamSynchronize(st), "cells");
        XMGN_CUDA(cudaMemsetAsync(ustart.p, 0, 4, st), "cells");
        cub::DeviceScan::InclusiveSum(nullptr, tb, counts.p, ustart.p + 1, nu, st);
        cub::DeviceScan::InclusiveSum(tmp.get(tb), tb, counts.p, ustart.p + 1, nu, st);
        k_knn<<<(c + 127) / 128, 128, 0, st>>>(spos.p, order.p, ucell.p, ustart.p, nu, c, kl, g, slack, rmax, nb.p);
        k_edge_keys<<<blocks_for((long long)c * kl), 256, 0, st>>>(nb.p, c, kl, (uint64_t)n, ekeys.p + kbase);
        kbase += 2LL * c * kl;
        XMGN_CUDA(cudaGetLastError(), "xmgn_build_graph: kNN");
      }
    }
    // ---- symmetrised union -> CSR by destination
    int end_bit = 1;
    while (end_bit < 64 && ((uint64_t)1 << end_bit) < (uint64_t)n * (uint64_t)n) ++end_bit;
    DBuf<uint64_t> sk(nkeys);
    cub::DeviceRadixSort::SortKeys(nullptr, tb, ekeys.p, sk.p, nkeys, 0, end_bit, st);
    cub::DeviceRadixSort::SortKeys(tmp.get(tb), tb, ekeys.p, sk.p, nkeys, 0, end_bit, st);
    DBuf<long long> ne_d(1);
    cub::DeviceSelect::Unique(nullptr, tb, sk.p, ekeys.p, ne_d.p, nkeys, st);
    cub::DeviceSelect::Unique(tmp.get(tb), tb, sk.p, ekeys.p, ne_d.p, nkeys, st);
    long long E = 0;
    XMGN_CUDA(cudaMemcpyAsync(&E, ne_d.p, 8, cudaMemcpyDeviceToHost, st), "unique");
    XMGN_CUDA(cudaStreamSynchronize(st), "unique");
    sk.free();
    DBuf<int64_t> doff(n + 1), dsrc(std::max<long long>(E, 1));
    k_csr<<<blocks_for(std::max<long long>(E, n + 1)), 256, 0, st>>>(ekeys.p, E, (uint64_t)n, doff.p, dsrc.p);
    ekeys.free();
    // ---- recursive coordinate bisection
    DBuf<int64_t> owner(n);
    {
      DBuf<int> perm(n);
      DBuf<uint64_t> rk(n), rks(n);
      k_iota<<<blocks_for(n), 256, 0, st>>>(perm.p, N);
      struct Seg { int start, len, p0, np; };
      std::vector<Seg> segs{{0, N, 0, n_parts}}, leaves;
      std::vector<float> hbb;
      while (!segs.empty()) {
        std::vector<Seg> next;
        for (const Seg& s : segs) {
          if (s.np == 1) { leaves.push_back(s); continue; }
          const int nbk = blocks_for(s.len);
          k_bbox<<<nbk, 256, 0, st>>>(pos, perm.p + s.start, s.len, bpart.p);
          hbb.resize(nbk * 6);
          XMGN_CUDA(cudaMemcpyAsync(hbb.data(), bpart.p, hbb.size() * 4, cudaMemcpyDeviceToHost, st), "rcb");
          XMGN_CUDA(cudaStreamSynchronize(st), "rcb");
          float mn[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, mx[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
          for (int b = 0; b < nbk; ++b)
            for (int c = 0; c < 3; ++c) { mn[c] = std::min(mn[c], hbb[6 * b + c]); mx[c] = std::max(mx[c], hbb[6 * b + 3 + c]); }
          int ax = 0;
          double best = -1;
          for (int c = 0; c < 3; ++c) {
            const double e = (double)mx[c] - (double)mn[c];
            if (e > best) { best = e; ax = c; }
          }
          k_rcb_keys<<<blocks_for(s.len), 256, 0, st>>>(pos, perm.p + s.start, s.len, ax, rk.p);
          cub::DeviceRadixSort::SortKeys(nullptr, tb, rk.p, rks.p, s.len, 0, 64, st);
          cub::DeviceRadixSort::SortKeys(tmp.get(tb), tb, rk.p, rks.p, s.len, 0, 64, st);
          k_rcb_unkey<<<blocks_for(s.len), 256, 0, st>>>(rks.p, s.len, perm.p + s.start);
          const int pl = s.np / 2;
          const int nl = (int)std::nearbyint((double)((int64_t)s.len * pl) / (double)s.np);
          next.push_back({s.start, nl, s.p0, pl});
          next.push_back({s.start + nl, s.len - nl, s.p0 + pl, s.np - pl});
        }
        segs.swap(next);
      }
      for (const Seg& s : leaves)
        if (s.len > 0) k_set_owner<<<blocks_for(s.len), 256, 0, st>>>(perm.p + s.start, s.len, s.p0, owner.p);
      XMGN_CUDA(cudaGetLastError(), "xmgn_build_graph: RCB");
    }
    // ---- halo rings and the (ring, id)-ordered lists
    auto* b = new xmgn_built_graph();
    try {
      b->n = n; b->E = E; b->P = n_parts; b->depth = halo_depth;
      b->owned_offsets.assign(n_parts + 1, 0);
      b->halo_offsets.assign(n_parts + 1, 0);
      b->owned.resize(n);
      {
        DBuf<int> ring(n), sel(n), nsel(1);
        DBuf<int64_t> sel64(n);
        thrust::counting_iterator<int> ids(0);
        for (int p = 0; p < n_parts; ++p) {
          int cnt = 0;
          cub::DeviceSelect::If(nullptr, tb, ids, sel.p, nsel.p, N, OwnedBy{owner.p, p}, st);
          cub::DeviceSelect::If(tmp.get(tb), tb, ids, sel.p, nsel.p, N, OwnedBy{owner.p, p}, st);
          XMGN_CUDA(cudaMemcpyAsync(&cnt, nsel.p, 4, cudaMemcpyDeviceToHost, st), "owned");
          XMGN_CUDA(cudaStreamSynchronize(st), "owned");
          k_i32_to_i64<<<blocks_for(cnt), 256, 0, st>>>(sel.p, cnt, sel64.p);
          XMGN_CUDA(cudaMemcpyAsync(b->owned.data() + b->owned_offsets[p], sel64.p, (size_t)cnt * 8,
                                    cudaMemcpyDeviceToHost, st), "owned");
          b->owned_offsets[p + 1] = b->owned_offsets[p] + cnt;
          k_ring_init<<<blocks_for(n), 256, 0, st>>>(owner.p, N, p, ring.p);
          for (int r = 1; r <= halo_depth; ++r) k_ring_step<<<blocks_for(n), 256, 0, st>>>(doff.p, dsrc.p, N, r, ring.p);
          int64_t hcount = 0;
          for (int r = 1; r <= halo_depth; ++r) {
            cub::DeviceSelect::If(nullptr, tb, ids, sel.p, nsel.p, N, InRing{ring.p, r}, st);
            cub::DeviceSelect::If(tmp.get(tb), tb, ids, sel.p, nsel.p, N, InRing{ring.p, r}, st);
            XMGN_CUDA(cudaMemcpyAsync(&cnt, nsel.p, 4, cudaMemcpyDeviceToHost, st), "halo");
            XMGN_CUDA(cudaStreamSynchronize(st), "halo");
            if (cnt == 0) break;
            k_i32_to_i64<<<blocks_for(cnt), 256, 0, st>>>(sel.p, cnt, sel64.p);
            const size_t o = b->halo.size();
            b->halo.resize(o + cnt);
            b->halo_ring.resize(o + cnt, r);
            XMGN_CUDA(cudaMemcpyAsync(b->halo.data() + o, sel64.p, (size_t)cnt * 8, cudaMemcpyDeviceToHost, st), "halo");
            XMGN_CUDA(cudaStreamSynchronize(st), "halo");
            hcount += cnt;
          }
          b->halo_offsets[p + 1] = b->halo_offsets[p] + hcount;
        }
      }
      b->offsets.resize(n + 1);
      b->sources.resize(E);
      b->owner.resize(n);
      XMGN_CUDA(cudaMemcpyAsync(b->offsets.data(), doff.p, (n + 1) * 8, cudaMemcpyDeviceToHost, st), "download");
      if (E) XMGN_CUDA(cudaMemcpyAsync(b->sources.data(), dsrc.p, E * 8, cudaMemcpyDeviceToHost, st), "download");
      XMGN_CUDA(cudaMemcpyAsync(b->owner.data(), owner.p, n * 8, cudaMemcpyDeviceToHost, st), "download");
      XMGN_CUDA(cudaStreamSynchronize(st), "download");
    } catch (...) {
      delete b;
      throw;
    }
    *out = b;
    return XMGN_OK;
  });
}

extern "C" xmgn_status xmgn_built_graph_desc(const xmgn_built_graph* b, xmgn_graph_desc* d) {
  if (!b || !d) return set_error(XMGN_EINVAL, "xmgn_built_graph_desc: null argument");
  std::memset(d, 0, sizeof(*d));
  d->n_nodes = b->n;
  d->n_edges = b->E;
  d->csr_offsets = b->offsets.data();
  d->csr_sources = b->sources.data();
  d->n_parts = b->P;
  d->halo_depth = b->depth;
  d->owned_offsets = b->owned_offsets.data();
  d->owned = b->owned.data();
  d->halo_offsets = b->halo_offsets.data();
  d->halo = b->halo.data();
  d->halo_ring = b->halo_ring.data();
  return XMGN_OK;
}

extern "C" xmgn_status xmgn_built_graph_owner(const xmgn_built_graph* b, int64_t* owner) {
  if (!b || !owner) return set_error(XMGN_EINVAL, "xmgn_built_graph_owner: null argument");
  std::memcpy(owner, b->owner.data(), b->owner.size() * 8);
  return XMGN_OK;
}

extern "C" void xmgn_built_graph_free(xmgn_built_graph* b) { delete b; }
