// TEST INFRASTRUCTURE ONLY -- never linked, loaded or called by the product
// path (paper_2411_17164_b200/).  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may use it.
//
// Plain, slow, FP64 CPU reference of the X-MeshGraphNet processor stack
// (arXiv 2411.17164) over a graph in CSR-by-destination form, plus its own
// halo-partition builder.  Every function cites the passage it restates.
// Readings of the paper are those of SURVEY.md §8(c) (listed in DESIGN.md).
//
//   MLP(x)  = z_{m+1},  z_1 = x W_1 + b_1,  z_{j+1} = SiLU(z_j) W_{j+1} + b_{j+1}
//   SiLU(t) = t / (1 + exp(-t))
//   LN(z)   = gamma * (z - mu) * (var + eps)^-1/2 + beta, biased var over H
//   edge    e^l_k = e^{l-1}_k + LN_e(MLP_e([e^{l-1}_k | h^{l-1}_src | h^{l-1}_dst]))
//                                        (Eq.1, read per NS)
//   agg     a^l_i = sum_{k: dst k = i} e^l_k  in CSR order   (Eq.2)
//   node    h^l_i = h^{l-1}_i + LN_n(MLP_n([h^{l-1}_i | a^l_i]))
//                                        (Eq.3, 155 Eq.4)
//   loss    L = sum_{i in O} <g_i, h^L_i>  (halo rows dropped)
//
// Backward is the hand-written adjoint of the above.  No BLAS:
// every row is produced by the same instruction sequence wherever it sits, and
// every reduction runs in a fixed order independent of the thread count, so
// results are bitwise reproducible.  Built with -ffp-contract=off.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#include <algorithm>
#include <omp.h>

namespace {

// ---- flat parameter layout: per layer, edge block then node
// block; W stored [in, out]; y = x W + b.
struct Block {
  int kin;                 // 3H (edge) or 2H (node)
  int64_t W[8], b[8];      // offsets of W_j, b_j (j = 0..m)
  int64_t gamma, beta;
};

int64_t block_size(int kin, int H, int m) {
  return (int64_t)kin * H + H + (int64_t)m * ((int64_t)H * H + H) + 2 * (int64_t)H;
}

Block make_block(int64_t base, int kin, int H, int m) {
  Block B;
  B.kin = kin;
  int64_t o = base;
  for (int j = 0; j <= m; ++j) {
    int kj = j == 0 ? kin : H;
    B.W[j] = o; o += (int64_t)kj * H;
    B.b[j] = o; o += H;
  }
  B.gamma = o; o += H;
  B.beta = o; o += H;
  return B;
}

Block edge_block(int l, int H, int m) {
  int64_t per = block_size(3 * H, H, m) + block_size(2 * H, H, m);
  return make_block((int64_t)l * per, 3 * H, H, m);
}
Block node_block(int l, int H, int m) {
  int64_t per = block_size(3 * H, H, m) + block_size(2 * H, H, m);
  return make_block((int64_t)l * per + block_size(3 * H, H, m), 2 * H, H, m);
}

inline double silu(double t) { return t / (1.0 + std::exp(-t)); }
inline double dsilu(double t) {  // sigma(t) (1 + t (1 - sigma(t)))
  double s = 1.0 / (1.0 + std::exp(-t));
  return s * (1.0 + t * (1.0 - s));
}

// y = x W + b for one row; W [kin, H] row-major.
void linear_row(const double* x, int kin, const double* W, const double* b, int H, double* y) {
  for (int o = 0; o < H; ++o) y[o] = 0.0;
  for (int i = 0; i < kin; ++i) {
    double xi = x[i];
    const double* w = W + (int64_t)i * H;
    for (int o = 0; o < H; ++o) y[o] += xi * w[o];
  }
  for (int o = 0; o < H; ++o) y[o] += b[o];
}

// Forward of one block over R rows: Y = LN(MLP(X)).  Optionally keeps the
// pre-activations Z[j][r][:] and LN statistics for the backward.
void block_forward(const Block& B, const double* P, int H, int m, double eps, int64_t R,
                   const double* X, double* Y, double* Z /*[(m+1)][R][H] or null*/,
                   double* mu /*[R] or null*/, double* rs /*[R] or null*/) {
#pragma omp parallel
  {
    std::vector<double> z((size_t)(m + 1) * H), a(H);
#pragma omp for schedule(static)
    for (int64_t r = 0; r < R; ++r) {
      const double* x = X + r * B.kin;
      linear_row(x, B.kin, P + B.W[0], P + B.b[0], H, &z[0]);
      for (int j = 1; j <= m; ++j) {
        for (int c = 0; c < H; ++c) a[c] = silu(z[(size_t)(j - 1) * H + c]);
        linear_row(&a[0], H, P + B.W[j], P + B.b[j], H, &z[(size_t)j * H]);
      }
      const double* zl = &z[(size_t)m * H];
      double s = 0.0;
      for (int c = 0; c < H; ++c) s += zl[c];
      double mean = s / H;
      double v = 0.0;
      for (int c = 0; c < H; ++c) { double d = zl[c] - mean; v += d * d; }
      v /= H;
      double r_ = 1.0 / std::sqrt(v + eps);
      for (int c = 0; c < H; ++c)
        Y[r * H + c] = P[B.gamma + c] * ((zl[c] - mean) * r_) + P[B.beta + c];
      if (Z)
        for (int j = 0; j <= m; ++j)
          std::memcpy(Z + ((size_t)j * R + r) * H, &z[(size_t)j * H], sizeof(double) * H);
      if (mu) mu[r] = mean;
      if (rs) rs[r] = r_;
    }
  }
}

// dW[i][o] += sum_r A[r][i] dZ[r][o]  (rows in ascending order, per output element)
void wgrad(const double* A, int64_t lda, const double* dZ, int64_t R, int kin, int H, double* dW) {
#pragma omp parallel for schedule(static)
  for (int i = 0; i < kin; ++i) {
    double* w = dW + (int64_t)i * H;
    for (int64_t r = 0; r < R; ++r) {
      double a = A[r * lda + i];
      const double* d = dZ + r * H;
      for (int o = 0; o < H; ++o) w[o] += a * d[o];
    }
  }
}

void colsum(const double* D, int64_t R, int H, double* out) {
#pragma omp parallel for schedule(static)
  for (int o = 0; o < H; ++o) {
    double s = out[o];
    for (int64_t r = 0; r < R; ++r) s += D[r * H + o];
    out[o] = s;
  }
}

// Backward of one block.  dY [R][H] upstream; writes dX [R][kin]; accumulates
// parameter gradients into G (same layout as P).
void block_backward(const Block& B, const double* P, int H, int m, double eps, int64_t R,
                    const double* X, const double* dY, double* dX, double* G) {
  std::vector<double> Z((size_t)(m + 1) * R * H), mu(R), rs(R), Y((size_t)R * H);
  block_forward(B, P, H, m, eps, R, X, &Y[0], &Z[0], &mu[0], &rs[0]);
  std::vector<double> dZ((size_t)(m + 1) * R * H), Xh((size_t)R * H);
  const double* gamma = P + B.gamma;
  // LayerNorm backward (x^ = (z - mu) r):
  //   dgamma = sum dY x^, dbeta = sum dY, dx^ = dY gamma,
  //   dz = r (dx^ - mean(dx^) - x^ mean(dx^ x^))
#pragma omp parallel
  {
    std::vector<double> dxh(H);
#pragma omp for schedule(static)
    for (int64_t r = 0; r < R; ++r) {
      const double* z = &Z[((size_t)m * R + r) * H];
      double* xh = &Xh[(size_t)r * H];
      double s1 = 0.0, s2 = 0.0;
      for (int c = 0; c < H; ++c) {
        xh[c] = (z[c] - mu[r]) * rs[r];
        dxh[c] = dY[r * H + c] * gamma[c];
        s1 += dxh[c];
        s2 += dxh[c] * xh[c];
      }
      s1 /= H;
      s2 /= H;
      double* dz = &dZ[((size_t)m * R + r) * H];
      for (int c = 0; c < H; ++c) dz[c] = rs[r] * (dxh[c] - s1 - xh[c] * s2);
    }
  }
  {  // dgamma, dbeta
    double* gg = G + B.gamma;
    double* gb = G + B.beta;
#pragma omp parallel for schedule(static)
    for (int c = 0; c < H; ++c) {
      double a = gg[c], b = gb[c];
      for (int64_t r = 0; r < R; ++r) { a += dY[r * H + c] * Xh[(size_t)r * H + c]; b += dY[r * H + c]; }
      gg[c] = a;
      gb[c] = b;
    }
  }
  std::vector<double> Aj((size_t)R * H);
  for (int j = m; j >= 1; --j) {
    // A_{j-1} = SiLU(Z_{j-1}); dW_j = A^T dZ_j; db_j = sum dZ_j;
    // dZ_{j-1} = (dZ_j W_j^T) * SiLU'(Z_{j-1})
    const double* Zp = &Z[(size_t)(j - 1) * R * H];
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < R * H; ++t) Aj[t] = silu(Zp[t]);
    const double* dZj = &dZ[(size_t)j * R * H];
    wgrad(&Aj[0], H, dZj, R, H, H, G + B.W[j]);
    colsum(dZj, R, H, G + B.b[j]);
    const double* W = P + B.W[j];
    double* dZp = &dZ[(size_t)(j - 1) * R * H];
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < R; ++r) {
      for (int i = 0; i < H; ++i) {
        double s = 0.0;
        const double* w = W + (int64_t)i * H;
        const double* d = dZj + r * H;
        for (int o = 0; o < H; ++o) s += d[o] * w[o];
        dZp[r * H + i] = s * dsilu(Zp[r * H + i]);
      }
    }
  }
  const double* dZ1 = &dZ[0];
  wgrad(X, B.kin, dZ1, R, B.kin, H, G + B.W[0]);
  colsum(dZ1, R, H, G + B.b[0]);
  const double* W1 = P + B.W[0];
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < R; ++r) {
    for (int i = 0; i < B.kin; ++i) {
      double s = 0.0;
      const double* w = W1 + (int64_t)i * H;
      const double* d = dZ1 + r * H;
      for (int o = 0; o < H; ++o) s += d[o] * w[o];
      dX[r * B.kin + i] = s;
    }
  }
}

void edge_inputs(int64_t E, int H, const int64_t* src, const int64_t* dst, const double* e,
                 const double* h, double* X) {
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < E; ++k) {
    double* x = X + k * 3 * H;
    std::memcpy(x, e + k * H, sizeof(double) * H);
    std::memcpy(x + H, h + src[k] * H, sizeof(double) * H);
    std::memcpy(x + 2 * H, h + dst[k] * H, sizeof(double) * H);
  }
}

void node_inputs(int64_t N, int H, const double* h, const double* a, double* X) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i) {
    std::memcpy(X + i * 2 * H, h + i * H, sizeof(double) * H);
    std::memcpy(X + i * 2 * H + H, a + i * H, sizeof(double) * H);
  }
}

std::vector<int64_t> dst_of(int64_t N, const int64_t* off) {
  std::vector<int64_t> d(off[N]);
  for (int64_t i = 0; i < N; ++i)
    for (int64_t k = off[i]; k < off[i + 1]; ++k) d[k] = i;
  return d;
}

}  // namespace

extern "C" {

int64_t oracle_param_count(int H, int L, int m) {
  return (int64_t)L * (block_size(3 * H, H, m) + block_size(2 * H, H, m));
}

// Full forward (Eq. 4 read per SURVEY §8(c)).
// h_all [(L+1)][N][H], e_all [(L+1)][E][H], a_all [L][N][H]; level 0 of h_all
// and e_all must hold h^0 and e^0 on entry.
int oracle_forward(int64_t N, const int64_t* off, const int64_t* src, int H, int L, int m,
                   double eps, const double* P, double* h_all, double* e_all, double* a_all) {
  const int64_t E = off[N];
  std::vector<int64_t> dst = dst_of(N, off);
  std::vector<double> X((size_t)E * 3 * H), Y((size_t)std::max(E, N) * H);
  for (int l = 1; l <= L; ++l) {
    const double* hp = h_all + (size_t)(l - 1) * N * H;
    const double* ep = e_all + (size_t)(l - 1) * E * H;
    double* hn = h_all + (size_t)l * N * H;
    double* en = e_all + (size_t)l * E * H;
    double* a = a_all + (size_t)(l - 1) * N * H;
    // edge update: e^l = e^{l-1} + LN(MLP([e | h_src | h_dst]))
    edge_inputs(E, H, src, &dst[0], ep, hp, &X[0]);
    block_forward(edge_block(l - 1, H, m), P, H, m, eps, E, &X[0], &Y[0], nullptr, nullptr, nullptr);
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < E * H; ++t) en[t] = ep[t] + Y[t];
    // aggregation: a_i = sum over in-edges in CSR order (Eq. 2)
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; ++i)
      for (int c = 0; c < H; ++c) {
        double s = 0.0;
        for (int64_t k = off[i]; k < off[i + 1]; ++k) s += en[k * H + c];
        a[i * H + c] = s;
      }
    // node update: h^l = h^{l-1} + LN(MLP([h | a]))  (Eq. 3)
    node_inputs(N, H, hp, a, &X[0]);
    block_forward(node_block(l - 1, H, m), P, H, m, eps, N, &X[0], &Y[0], nullptr, nullptr, nullptr);
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < N * H; ++t) hn[t] = hp[t] + Y[t];
  }
  return 0;
}

// Backward of L = sum_i <g_i, h^L_i> (g zero on rows outside the loss set,
// PAPER.md:197).  G (param grads) is overwritten; grad_h0 [N][H], grad_e0 [E][H].
int oracle_backward(int64_t N, const int64_t* off, const int64_t* src, int H, int L, int m,
                    double eps, const double* P, const double* h_all, const double* e_all,
                    const double* a_all, const double* g, double* G, double* grad_h0,
                    double* grad_e0) {
  const int64_t E = off[N];
  std::vector<int64_t> dst = dst_of(N, off);
  std::memset(G, 0, sizeof(double) * oracle_param_count(H, L, m));
  // out-edge lists (edges grouped by source, ascending edge id)
  std::vector<int64_t> ooff(N + 1, 0), oedge(E);
  for (int64_t k = 0; k < E; ++k) ooff[src[k] + 1]++;
  for (int64_t i = 0; i < N; ++i) ooff[i + 1] += ooff[i];
  {
    std::vector<int64_t> fill(ooff.begin(), ooff.end() - 1);
    for (int64_t k = 0; k < E; ++k) oedge[fill[src[k]]++] = k;
  }
  std::vector<double> Gh(g, g + (size_t)N * H), Ge((size_t)E * H, 0.0);
  std::vector<double> X((size_t)std::max(3 * E, 2 * N) * H), dX((size_t)std::max(3 * E, 2 * N) * H);
  std::vector<double> Ga((size_t)N * H), Gn((size_t)N * H), Gep((size_t)E * H);
  for (int l = L; l >= 1; --l) {
    const double* hp = h_all + (size_t)(l - 1) * N * H;
    const double* ep = e_all + (size_t)(l - 1) * E * H;
    const double* a = a_all + (size_t)(l - 1) * N * H;
    // node block: dX = [dh | da]
    node_inputs(N, H, hp, a, &X[0]);
    block_backward(node_block(l - 1, H, m), P, H, m, eps, N, &X[0], &Gh[0], &dX[0], G);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; ++i)
      for (int c = 0; c < H; ++c) {
        Gn[i * H + c] = Gh[i * H + c] + dX[i * 2 * H + c];
        Ga[i * H + c] = dX[i * 2 * H + H + c];
      }
    // G_e' = G_e + da[dst]  (the aggregation's adjoint)
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < E; ++k)
      for (int c = 0; c < H; ++c) Gep[k * H + c] = Ge[k * H + c] + Ga[dst[k] * H + c];
    // edge block: dX = [de | dh_src | dh_dst]
    edge_inputs(E, H, src, &dst[0], ep, hp, &X[0]);
    block_backward(edge_block(l - 1, H, m), P, H, m, eps, E, &X[0], &Gep[0], &dX[0], G);
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < E; ++k)
      for (int c = 0; c < H; ++c) Ge[k * H + c] = Gep[k * H + c] + dX[k * 3 * H + c];
    // scatter dh_dst over in-edges (CSR order) and dh_src over out-edges (edge order)
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; ++i)
      for (int c = 0; c < H; ++c) {
        double s = Gn[i * H + c];
        for (int64_t k = off[i]; k < off[i + 1]; ++k) s += dX[k * 3 * H + 2 * H + c];
        for (int64_t t = ooff[i]; t < ooff[i + 1]; ++t) s += dX[oedge[t] * 3 * H + H + c];
        Gh[i * H + c] = s;
      }
  }
  std::memcpy(grad_h0, &Gh[0], sizeof(double) * N * H);
  std::memcpy(grad_e0, &Ge[0], sizeof(double) * E * H);
  return 0;
}

// Halo partition of one owned set:
// V_p = owned ∪ {v : undirected hop distance(v, owned) <= depth}; local order
// ring-major, ascending global id inside a ring; local in-edges keep the
// global CSR order and exist iff both endpoints are local; rev[k] is the local
// index of the reverse edge (-1 if absent).  Buffers sized N+1 / E by the caller.
int oracle_local_graph(int64_t N, const int64_t* off, const int64_t* src, int64_t n_owned,
                       const int64_t* owned, int depth, int64_t* n_local_out, int64_t* e_local_out,
                       int64_t* local_gid, int32_t* local_ring, int64_t* loff, int64_t* lsrc,
                       int64_t* legid, int64_t* rev) {
  const int64_t E = off[N];
  std::vector<int64_t> ooff(N + 1, 0), odst(E);
  for (int64_t k = 0; k < E; ++k) ooff[src[k] + 1]++;
  for (int64_t i = 0; i < N; ++i) ooff[i + 1] += ooff[i];
  {
    std::vector<int64_t> fill(ooff.begin(), ooff.end() - 1);
    for (int64_t i = 0; i < N; ++i)
      for (int64_t k = off[i]; k < off[i + 1]; ++k) odst[fill[src[k]]++] = i;
  }
  std::vector<int32_t> dist(N, -1);
  std::vector<int64_t> frontier(owned, owned + n_owned), next;
  for (int64_t t = 0; t < n_owned; ++t) dist[owned[t]] = 0;
  for (int r = 1; r <= depth; ++r) {
    next.clear();
    for (int64_t v : frontier) {
      for (int64_t k = off[v]; k < off[v + 1]; ++k)
        if (dist[src[k]] < 0) { dist[src[k]] = r; next.push_back(src[k]); }
      for (int64_t t = ooff[v]; t < ooff[v + 1]; ++t)
        if (dist[odst[t]] < 0) { dist[odst[t]] = r; next.push_back(odst[t]); }
    }
    frontier.swap(next);
  }
  std::vector<int64_t> order;
  for (int64_t v = 0; v < N; ++v)
    if (dist[v] >= 0) order.push_back(v);
  std::stable_sort(order.begin(), order.end(),
                   [&](int64_t a, int64_t b) { return dist[a] < dist[b]; });
  const int64_t nl = (int64_t)order.size();
  std::vector<int64_t> lid(N, -1);
  for (int64_t t = 0; t < nl; ++t) { lid[order[t]] = t; local_gid[t] = order[t]; local_ring[t] = dist[order[t]]; }
  int64_t el = 0;
  loff[0] = 0;
  for (int64_t t = 0; t < nl; ++t) {
    int64_t v = order[t];
    for (int64_t k = off[v]; k < off[v + 1]; ++k)
      if (lid[src[k]] >= 0) { lsrc[el] = lid[src[k]]; legid[el] = k; ++el; }
    loff[t + 1] = el;
  }
  for (int64_t t = 0; t < nl; ++t)
    for (int64_t k = loff[t]; k < loff[t + 1]; ++k) {
      int64_t j = lsrc[k];
      rev[k] = -1;
      for (int64_t q = loff[j]; q < loff[j + 1]; ++q)
        if (lsrc[q] == t) { rev[k] = q; break; }
    }
  *n_local_out = nl;
  *e_local_out = el;
  return 0;
}

}  // extern "C"
