// Workspace, forward and backward of the processor on one GPU (call
// stacks 3-4).  Host code only sequences launches; every arithmetic step runs in
// the kernels of chain.cuh / kernels.cu.
//
// Algorithmic restatement used here (identical function to include/xmgn.h):
//   [e | h_src | h_dst] W1e = e W1e_e + (h W1e_s)[src] + (h W1e_d)[dst],
// so each layer first projects the nodes, P = h [W1e_s | W1e_d] (N x 2H, FP32),
// and the edge MLP's first GEMM has K = H instead of 3H.
// The backward mirrors it: d(P_src)[i] / d(P_dst)[i] are segment sums of dZ1
// over out-/in-edges (rev permutation; no atomics), then one node-level GEMM.
//
// Halo shrinking: with ring-major numbering layer l only
// updates destinations of ring <= L-l, a prefix of nodes (n_l) and of edges
// (E_l); the skipped rows feed only discarded halo outputs.
#include <cuda_runtime.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "graph.h"
#include "kernels_launch.h"
#include "tmap.h"

namespace xmgn {

typedef __nv_bfloat16 bf16;

struct DPart {
  int *off = nullptr, *src = nullptr, *dst = nullptr, *rev = nullptr;
};

struct BfBuf {       // BF16 tensor with an optional lo half (FP32 check mode)
  bf16* p = nullptr;
  long long lo = 0;  // element offset of the lo half (0 when not split)
};

}  // namespace xmgn

struct xmgn_workspace {
  const xmgn_graph* g = nullptr;
  xmgn_model_cfg cfg{};
  int dev = 0, H = 0, L = 0, m = 0, sms = 148;
  bool split = false, f16 = false;
  int64_t Nmax = 0, Emax = 0, Rmax = 0;
  std::vector<xmgn::DPart> dparts;
  std::vector<void*> allocs;
  size_t bytes = 0;
  // packed weights
  int S1 = 0, S2 = 0;
  xmgn::BfBuf wk1, wk2;
  xmgn::PackJob* d_jobs = nullptr;
  int njobs = 0;
  // checkpoints (per layer) and live streams
  xmgn::BfBuf e_ck, h_ck, a_ck;   // e_ck [L+1][Emax][H] (the 16-bit edge stream), h_ck / a_ck [L][Nmax][H]
  xmgn::BfBuf z1_ck;              // [L][Emax][H] 16-bit z_1 of the edge MLP (16-bit modes, if HBM allows)
  bool use_z1 = false;
  float *h_buf[2] = {nullptr, nullptr};
  float *e32[2] = {nullptr, nullptr};  // BF16 mode: the edge residual stream in FP32 (ping-pong)
  bool e32_mode = false;
  // BF16 mode: the node MLP's first GEMM and the pre-projection P take 2 x BF16 operands
  // (hi + lo, forward only); P is stored FP16 in every 16-bit mode
  bool bsplit = false;
  xmgn::BfBuf wkx;                // [L][3][H][4H]: [W0h^T W0a^T W0h^T W0a^T]; [W0s^T W0s^T]; [W0d^T W0d^T]
  xmgn::bf16* hlo[2] = {nullptr, nullptr};  // lo halves of h^l (ping-pong by l)
  xmgn::bf16* alo = nullptr;      // lo half of a^l
  // per-row LayerNorm (mean, rstd) of every layer's edge / node update, written by the forward
  // and read by the backward instead of a statistics pass (16-bit training modes;
  // XMGN_LN_STATS=0: off)
  float2* lnst_e = nullptr;       // [L][Emax]
  float2* lnst_n = nullptr;       // [L][Nmax]
  xmgn::BfBuf P;                  // node pre-projections, one per layer [L][Nmax][2H], 16-bit (kept for the bwd)
  // backward
  float* Gh = nullptr;            // dL/dh (FP32, node level)
  xmgn::BfBuf Ge[2], Ga;          // dL/de (16-bit edge stream, ping-pong), dL/da (16-bit)
  xmgn::BfBuf scrA[2], scrS[2], scrZ[3], D;
  float* part = nullptr;  // wgrad split-K partials
  int part_splits = 0;
  float* colsum = nullptr;        // per-tile column-sum partials (chain.cuh), colsum_cap floats
  size_t colsum_cap = 0;
  float* cs_tmp = nullptr;        // [NV_MAX][CS_SEG][H] first-level sums of the colsum reduce
  int cs_slot[xmgn::NV_MAX];      // slot map of the last backward chain launch
  int cs_nct = 0;                 // its CTA tiles
  unsigned int* d_amax = nullptr;  // max|g| bits of the current backward's seed
  float* d_scale = nullptr;        // {S, 1/S}: the backward's power-of-two loss scale
  int last_fwd = -1;
  int gc_last = 0;      // which G_e buffer holds dL/de^0 after the last backward
  // ---- the model around the processor (NEXT-1), allocated at the first xmgn_model_fwd
  bool io_ready = false;
  int64_t Omax = 0;               // largest owned set
  int S3 = 0;                     // H x H slots of wioH
  xmgn::BfBuf wio64, wioH;        // encoder W1^T [2][H][64] (zero-padded K); [S3][H][H] (W^T fwd, W dgrad)
  xmgn::PackJob* d_jobs_io = nullptr;
  int njobs_io = 0;
  xmgn::BfBuf Xn, Xe;             // 16-bit z-scored inputs [Nmax][64], [Emax][64]
  xmgn::BfBuf hL16;               // 16-bit h^L of the owned rows [Omax][H] (the decoder's operand)
  float* zdec = nullptr;          // FP32 [Omax][H]: A_{m-1} W_{m-1} of the decoder (no bias)
  xmgn::BfBuf dZdec;              // 16-bit [Omax][H]: S x dL/dz_{m-1} from the head
  float* gdec = nullptr;          // FP32 [Omax][H]: dL/dh^L (the processor's upstream gradient)
  double* sse_part = nullptr;     // per-warp SSE partials of the head
  float* wpart = nullptr;         // per-warp [H*4 + 4] partials of dW_m, db_m
  float* thin_part = nullptr;     // per-block [24][H] partials of the encoders' dW_1
  float* d_scale_dec = nullptr;   // {S, 1/S} of the decoder backward
  int last_model_fwd = -1;        // part of the last xmgn_model_fwd with targets (else -1)
  int head_warps = 0;
  bool infer = false;   // inference workspace: forward only, per-layer buffers ping-ponged
  bool pipe = true;     // N-half-pipelined chain kernel where a program allows it (XMGN_PIPE=0: off)
  bool prm_table = true;  // per-launch static bias/gamma/beta table in the chain kernels (XMGN_PRM_TABLE=0: off)
  // edge db_0 from the node-level D_dst column sums (XMGN_DB0_NODE=1).  Off by default: CFG4 -0.8%,
  // but the BF16 CFG2 run hung with it (profiles/r03k_db0_node_hang.txt; root cause not found)
  bool db0_node = false;
  bool dyn = false;     // dynamic tile scheduling in the chain kernels (XMGN_DYN=1, needs XMGN_STATIC_TILES=0)
  bool dyn_fwd = true;  // dynamic tiles in the edge-forward kernel (XMGN_DYN_FWD=0: off)
  int* d_tile_counter = nullptr;
  // checkpoint slot of layer l's tensors (training: one per layer; inference: ping-pong)
  long long ck(int l) const { return infer ? (l & 1) : l; }
};

namespace xmgn {

static void* dalloc(xmgn_workspace* ws, size_t bytes) {
  void* p = nullptr;
  bytes = (bytes + 255) & ~size_t(255);
  XMGN_CUDA(cudaMalloc(&p, bytes ? bytes : 256), "xmgn_workspace_create: cudaMalloc");
  ws->allocs.push_back(p);
  ws->bytes += bytes;
  return p;
}
static BfBuf bfalloc(xmgn_workspace* ws, size_t count) {
  BfBuf b;
  const int F = ws->split ? 2 : 1;
  b.p = static_cast<bf16*>(dalloc(ws, count * F * sizeof(bf16)));
  b.lo = ws->split ? (long long)count : 0;
  return b;
}

// ---- parameter layout (include/xmgn.h; an independent restatement of SURVEY §8(b))
struct Layout {
  int H, L, m;
  int64_t bs(int kin) const { return (int64_t)kin * H + H + (int64_t)m * ((int64_t)H * H + H) + 2 * (int64_t)H; }
  int64_t per() const { return bs(3 * H) + bs(2 * H); }
  int64_t base(int l, int blk) const { return l * per() + (blk ? bs(3 * H) : 0); }
  int kin(int blk) const { return blk ? 2 * H : 3 * H; }
  int64_t W(int l, int blk, int j) const {
    return base(l, blk) + (j == 0 ? 0 : (int64_t)kin(blk) * H + H + (int64_t)(j - 1) * ((int64_t)H * H + H));
  }
  int64_t b(int l, int blk, int j) const { return W(l, blk, j) + (int64_t)(j == 0 ? kin(blk) : H) * H; }
  int64_t gamma(int l, int blk) const { return base(l, blk) + (int64_t)kin(blk) * H + H + (int64_t)m * ((int64_t)H * H + H); }
  int64_t beta(int l, int blk) const { return gamma(l, blk) + H; }
  int64_t count() const { return (int64_t)L * per(); }
};

// Wk1 slots (rows of H, K = H): forward W^T and dgrad W for every H-wide operand.
enum { SL_E1T = 0, SL_PST = 1, SL_PDT = 2, SL_EJT = 3 };
static int sl_njt(int m) { return 3 + m; }        // node W_j^T, j = 1..m
static int sl_ej(int m) { return 3 + 2 * m; }     // edge W_j (dgrad), j = 1..m
static int sl_e1e(int m) { return 3 + 3 * m; }    // edge W_0 rows of e (dgrad)
static int sl_nj(int m) { return 4 + 3 * m; }     // node W_j (dgrad), j = 1..m
static int sl_n1h(int m) { return 4 + 4 * m; }    // node W_0 rows of h (dgrad)
static int sl_n1a(int m) { return 5 + 4 * m; }    // node W_0 rows of agg (dgrad)
static int n_sl1(int m) { return 6 + 4 * m; }
enum { SL2_N1T = 0, SL2_SD = 1 };                 // Wk2 (K = 2H): node W_0^T; [W_s | W_d] (proj bwd)

static std::vector<PackJob> pack_jobs(xmgn_workspace* ws) {
  const int H = ws->H, m = ws->m;
  Layout Ly{H, ws->L, m};
  std::vector<PackJob> J;
  auto job = [&](BfBuf& buf, int ld, long long row0, int col0, int rows, int cols, long long src, long long sr,
                 long long sc) {
    PackJob j;
    j.dst = buf.p + row0 * ld + col0;
    j.lo_off = buf.lo;
    j.ld = ld; j.rows = rows; j.cols = cols; j.src = src; j.sr = sr; j.sc = sc;
    J.push_back(j);
  };
  for (int l = 0; l < ws->L; ++l) {
    auto r1 = [&](int slot) { return (long long)(l * ws->S1 + slot) * H; };
    auto r2 = [&](int slot) { return (long long)(l * ws->S2 + slot) * H; };
    const int64_t We0 = Ly.W(l, 0, 0), Wn0 = Ly.W(l, 1, 0);
    // transposed (forward, B[n=out][k=in] = W[in][out])
    job(ws->wk1, H, r1(SL_E1T), 0, H, H, We0, 1, H);
    job(ws->wk1, H, r1(SL_PST), 0, H, H, We0 + (int64_t)H * H, 1, H);
    job(ws->wk1, H, r1(SL_PDT), 0, H, H, We0 + 2 * (int64_t)H * H, 1, H);
    for (int j = 1; j <= m; ++j) {
      job(ws->wk1, H, r1(SL_EJT + j - 1), 0, H, H, Ly.W(l, 0, j), 1, H);
      job(ws->wk1, H, r1(sl_njt(m) + j - 1), 0, H, H, Ly.W(l, 1, j), 1, H);
      // as stored (dgrad, B[n=in][k=out] = W[in][out])
      job(ws->wk1, H, r1(sl_ej(m) + j - 1), 0, H, H, Ly.W(l, 0, j), H, 1);
      job(ws->wk1, H, r1(sl_nj(m) + j - 1), 0, H, H, Ly.W(l, 1, j), H, 1);
    }
    job(ws->wk1, H, r1(sl_e1e(m)), 0, H, H, We0, H, 1);
    job(ws->wk1, H, r1(sl_n1h(m)), 0, H, H, Wn0, H, 1);
    job(ws->wk1, H, r1(sl_n1a(m)), 0, H, H, Wn0 + (int64_t)H * H, H, 1);
    job(ws->wk2, 2 * H, r2(SL2_N1T), 0, H, 2 * H, Wn0, 1, H);
    job(ws->wk2, 2 * H, r2(SL2_SD), 0, H, H, We0 + (int64_t)H * H, H, 1);
    job(ws->wk2, 2 * H, r2(SL2_SD), H, H, H, We0 + 2 * (int64_t)H * H, H, 1);
    if (ws->bsplit) {   // K-duplicated transposed weights: [A_hi | A_lo] x [W; W] = A W
      auto rx = [&](int slot) { return (long long)(l * 3 + slot) * H; };
      for (int d = 0; d < 2; ++d) {
        job(ws->wkx, 4 * H, rx(0), d * 2 * H, H, 2 * H, Wn0, 1, H);
        job(ws->wkx, 4 * H, rx(1), d * H, H, H, We0 + (int64_t)H * H, 1, H);
        job(ws->wkx, 4 * H, rx(2), d * H, H, H, We0 + 2 * (int64_t)H * H, 1, H);
      }
    }
  }
  return J;
}

// ---- tensor maps
static CUtensorMap map_rows(const bf16* base, long long rows, int width, int box_rows, bool f16) {
  return tmap16(base, (uint64_t)width, (uint64_t)(rows > 0 ? rows : 1), (uint64_t)width, 64, box_rows, f16);
}

// ---- chain program builder
struct Prog {
  ChainParams p;
  int n = 0;
  int next_map = 8;   // map slots 8.. hold the epilogues' TMA row inputs
  bool f16 = false;   // tensor-map element type of the 16-bit operands
  explicit Prog(const xmgn_workspace* ws) : f16(ws->f16) { std::memset(&p, 0, sizeof(p)); }
  Step& add() {
    Step& s = p.steps[n++];
    std::memset(&s, 0, sizeof(s));
    s.a_map1 = -1;
    s.in_map = -1;
    s.gsrc_map = -1;
    s.st_map = -1;
    return s;
  }
  // TMA gather source over P [rows][2H] 16-bit: 1-row boxes of 64 columns
  int gather_map(const bf16* base, long long rows, int width) {   // (P is FP16 in every 16-bit mode)
    if (next_map >= MAX_MAPS) throw Fail{set_error(XMGN_ESTATE, "internal: out of tensor-map slots")};
    p.maps[next_map] = tmap16(base, width, (uint64_t)(rows > 0 ? rows : 1), width, 64, 1, true);
    return next_map++;
  }
  // TMA source of an epilogue row input: 16-bit rows [0, rows) x H, rows > 0 (rows beyond read zero)
  int in_map(const bf16* base, long long rows, int H) {
    if (next_map >= MAX_MAPS) throw Fail{set_error(XMGN_ESTATE, "internal: out of tensor-map slots")};
    if (rows <= 0) throw Fail{set_error(XMGN_ESTATE, "internal: empty TMA input map")};
    p.maps[next_map] = tmap16(base, H, (uint64_t)rows, H, 64, 128, f16);
    return next_map++;
  }
};

static bool epi_writes_act(const Step& s) { return step_writes_act(s); }

// persistent grid: one cluster (CTA pair) per SM pair and resident CTA slot, at most one per pair tile
static int chain_grid(xmgn_workspace* ws, int M) {
  const int pair_tiles = (M + 255) / 256;
  const int slots = ws->sms / 2 * chain_ctas_per_sm(ws->H, ws->split);
  return 2 * (pair_tiles < slots ? pair_tiles : slots);
}

// Derive the ACT hand-off controls (chain.cuh) and launch.
static void run_prog(xmgn_workspace* ws, const char* name, Prog& pr, int M, const int* src, const int* dst, bool bwd,
                     cudaStream_t st) {
  if (M <= 0) return;
  ChainParams& p = pr.p;
  p.n_steps = pr.n;
  p.M = M;
  p.src = src;
  p.dst = dst;
  p.eps = ws->cfg.ln_eps;
  const int n = pr.n;
  if (epi_writes_act(p.steps[n - 1])) throw Fail{set_error(XMGN_ESTATE, "internal: program ends writing ACT")};
  for (int s = 0; s < n; ++s) {
    Step& S = p.steps[s];
    S.ctl = 0;
    if (S.a_src == A_ACT) {
      if (s == 0) throw Fail{set_error(XMGN_ESTATE, "internal: program starts with A_ACT")};
      if (epi_writes_act(p.steps[s - 1])) S.ctl |= CTL_WAIT_ACT;
    } else {
      // ACT used since the previous A_TMA step (cyclically)?
      bool used = false;
      for (int t = 1; t < n; ++t) {
        const Step& T = p.steps[(s - t + n) % n];
        if (T.a_src == A_ACT || epi_writes_act(T)) used = true;
        if (T.a_src == A_TMA) break;
      }
      if (used) S.ctl |= CTL_NEED_ACT_FREE;
    }
  }
  // static parameter table (chain.cuh ChainParams::n_prm): the program's distinct bias / gamma /
  // beta vectors (null = one zero row) if they fit the kernel's 6-row PRM region
  {
    p.n_prm = 0;
    int n = 0;
    bool fits = !ws->split && ws->prm_table;
    for (int s = 0; s < pr.n && fits; ++s) {
      const float* v3[3] = {p.steps[s].bias, p.steps[s].gamma, p.steps[s].beta};
      for (int k = 0; k < 3 && fits; ++k) {
        int slot = -1;
        for (int i = 0; i < n; ++i)
          if (p.prm_src[i] == v3[k]) slot = i;
        if (slot < 0) {
          if (n == 6) { fits = false; break; }
          p.prm_src[n] = v3[k];
          slot = n++;
        }
        p.prm_slot[s][k] = (signed char)slot;
      }
    }
    if (fits) p.n_prm = n;
  }
  // weight maps
  const int NB = (ws->H < 256 ? ws->H : 256) / 2;   // B rows per CTA of a pair
  const long long r1 = (long long)ws->L * ws->S1 * ws->H, r2 = (long long)ws->L * ws->S2 * ws->H;
  const bool f16 = ws->f16;
  p.maps[0] = tmap16(ws->wk1.p, ws->H, r1, ws->H, 64, NB, f16);
  p.maps[1] = ws->split ? tmap16(ws->wk1.p + ws->wk1.lo, ws->H, r1, ws->H, 64, NB, f16) : p.maps[0];
  p.maps[2] = tmap16(ws->wk2.p, 2 * ws->H, r2, 2 * ws->H, 64, NB, f16);
  p.maps[3] = ws->split ? tmap16(ws->wk2.p + ws->wk2.lo, 2 * ws->H, r2, 2 * ws->H, 64, NB, f16) : p.maps[2];
  if (ws->bsplit)   // slot 1 (the SPLIT-mode lo slot) holds the K-duplicated weights
    p.maps[1] = tmap16(ws->wkx.p, 4 * ws->H, (long long)ws->L * 3 * ws->H, 4 * ws->H, 64, NB, f16);
  const int grid = chain_grid(ws, M);
  const int pair_tiles = (M + 255) / 256;
  p.colsum = bwd ? ws->colsum : nullptr;
  if (bwd) {
    // column-sum vectors this program writes -> consecutive slots of per-tile partials (each
    // written once per launch: no zeroing)
    bool used[NV_MAX] = {false, false, false, false, false};
    for (int s = 0; s < n; ++s) {
      const Step& S = p.steps[s];
      if (S.epi == EPI_LN_BWD) {
        used[0] = true;
        if (S.flags & EF_COLSUM_ALL) used[1] = used[2] = true;
      }
      if (S.epi == EPI_DSILU && (S.flags & EF_COLSUM_ALL)) used[S.vec0] = true;
    }
    int ns = 0;
    for (int v = 0; v < NV_MAX; ++v) p.cs_slot[v] = used[v] ? ns++ : -1;
    const int nct = 2 * pair_tiles;
    p.cs_vstride = (long long)nct * 4 * ws->H;
    if ((size_t)ns * (size_t)p.cs_vstride > ws->colsum_cap)
      throw Fail{set_error(XMGN_ESTATE, "internal: column-sum partials exceed the workspace (%d slots x %d tiles)", ns,
                           nct)};
    for (int v = 0; v < NV_MAX; ++v) ws->cs_slot[v] = p.cs_slot[v];
    ws->cs_nct = nct;
  }
  const bool pipe = ws->pipe && chain_can_pipe(ws->H, ws->split, p);
  // dynamic tiles: every program with XMGN_DYN=1 (needs XMGN_STATIC_TILES=0), and the edge forward
  // (its kernel compiles the queue in; XMGN_DYN_FWD=0: static)
  const bool dyn = ws->dyn || (ws->dyn_fwd && !strcmp(name, "chain_edge_fwd")) ||
                   (ws->dyn_fwd && chain_dyn(ws->H, ws->split));
  p.tile_counter = dyn ? ws->d_tile_counter : nullptr;
  if (dyn) XMGN_CUDA(cudaMemsetAsync(ws->d_tile_counter, 0, sizeof(int), st), "tile counter");
  {
    ProfScope ps(name, st);
    launch_chain(ws->H, ws->split, ws->f16, bwd, p, grid, st, pipe);
  }
  XMGN_CUDA(cudaGetLastError(), "chain kernel launch");
}



static void set_a(xmgn_workspace* ws, Prog& pr, int slot, const BfBuf& b, long long rows, int width) {
  pr.p.maps[slot] = map_rows(b.p, rows, width, 128, ws->f16);
  pr.p.maps[slot + 1] = ws->split ? map_rows(b.p + b.lo, rows, width, 128, ws->f16) : pr.p.maps[slot];
}

static BfBuf at(const BfBuf& b, long long elem) { return BfBuf{b.p + elem, b.lo}; }

// weight-gradient GEMM + fixed-order reduction into grad[dst .. dst + Hin*Hout); with
// bias_dst >= 0 an extra all-ones A tile also yields grad[bias_dst + c] += sum_rows B[:, c].
// Hin = 0 computes only that column sum.
static void wgrad(xmgn_workspace* ws, const BfBuf& a0, const BfBuf& a1, int a_width, int a_split_tiles, const BfBuf& b,
                  int b_width, int b_col0, long long rows, int Hin, float* grad, long long dst, cudaStream_t st,
                  long long bias_dst = -1, const float* inv = nullptr) {
  if (rows <= 0) return;
  const int H = ws->H;
  WgradParams p;
  std::memset(&p, 0, sizeof(p));
  const BfBuf& a0r = a0.p ? a0 : b;
  const int aw = a0.p ? a_width : b_width;
  const bool f16 = ws->f16;
  p.a0 = tmap16(a0r.p, aw, rows, aw, 64, 64, f16);
  p.a0lo = ws->split ? tmap16(a0r.p + a0r.lo, aw, rows, aw, 64, 64, f16) : p.a0;
  const BfBuf& a1r = a1.p ? a1 : a0r;
  p.a1 = tmap16(a1r.p, aw, rows, aw, 64, 64, f16);
  p.a1lo = ws->split ? tmap16(a1r.p + a1r.lo, aw, rows, aw, 64, 64, f16) : p.a1;
  p.b = tmap16(b.p, b_width, rows, b_width, 64, 64, f16);
  p.blo = ws->split ? tmap16(b.p + b.lo, b_width, rows, b_width, 64, 64, f16) : p.b;
  p.a_split_tiles = a_split_tiles;
  p.b_col0 = b_col0;
  p.rows = (int)rows;
  p.Hin = Hin;
  p.Hout = H;
  p.ones_tile = bias_dst >= 0;
  const int NT = H >= 256 ? 256 : H;
  const int tiles = (Hin / 128 + (p.ones_tile ? 1 : 0)) * (H / NT);
  const int chunks = (int)((rows + 63) / 64);
  // one wave: tiles x S <= SMs x resident CTAs per SM (no tail wave)
  int S = ws->sms * wgrad_ctas_per_sm(H, ws->split) / tiles;
  if (S > chunks) S = chunks;
  if (S > ws->part_splits) S = ws->part_splits;
  if (S < 1) S = 1;
  p.n_split = S;
  p.part = ws->part;
  {
    ProfScope ps("wgrad", st);
    launch_wgrad(p, ws->split, ws->f16, st);
  }
  XMGN_CUDA(cudaGetLastError(), "wgrad launch");
  const long long ld = (long long)(Hin + (p.ones_tile ? 128 : 0)) * H;
  if (!inv) inv = ws->d_scale + 1;
  // weight and bias partials are contiguous per split: one fixed-order reduce launch for both
  if (Hin > 0 && p.ones_tile)
    launch_reduce_part(ws->part, S, (long long)Hin * H + H, ld, grad + dst, st, inv, (long long)Hin * H,
                       grad + bias_dst);
  else if (Hin > 0) launch_reduce_part(ws->part, S, (long long)Hin * H, ld, grad + dst, st, inv);
  else if (p.ones_tile) launch_reduce_part(ws->part + (long long)Hin * H, S, H, ld, grad + bias_dst, st, inv);
}

// grad[off[v] + c] += (1/S) sum over the last backward launch's tiles and quadrants of vector v
static void reduce_colsums(xmgn_workspace* ws, const ColsumDst& d, float* grad, cudaStream_t st) {
  ColsumDst dd = d;
  for (int v = 0; v < NV_MAX; ++v)
    if (dd.off[v] >= 0 && ws->cs_slot[v] < 0)
      throw Fail{set_error(XMGN_ESTATE, "internal: column-sum vector %d was not written", v)};
  launch_reduce_colsum(ws->colsum, ws->cs_nct, ws->cs_slot, ws->H, dd, ws->cs_tmp, grad, st, ws->d_scale + 1);
}

static void colsum_reduce(xmgn_workspace* ws, int blk, int l, float* grad, int grid_used, cudaStream_t st,
                          bool gamma_only = false) {
  (void)grid_used;
  Layout Ly{ws->H, ws->L, ws->m};
  ColsumDst d;
  for (int v = 0; v < NV_MAX; ++v) d.off[v] = -1;
  d.off[0] = Ly.gamma(l, blk);
  if (!gamma_only) {
    d.off[1] = Ly.beta(l, blk);
    d.off[2] = Ly.b(l, blk, ws->m);
    d.off[3] = Ly.b(l, blk, ws->m - 1);
    if (ws->m >= 2) d.off[4] = Ly.b(l, blk, ws->m - 2);
  }
  reduce_colsums(ws, d, grad, st);
}

}  // namespace xmgn

using namespace xmgn;

extern "C" size_t xmgn_param_count(const xmgn_model_cfg* c) {
  if (!c || c->hidden <= 0 || c->layers <= 0 || c->mlp_hidden_layers < 1) return 0;
  Layout Ly{c->hidden, c->layers, c->mlp_hidden_layers};
  return (size_t)Ly.count();
}

static xmgn_status workspace_create(const xmgn_graph* g, const xmgn_model_cfg* cfg, xmgn_workspace** out,
                                    bool infer) {
  return guarded("xmgn_workspace_create", [&]() -> xmgn_status {
    if (!g || !cfg || !out) return set_error(XMGN_EINVAL, "xmgn_workspace_create: null argument");
    *out = nullptr;
    const int H = cfg->hidden, L = cfg->layers, m = cfg->mlp_hidden_layers;
    if (!(H == 128 || H == 256 || H == 512))
      return set_error(XMGN_EUNSUPPORTED, "xmgn_workspace_create: hidden=%d (kernels built for 128, 256, 512)", H);
    if (m < 1 || m > 2) return set_error(XMGN_EUNSUPPORTED, "xmgn_workspace_create: mlp_hidden_layers=%d (1 or 2)", m);
    if (L < 1) return set_error(XMGN_EINVAL, "xmgn_workspace_create: layers=%d", L);
    if (cfg->precision == XMGN_PREC_FP32_CHECK && H != 128)
      return set_error(XMGN_EUNSUPPORTED, "xmgn_workspace_create: FP32 check mode is built for hidden=128 only");
    if (cfg->precision != XMGN_PREC_BF16 && cfg->precision != XMGN_PREC_FP32_CHECK &&
        cfg->precision != XMGN_PREC_FP16)
      return set_error(XMGN_EINVAL, "xmgn_workspace_create: precision=%d", cfg->precision);
    if (L > g->depth)
      return set_error(XMGN_EHALO,
                       "xmgn_workspace_create: layers=%d exceeds halo_depth=%d (owned outputs would differ from the "
                       "full graph, PAPER.md:172)",
                       L, g->depth);
    XMGN_CUDA(cudaSetDevice(g->device), "xmgn_workspace_create: cudaSetDevice");
    auto* ws = new xmgn_workspace();
    try {
      ws->g = g;
      ws->cfg = *cfg;
      ws->infer = infer;
      { const char* pe = getenv("XMGN_PIPE"); ws->pipe = !(pe && atoi(pe) == 0); }
      { const char* pt = getenv("XMGN_PRM_TABLE"); ws->prm_table = !(pt && atoi(pt) == 0); }
      { const char* db = getenv("XMGN_DB0_NODE"); ws->db0_node = db && atoi(db) == 1; }
      { const char* de = getenv("XMGN_DYN"); ws->dyn = de && atoi(de) == 1; }   // see XMGN_STATIC_TILES
      { const char* df = getenv("XMGN_DYN_FWD"); ws->dyn_fwd = !(df && atoi(df) == 0); }
      ws->dev = g->device;
      ws->H = H; ws->L = L; ws->m = m;
      ws->split = cfg->precision == XMGN_PREC_FP32_CHECK;
      ws->f16 = cfg->precision == XMGN_PREC_FP16;
      cudaDeviceGetAttribute(&ws->sms, cudaDevAttrMultiProcessorCount, g->device);
      for (const Part& P : g->parts) {
        ws->Nmax = std::max(ws->Nmax, P.n_local);
        ws->Emax = std::max(ws->Emax, P.e_local);
      }
      ws->Rmax = std::max(ws->Nmax, ws->Emax);
      // graph arrays
      for (const Part& P : g->parts) {
        DPart d;
        std::vector<int32_t> off32(P.offsets.begin(), P.offsets.end());
        d.off = (int*)dalloc(ws, off32.size() * 4);
        d.src = (int*)dalloc(ws, P.e_local * 4);
        d.dst = (int*)dalloc(ws, P.e_local * 4);
        d.rev = (int*)dalloc(ws, P.e_local * 4);
        XMGN_CUDA(cudaMemcpy(d.off, off32.data(), off32.size() * 4, cudaMemcpyHostToDevice), "upload");
        XMGN_CUDA(cudaMemcpy(d.src, P.src.data(), P.e_local * 4, cudaMemcpyHostToDevice), "upload");
        XMGN_CUDA(cudaMemcpy(d.dst, P.dst.data(), P.e_local * 4, cudaMemcpyHostToDevice), "upload");
        XMGN_CUDA(cudaMemcpy(d.rev, P.rev.data(), P.e_local * 4, cudaMemcpyHostToDevice), "upload");
        ws->dparts.push_back(d);
      }
      const size_t NH = (size_t)ws->Nmax * H, EH = (size_t)ws->Emax * H, RH = (size_t)ws->Rmax * H;
      ws->S1 = n_sl1(m);
      ws->S2 = 2;
      ws->wk1 = bfalloc(ws, (size_t)L * ws->S1 * H * H);
      ws->wk2 = bfalloc(ws, (size_t)L * ws->S2 * H * 2 * H);
      ws->bsplit = cfg->precision == XMGN_PREC_BF16;
      if (ws->bsplit) ws->wkx = bfalloc(ws, (size_t)L * 3 * H * 4 * H);
      std::vector<PackJob> jobs = pack_jobs(ws);
      ws->njobs = (int)jobs.size();
      ws->d_jobs = (PackJob*)dalloc(ws, jobs.size() * sizeof(PackJob));
      XMGN_CUDA(cudaMemcpy(ws->d_jobs, jobs.data(), jobs.size() * sizeof(PackJob), cudaMemcpyHostToDevice), "upload");
      // training keeps every layer's 16-bit operands (activation checkpoints);
      // inference ping-pongs them: ~2 layers of activation memory
      const int ckL = infer ? 2 : L;
      ws->e_ck = bfalloc(ws, (size_t)(infer ? 2 : L + 1) * EH);
      ws->h_ck = bfalloc(ws, (size_t)ckL * NH);
      ws->a_ck = bfalloc(ws, (size_t)(infer ? 1 : L) * NH);
      for (int i = 0; i < 2; ++i) ws->h_buf[i] = (float*)dalloc(ws, NH * 4);
      // BF16 operands (8-bit mantissa) need the edge residual stream and the aggregation in
      // FP32 to stay inside north_star's 2e-2 x RMS at 15 layers (rung R1);
      // FP16 operands meet it with the 16-bit stream
      ws->e32_mode = cfg->precision == XMGN_PREC_BF16;
      if (ws->e32_mode)
        for (int i = 0; i < 2; ++i) ws->e32[i] = (float*)dalloc(ws, EH * 4);
      {
        const char* le = getenv("XMGN_LN_STATS");
        if (!infer && !ws->split && !(le && atoi(le) == 0)) {
          ws->lnst_e = (float2*)dalloc(ws, (size_t)L * ws->Emax * sizeof(float2));
          ws->lnst_n = (float2*)dalloc(ws, (size_t)L * ws->Nmax * sizeof(float2));
        }
      }
      if (ws->bsplit) {
        for (int i = 0; i < 2; ++i) ws->hlo[i] = (bf16*)dalloc(ws, NH * 2);
        ws->alo = (bf16*)dalloc(ws, NH * 2);
      }
      ws->P = bfalloc(ws, (size_t)ckL * 2 * NH);
      if (!infer) {
        ws->Ge[0] = bfalloc(ws, EH);
        ws->Ge[1] = bfalloc(ws, EH);
        ws->Gh = (float*)dalloc(ws, NH * 4);
        ws->Ga = bfalloc(ws, NH);
        for (int j = 0; j < m; ++j) { ws->scrA[j] = bfalloc(ws, RH); ws->scrS[j] = bfalloc(ws, RH); }
        for (int j = 0; j <= m; ++j) ws->scrZ[j] = bfalloc(ws, RH);
        ws->D = bfalloc(ws, 2 * NH);
        ws->part_splits = 64;   // more splits cost more in k_reduce_part than they save (r03f)
        ws->part = (float*)dalloc(ws, (size_t)ws->part_splits * (2 * H + 128) * H * 4);
        // per-tile partials: edge programs write one vector (dgamma), node programs up to NV_MAX
        const size_t nct_e = 2 * (size_t)((ws->Emax + 255) / 256), nct_n = 2 * (size_t)((ws->Nmax + 255) / 256);
        ws->colsum_cap = std::max(nct_e, NV_MAX * nct_n) * 4 * H;
        ws->colsum = (float*)dalloc(ws, ws->colsum_cap * 4);
        ws->cs_tmp = (float*)dalloc(ws, (size_t)NV_MAX * CS_SEG * H * 4);
      }
      ws->d_amax = (unsigned int*)dalloc(ws, 4);
      ws->d_tile_counter = (int*)dalloc(ws, 4);
      ws->d_scale = (float*)dalloc(ws, 2 * sizeof(float));
      // Opt-in (XMGN_Z1=1) memory-for-speed mode: z_1 checkpoints (+L x E x H x 2 bytes) let
      // the backward skip the first edge GEMM's recompute (edge bwd -5%).  Off by default: at
      // CFG4 on one GPU they would not leave room for the 62 GB of resident inputs.
      // Explicitly requested: failing to allocate it is an error (ENOMEM), never a silent
      // fall-back to the default mode.
      const char* z1env = getenv("XMGN_Z1");
      if (!infer && z1env && atoi(z1env) == 1) {
        if (ws->split)
          throw Fail{set_error(XMGN_EUNSUPPORTED, "xmgn_workspace_create: XMGN_Z1=1 needs a 16-bit precision mode")};
        ws->z1_ck = bfalloc(ws, (size_t)L * EH);
        ws->use_z1 = true;
      }
    } catch (...) {
      xmgn_workspace_free(ws);
      throw;
    }
    *out = ws;
    return XMGN_OK;
  });
}

extern "C" xmgn_status xmgn_workspace_create(const xmgn_graph* g, const xmgn_model_cfg* cfg, xmgn_workspace** out) {
  return workspace_create(g, cfg, out, false);
}
extern "C" xmgn_status xmgn_workspace_create_infer(const xmgn_graph* g, const xmgn_model_cfg* cfg,
                                                   xmgn_workspace** out) {
  return workspace_create(g, cfg, out, true);
}

extern "C" size_t xmgn_workspace_bytes(const xmgn_workspace* ws) { return ws ? ws->bytes : 0; }

extern "C" void xmgn_workspace_free(xmgn_workspace* ws) {
  if (!ws) return;
  for (void* p : ws->allocs) cudaFree(p);
  delete ws;
}

static inline int64_t n_at(const Part& P, int L, int l) {  // rows of layer l (ring <= L-l)
  return P.ring_nodes[L - l + 1];
}
static inline int64_t e_at(const Part& P, int L, int l) { return P.ring_edges[L - l + 1]; }

// The processor forward of partition `part`.  staged: the encoders (xmgn_model_fwd) already
// wrote h^0 (FP32 h0 = h_buf[0] and its 16-bit copy h_ck[0]) and e^0 (16-bit e_ck[0], FP32 e0 =
// e32[0] in the BF16 mode); hL16 (may be null): also write h^L of the owned rows in 16 bits.
static void proc_fwd(xmgn_workspace* ws, int part, const float* params, const float* h0, const float* e0,
                     float* h_out, bool staged, bf16* hL16, cudaStream_t st) {
  {
    const Part& P = ws->g->parts[part];
    const DPart& dp = ws->dparts[part];
    const int H = ws->H, L = ws->L, m = ws->m;
    const long long NH = ws->Nmax * (long long)H, EH = ws->Emax * (long long)H;
    Layout Ly{H, L, m};
    launch_pack(ws->f16, params, ws->d_jobs, ws->njobs, st);
    const int64_t n0 = n_at(P, L, 0), e1 = e_at(P, L, 1);
    if (!staged) {
      launch_to_bf16(ws->f16, h0, ws->h_ck.p, ws->h_ck.lo, n0 * H, st);
      launch_to_bf16(ws->f16, e0, ws->e_ck.p, ws->e_ck.lo, e1 * H, st);
    }
    if (ws->bsplit)   // h^0 = hi + lo (hi rewritten with the same RNE bits)
      launch_to_bf16x2(h0, ws->h_ck.p, ws->hlo[0], n0 * H, st);
    const int W1 = 0, W2 = 2;  // weight map slots
    auto r1 = [&](int l, int slot) { return (l * ws->S1 + slot) * H; };
    auto r2 = [&](int l, int slot) { return (l * ws->S2 + slot) * H; };
    auto Pl = [&](int li) { return ws->P.p + ws->ck(li) * 2 * NH; };   // P of layer li + 1
    // P = h^l [W1e_s | W1e_d] for layer l + 1 as its own launch (layer 1; BF16 mode: every layer,
    // from 2 x BF16 h^l = [h_hi | h_lo] against [W; W]); 16-bit modes store P in FP16
    auto proj = [&](int l) {
      const int64_t nr = n_at(P, L, l);
      Prog pr(ws);
      const BfBuf hck = at(ws->h_ck, ws->ck(l) * NH);
      set_a(ws, pr, 4, hck, nr, H);
      if (ws->bsplit) pr.p.maps[5] = map_rows(ws->hlo[l & 1], nr, H, 128, false);
      for (int half = 0; half < 2; ++half) {
        Step& s = pr.add();
        s.a_src = A_TMA; s.a_map0 = 4; s.K = H;
        s.b_map = W1; s.b_row0 = r1(l, half ? SL_PDT : SL_PST);
        if (ws->bsplit) {
          s.a_map1 = 5; s.a_ksplit = H; s.K = 2 * H;
          s.b_map = 1; s.b_row0 = (l * 3 + 1 + half) * H;
        }
        s.epi = EPI_STORE; s.flags = EF_OUT16 | (ws->split ? 0 : EF_OUT_HALF);
        s.bf_out = Pl(l); s.bf_lo = ws->P.lo; s.ld_out = 2 * H;
        s.col0 = half * H;
      }
      run_prog(ws, "chain_proj", pr, (int)nr, nullptr, nullptr, false, st);
    };
    proj(0);
    int cur = 0, ce = 0;   // ping-pong indices of the FP32 node (and BF16-mode edge) streams
    for (int l = 1; l <= L; ++l) {
      const int li = l - 1;
      const int64_t nl = n_at(P, L, l), el = e_at(P, L, l);
      const float* h_in = l == 1 ? h0 : ws->h_buf[cur];
      BfBuf eck_next = at(ws->e_ck, ws->ck(l) * EH);
      float* hn = l == L ? h_out : ws->h_buf[cur ^ 1];
      BfBuf eck_prev = at(ws->e_ck, ws->ck(li) * EH), hck_prev = at(ws->h_ck, ws->ck(li) * NH);
      BfBuf ack = at(ws->a_ck, ws->infer ? 0 : (long long)li * NH);
      {  // edge update (Eq. 1)
        Prog pr(ws);
        set_a(ws, pr, 4, eck_prev, el, H);
        for (int j = 0; j < m; ++j) {
          Step& s = pr.add();
          s.a_src = j == 0 ? A_TMA : A_ACT; s.a_map0 = 4; s.K = H;
          s.b_map = W1; s.b_row0 = r1(li, j == 0 ? SL_E1T : SL_EJT + j - 1);
          s.epi = EPI_SILU; s.bias = params + Ly.b(li, 0, j);
          if (j == 0) {
            s.flags |= EF_GATHER_P; s.gather16 = Pl(li); s.gather16_lo = ws->P.lo;
            if (!ws->split) s.gsrc_map = pr.gather_map(Pl(li), P.n_local, 2 * H);
            if (ws->use_z1) { s.flags |= EF_STORE_Z; s.scr_z = ws->z1_ck.p + (long long)li * EH; }
          }
        }
        // e^l = e^{l-1} + LN(..): the edge stream itself is 16-bit (checkpoint = next operand);
        // BF16 mode carries it in FP32 and writes the 16-bit operand / checkpoint beside it
        Step& s = pr.add();
        s.a_src = A_ACT; s.K = H; s.b_map = W1; s.b_row0 = r1(li, SL_EJT + m - 1);
        s.epi = EPI_LN_FWD; s.bias = params + Ly.b(li, 0, m);
        s.gamma = params + Ly.gamma(li, 0); s.beta = params + Ly.beta(li, 0);
        if (ws->e32_mode) {
          s.flags = EF_STORE_F32 | EF_STORE_BF;
          s.f_in = l == 1 ? e0 : ws->e32[ce]; s.ld_in = H;
          s.f_out = ws->e32[ce ^ 1]; s.ld_out = H;
        } else {
          s.flags = EF_RES16 | EF_STORE_BF;
          s.res16 = eck_prev.p; s.res16_lo = eck_prev.lo;
          if (!ws->split && el > 0) s.in_map = pr.in_map(eck_prev.p, el, H);   // residual e^{l-1} rows
        }
        s.bf_out = eck_next.p; s.bf_lo = eck_next.lo;
        if (ws->lnst_e) { s.flags |= EF_ST_SAVE; s.ln_st = ws->lnst_e + (long long)li * ws->Emax; }
        run_prog(ws, "chain_edge_fwd", pr, (int)el, dp.src, dp.dst, false, st);
      }
      // aggregation (Eq. 2) -> a^l (BF16 operand + checkpoint)
      { ProfScope ps("aggregate", st);
      if (ws->e32_mode) launch_aggregate32(H, dp.off, ws->e32[ce ^ 1], ack.p, ws->bsplit ? ws->alo : nullptr, (int)nl, st);
      else launch_aggregate(ws->f16, H, dp.off, eck_next.p, eck_next.lo, ack.p, ack.lo, (int)nl, st); }
      ce ^= 1;
      XMGN_CUDA(cudaGetLastError(), "aggregate launch");
      {  // node update (Eq. 3) [+ P for layer l+1]
        Prog pr(ws);
        set_a(ws, pr, 4, hck_prev, nl, H);
        set_a(ws, pr, 6, ack, nl, H);
        if (ws->bsplit) {   // A = [h_hi | a_hi | h_lo | a_lo] (slots 4..7), B = [W0; W0]
          pr.p.maps[5] = pr.p.maps[6];
          pr.p.maps[6] = map_rows(ws->hlo[li & 1], nl, H, 128, false);
          pr.p.maps[7] = map_rows(ws->alo, nl, H, 128, false);
        }
        for (int j = 0; j < m; ++j) {
          Step& s = pr.add();
          s.a_src = j == 0 ? A_TMA : A_ACT; s.a_map0 = 4; s.a_map1 = 6; s.a_ksplit = H;
          s.K = j == 0 ? 2 * H : H;
          s.b_map = j == 0 ? W2 : W1; s.b_row0 = j == 0 ? r2(li, SL2_N1T) : r1(li, sl_njt(m) + j - 1);
          if (j == 0 && ws->bsplit) { s.a_map1 = 5; s.K = 4 * H; s.b_map = 1; s.b_row0 = li * 3 * H; }
          s.epi = EPI_SILU; s.bias = params + Ly.b(li, 1, j);
        }
        Step& s = pr.add();
        s.a_src = A_ACT; s.K = H; s.b_map = W1; s.b_row0 = r1(li, sl_njt(m) + m - 1);
        s.epi = EPI_LN_FWD; s.bias = params + Ly.b(li, 1, m);
        s.gamma = params + Ly.gamma(li, 1); s.beta = params + Ly.beta(li, 1);
        s.f_in = h_in; s.ld_in = H; s.f_out = hn; s.ld_out = H;
        s.flags = EF_STORE_F32;
        if (ws->lnst_n) { s.flags |= EF_ST_SAVE; s.ln_st = ws->lnst_n + (long long)li * ws->Nmax; }
        if (l == L && hL16) {
          s.flags |= EF_STORE_BF;
          s.bf_out = hL16; s.bf_lo = 0;
        }
        if (l < L && ws->bsplit) {   // h^l = hi + lo; P of layer l + 1 by proj(l) below
          s.flags |= EF_STORE_BF | EF_STORE_LO;
          s.bf_out = ws->h_ck.p + ws->ck(l) * NH; s.bf_lo = 0;
          s.lo_out = ws->hlo[l & 1];
        } else if (l < L) {
          s.flags |= EF_STORE_BF | EF_WRITE_ACT;
          s.bf_out = ws->h_ck.p + ws->ck(l) * NH; s.bf_lo = ws->h_ck.lo;
          for (int half = 0; half < 2; ++half) {
            Step& q = pr.add();
            q.a_src = A_ACT; q.K = H; q.b_map = W1; q.b_row0 = r1(l, half ? SL_PDT : SL_PST);
            q.epi = EPI_STORE; q.flags = EF_OUT16 | (ws->split ? 0 : EF_OUT_HALF);
            q.bf_out = Pl(l); q.bf_lo = ws->P.lo; q.ld_out = 2 * H;
            q.col0 = half * H;
          }
        }
        run_prog(ws, "chain_node_fwd", pr, (int)nl, nullptr, nullptr, false, st);
      }
      if (ws->bsplit && l < L) proj(l);
      cur ^= 1;
    }
    ws->last_fwd = part;
  }
}

extern "C" xmgn_status xmgn_processor_fwd(xmgn_workspace* ws, int part, const float* params, const float* h0,
                                          const float* e0, float* h_out, void* stream) {
  return guarded("xmgn_processor_fwd", [&]() -> xmgn_status {
    if (!ws || !params || !h0 || !e0 || !h_out) return set_error(XMGN_EINVAL, "xmgn_processor_fwd: null argument");
    if (part < 0 || part >= (int)ws->g->parts.size())
      return set_error(XMGN_EINVAL, "xmgn_processor_fwd: part=%d outside [0,%d)", part, (int)ws->g->parts.size());
    XMGN_CUDA(cudaSetDevice(ws->dev), "xmgn_processor_fwd: cudaSetDevice");
    ws->last_model_fwd = -1;
    proc_fwd(ws, part, params, h0, e0, h_out, false, nullptr, (cudaStream_t)stream);
    return XMGN_OK;
  });
}

extern "C" xmgn_status xmgn_processor_bwd(xmgn_workspace* ws, int part, const float* params, const float* grad_h_out,
                                          float* grad_params, float* grad_h0, float* grad_e0, void* stream) {
  return guarded("xmgn_processor_bwd", [&]() -> xmgn_status {
    if (!ws || !params || !grad_h_out || !grad_params)
      return set_error(XMGN_EINVAL, "xmgn_processor_bwd: null argument");
    if (ws->infer)
      return set_error(XMGN_ESTATE, "xmgn_processor_bwd: inference workspace (no checkpoints; use xmgn_workspace_create)");
    if (part != ws->last_fwd)
      return set_error(XMGN_ESTATE, "xmgn_processor_bwd: part=%d but the workspace holds the forward of part %d",
                       part, ws->last_fwd);
    XMGN_CUDA(cudaSetDevice(ws->dev), "xmgn_processor_bwd: cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    const Part& P = ws->g->parts[part];
    const DPart& dp = ws->dparts[part];
    const int H = ws->H, L = ws->L, m = ws->m;
    const long long NH = ws->Nmax * (long long)H, EH = ws->Emax * (long long)H;
    auto Pl = [&](int li) { return ws->P.p + (long long)li * 2 * NH; };   // the forward's P of layer li + 1
    Layout Ly{H, L, m};
    const int W1 = 0, W2 = 2;
    auto r1 = [&](int l, int slot) { return (l * ws->S1 + slot) * H; };
    auto r2 = [&](int l, int slot) { return (l * ws->S2 + slot) * H; };
    launch_pack(ws->f16, params, ws->d_jobs, ws->njobs, st);
    // seed: dL/dh^L on owned rows (the loss mask of PAPER.md:197 is the prefix)
    // (times S, a power of two putting max|g| in [1, 2): every gradient that leaves is
    // multiplied by 1/S again -- exact loss scaling of the 16-bit gradient streams)
    launch_seed_scale(grad_h_out, (long long)P.n_owned * H, ws->d_amax, ws->Gh, ws->d_scale, st);
    const BfBuf none{};
    int gc = 0;   // which G_e buffer holds G_e^l
    for (int l = L; l >= 1; --l) {
      const int li = l - 1;
      const int64_t nl = n_at(P, L, l), el = e_at(P, L, l), nprev = n_at(P, L, l - 1);
      const int64_t enext = l < L ? e_at(P, L, l + 1) : 0;
      BfBuf eck = at(ws->e_ck, (long long)li * EH), hck = at(ws->h_ck, (long long)li * NH);
      BfBuf ack = at(ws->a_ck, (long long)li * NH);
      // common recompute + dgrad program of an MLP block (blk 0 edge, 1 node)
      auto mlp_bwd = [&](Prog& pr, int blk) {
        const long long rows = blk ? nl : el;
        for (int j = 0; j < m; ++j) {
          Step& s = pr.add();
          s.a_src = j == 0 ? A_TMA : A_ACT; s.a_map0 = 4;
          if (blk == 1) { s.a_map1 = 6; s.a_ksplit = H; }
          s.K = (j == 0 && blk == 1) ? 2 * H : H;
          s.b_map = (j == 0 && blk == 1) ? W2 : W1;
          s.b_row0 = j == 0 ? (blk ? r2(li, SL2_N1T) : r1(li, SL_E1T))
                            : r1(li, (blk ? sl_njt(m) : SL_EJT) + j - 1);
          s.epi = EPI_SILU; s.bias = params + Ly.b(li, blk, j);
          s.flags = EF_STORE_A | EF_STORE_S;
          s.scr_a = ws->scrA[j].p; s.scr_s = ws->scrS[j].p; s.lo_off = ws->scrA[j].lo;
          if (!ws->split && rows > 0) s.st_map = pr.in_map(ws->scrA[j].p, rows, H);   // A_j = the ACT tile, TMA-stored
          if (j == 0 && blk == 0) {
            if (ws->use_z1 && rows > 0) {
              // z_1 from the forward's checkpoint: no GEMM, no gathers (a K = 0 step)
              s.K = 0; s.bias = nullptr;
              s.flags |= EF_FROM_IN;
              s.in_map = pr.in_map(ws->z1_ck.p + (long long)li * EH, rows, H);
            } else {
              s.flags |= EF_GATHER_P; s.gather16 = Pl(li); s.gather16_lo = ws->P.lo;
              if (!ws->split) s.gsrc_map = pr.gather_map(Pl(li), P.n_local, 2 * H);
            }
          }
        }
        Step& s = pr.add();
        s.a_src = A_ACT; s.K = H; s.b_map = W1; s.b_row0 = r1(li, (blk ? sl_njt(m) : SL_EJT) + m - 1);
        s.epi = EPI_LN_BWD; s.bias = params + Ly.b(li, blk, m);
        if (blk == 1) s.flags |= EF_COLSUM_ALL;
        if (blk == 0 && ws->lnst_e) { s.flags |= EF_ST_LOAD; s.ln_st = ws->lnst_e + (long long)li * ws->Emax; }
        if (blk == 1 && ws->lnst_n) { s.flags |= EF_ST_LOAD; s.ln_st = ws->lnst_n + (long long)li * ws->Nmax; }
        s.gamma = params + Ly.gamma(li, blk); s.beta = params + Ly.beta(li, blk);
        s.f_in = ws->Gh; s.ld_in = H;
        s.valid_in = blk ? (int)nl : (int)enext;
        if (blk == 0) {
          s.flags |= EF_G16;
          s.g16 = ws->Ge[gc].p; s.g16_lo = ws->Ge[gc].lo; s.ga16 = ws->Ga.p; s.ga16_lo = ws->Ga.lo;
          // G_e rows (< valid_in; none in the top layer, whose G_e is zero)
          if (!ws->split && enext > 0) s.in_map = pr.in_map(ws->Ge[gc].p, enext, H);
        }
        s.scr_z = ws->scrZ[m].p; s.lo_off = ws->scrZ[m].lo;
        if (!ws->split && rows > 0) s.st_map = pr.in_map(ws->scrZ[m].p, rows, H);   // dZ_m = the ACT tile, TMA-stored
        for (int j = m; j >= 1; --j) {
          Step& d = pr.add();
          d.a_src = A_ACT; d.K = H; d.b_map = W1; d.b_row0 = r1(li, (blk ? sl_nj(m) : sl_ej(m)) + j - 1);
          d.epi = EPI_DSILU; d.flags = (blk == 1 ? EF_COLSUM_ALL : 0) | EF_DISCARD; d.scr_s = ws->scrS[j - 1].p; d.scr_z = ws->scrZ[j - 1].p; d.lo_off = ws->scrZ[j - 1].lo;
          if (!ws->split && rows > 0) d.in_map = pr.in_map(ws->scrS[j - 1].p, rows, H);   // S'_{j-1} rows
          if (!ws->split && rows > 0) d.st_map = pr.in_map(ws->scrZ[j - 1].p, rows, H);   // dZ_{j-1} = the ACT tile
          d.vec0 = 3 + (m - j);
        }
      };
      {  // node block backward
        Prog pr(ws);
        set_a(ws, pr, 4, hck, nl, H);
        set_a(ws, pr, 6, ack, nl, H);
        mlp_bwd(pr, 1);
        Step& a = pr.add();   // dh: G_h += dZ0 W0[h rows]^T
        a.a_src = A_ACT; a.K = H; a.b_map = W1; a.b_row0 = r1(li, sl_n1h(m));
        a.epi = EPI_ADD; a.f_in = ws->Gh; a.f_out = ws->Gh; a.ld_in = a.ld_out = H; a.valid_in = (int)nl;
        Step& b = pr.add();   // da: G_a = dZ0 W0[agg rows]^T
        b.a_src = A_ACT; b.K = H; b.b_map = W1; b.b_row0 = r1(li, sl_n1a(m));
        b.epi = EPI_STORE; b.flags = EF_OUT16; b.bf_out = ws->Ga.p; b.bf_lo = ws->Ga.lo; b.ld_out = H; b.col0 = 0;
        run_prog(ws, "chain_node_bwd", pr, (int)nl, nullptr, nullptr, true, st);
        colsum_reduce(ws, 1, li, grad_params, chain_grid(ws, (int)nl), st);
        wgrad(ws, hck, ack, H, H / 128, ws->scrZ[0], H, 0, nl, 2 * H, grad_params, Ly.W(li, 1, 0), st);
        for (int j = 1; j <= m; ++j)
          wgrad(ws, ws->scrA[j - 1], none, H, H / 128, ws->scrZ[j], H, 0, nl, H, grad_params, Ly.W(li, 1, j), st);
      }
      // P for layer l: the forward's checkpoint (no recompute)
      {  // edge block backward
        Prog pr(ws);
        set_a(ws, pr, 4, eck, el, H);
        mlp_bwd(pr, 0);
        Step& a = pr.add();   // G_e^{l-1} = G_e' + dZ0 W0[e rows]^T
        a.a_src = A_ACT; a.K = H; a.b_map = W1; a.b_row0 = r1(li, sl_e1e(m));
        a.epi = EPI_ADD; a.flags = EF_G16; a.g16 = ws->Ge[gc].p; a.g16_lo = ws->Ge[gc].lo;
        if (!ws->split && el > 0) a.in_map = pr.in_map(ws->Ge[gc].p, el, H);   // G_e' rows
        a.g16_out = ws->Ge[gc ^ 1].p;
        run_prog(ws, "chain_edge_bwd", pr, (int)el, dp.src, dp.dst, true, st);
        colsum_reduce(ws, 0, li, grad_params, chain_grid(ws, (int)el), st, /*gamma_only=*/true);
        // bias gradients ride on the weight-gradient GEMMs (all-ones A tile); dbeta = sum_rows G_e';
        // db_0 = sum_rows dZ0 = sum over nodes of D_dst (every active edge has one destination) rides
        // on the node-level dW_d wgrad below when XMGN_DB0_NODE=1 (default: this edge-level wgrad)
        wgrad(ws, eck, none, H, H / 128, ws->scrZ[0], H, 0, el, H, grad_params, Ly.W(li, 0, 0), st,
              ws->db0_node ? -1 : Ly.b(li, 0, 0));
        for (int j = 1; j <= m; ++j)
          wgrad(ws, ws->scrA[j - 1], none, H, H / 128, ws->scrZ[j], H, 0, el, H, grad_params, Ly.W(li, 0, j), st,
                Ly.b(li, 0, j));
        wgrad(ws, none, none, H, 0, ws->Ge[gc], H, 0, el, 0, grad_params, 0, st, Ly.beta(li, 0));
        gc ^= 1;   // G_e^{l-1} now lives in the other buffer
        ws->gc_last = gc;
      }
      // D = [sum over out-edges | sum over in-edges] of dZ0 (adjoint of the P gathers)
      { ProfScope ps("segsum", st);
      launch_segsum(ws->f16, H, dp.off, dp.rev, ws->scrZ[0].p, ws->scrZ[0].lo, ws->D.p, ws->D.lo, (int)nprev, (int)el, st); }
      XMGN_CUDA(cudaGetLastError(), "segsum launch");
      {  // G_h^{l-1} = [rows < n_l] G_h + D [W_s | W_d]^T
        Prog pr(ws);
        set_a(ws, pr, 4, ws->D, nprev, 2 * H);
        Step& s = pr.add();
        s.a_src = A_TMA; s.a_map0 = 4; s.K = 2 * H; s.b_map = W2; s.b_row0 = r2(li, SL2_SD);
        s.epi = EPI_ADD; s.f_in = ws->Gh; s.f_out = ws->Gh; s.ld_in = s.ld_out = H; s.valid_in = (int)nl;
        run_prog(ws, "chain_projbwd", pr, (int)nprev, nullptr, nullptr, false, st);
      }
      // dW_s = h^T D_src, dW_d = h^T D_dst
      wgrad(ws, hck, none, H, H / 128, ws->D, 2 * H, 0, nprev, H, grad_params, Ly.W(li, 0, 0) + (long long)H * H, st);
      wgrad(ws, hck, none, H, H / 128, ws->D, 2 * H, H, nprev, H, grad_params, Ly.W(li, 0, 0) + 2LL * H * H, st,
            ws->db0_node ? Ly.b(li, 0, 0) : -1);
    }
    const int64_t n0 = n_at(P, L, 0), e1 = e_at(P, L, 1);
    if (grad_h0) {
      launch_scale_copy(ws->Gh, n0 * H, ws->d_scale + 1, grad_h0, st);
      if (P.n_local > n0)
        XMGN_CUDA(cudaMemsetAsync(grad_h0 + n0 * H, 0, (P.n_local - n0) * H * sizeof(float), st), "grad_h0");
    }
    if (grad_e0) {
      launch_to_f32(ws->f16, ws->Ge[gc].p, ws->Ge[gc].lo, grad_e0, e1 * H, st, ws->d_scale + 1);
      if (P.e_local > e1)
        XMGN_CUDA(cudaMemsetAsync(grad_e0 + e1 * H, 0, (P.e_local - e1) * H * sizeof(float), st), "grad_e0");
    }
    return XMGN_OK;
  });
}

// ================================================================ the model around the processor (NEXT-1)
// encoders -> processor -> decoder -> owned-row MSE (PAPER.md:161, 197, 219,
// 234).  The encoders' and decoder's H x H layers run as k_chain programs on the tensor cores (the
// encoders' first layer with K = 64: the 24 / 4 inputs zero-padded to one operand box); the
// decoder's 4-wide output layer, the loss and the encoders' first-layer weight gradient are thin
// CUDA-core kernels (io_kernels.cu).
namespace xmgn {

// IO parameter layout (include/xmgn.h; restated independently of oracle/model.py): node encoder,
// edge encoder [W_0 (F x H), b_0, W_j (H x H), b_j for j = 1..m, gamma, beta], decoder [W_0, b_0,
// ..., W_{m-1}, b_{m-1} (H x H), W_m (H x 4), b_m (4)].  blk 0 / 1 / 2 = node enc / edge enc / dec.
struct IoLayout {
  int H, m;
  int fin(int blk) const { return blk == 0 ? IO_F_NODE : IO_F_EDGE; }
  int64_t kin(int blk, int j) const { return j == 0 && blk < 2 ? fin(blk) : H; }
  int64_t nout(int blk, int j) const { return blk == 2 && j == m ? IO_DOUT : H; }
  int64_t lin(int blk, int j) const { return kin(blk, j) * nout(blk, j) + nout(blk, j); }
  int64_t size(int blk) const {
    int64_t o = blk < 2 ? 2 * (int64_t)H : 0;
    for (int j = 0; j <= m; ++j) o += lin(blk, j);
    return o;
  }
  int64_t base(int blk) const { return blk == 0 ? 0 : (blk == 1 ? size(0) : size(0) + size(1)); }
  int64_t W(int blk, int j) const {
    int64_t o = base(blk);
    for (int i = 0; i < j; ++i) o += lin(blk, i);
    return o;
  }
  int64_t b(int blk, int j) const { return W(blk, j) + kin(blk, j) * nout(blk, j); }
  int64_t gamma(int blk) const { return b(blk, m) + H; }
  int64_t beta(int blk) const { return gamma(blk) + H; }
  int64_t count() const { return base(2) + size(2); }
};
// wioH slots of H rows: encoder blk: W_j^T at 2m blk + j - 1, W_j (dgrad) at 2m blk + m + j - 1
// (j = 1..m); decoder: W_j^T at 4m + j, W_j at 5m + j (j = 0..m-1)
static long long io_T(int m, int blk, int j) { return blk < 2 ? 2 * m * blk + j - 1 : 4 * m + j; }
static long long io_D(int m, int blk, int j) { return blk < 2 ? 2 * m * blk + m + j - 1 : 5 * m + j; }

static void ensure_io(xmgn_workspace* ws) {
  if (ws->io_ready) return;
  const int H = ws->H, m = ws->m;
  for (const Part& P : ws->g->parts) ws->Omax = std::max(ws->Omax, P.n_owned);
  const int64_t O = std::max<int64_t>(ws->Omax, 1);
  IoLayout Io{H, m};
  ws->S3 = 6 * m;
  ws->wio64 = bfalloc(ws, (size_t)2 * H * IO_IN_COLS);
  XMGN_CUDA(cudaMemset(ws->wio64.p, 0, (size_t)2 * H * IO_IN_COLS * sizeof(bf16)), "io weights");  // K padding
  ws->wioH = bfalloc(ws, (size_t)ws->S3 * H * H);
  std::vector<PackJob> J;
  auto job = [&](BfBuf& buf, int ld, long long row0, int rows, int cols, long long src, long long sr, long long sc) {
    PackJob j;
    j.dst = buf.p + row0 * ld;
    j.lo_off = 0;
    j.ld = ld; j.rows = rows; j.cols = cols; j.src = src; j.sr = sr; j.sc = sc;
    J.push_back(j);
  };
  for (int blk = 0; blk < 2; ++blk) {
    job(ws->wio64, IO_IN_COLS, (long long)blk * H, H, Io.fin(blk), Io.W(blk, 0), 1, H);
    for (int j = 1; j <= m; ++j) {
      job(ws->wioH, H, io_T(m, blk, j) * H, H, H, Io.W(blk, j), 1, H);
      job(ws->wioH, H, io_D(m, blk, j) * H, H, H, Io.W(blk, j), H, 1);
    }
  }
  for (int j = 0; j < m; ++j) {
    job(ws->wioH, H, io_T(m, 2, j) * H, H, H, Io.W(2, j), 1, H);
    job(ws->wioH, H, io_D(m, 2, j) * H, H, H, Io.W(2, j), H, 1);
  }
  ws->njobs_io = (int)J.size();
  ws->d_jobs_io = (PackJob*)dalloc(ws, J.size() * sizeof(PackJob));
  XMGN_CUDA(cudaMemcpy(ws->d_jobs_io, J.data(), J.size() * sizeof(PackJob), cudaMemcpyHostToDevice), "upload");
  ws->Xn = bfalloc(ws, (size_t)std::max<int64_t>(ws->Nmax, 1) * IO_IN_COLS);
  ws->Xe = bfalloc(ws, (size_t)std::max<int64_t>(ws->Emax, 1) * IO_IN_COLS);
  ws->hL16 = bfalloc(ws, (size_t)O * H);
  ws->zdec = (float*)dalloc(ws, (size_t)O * H * 4);
  ws->sse_part = (double*)dalloc(ws, (size_t)dec_head_warps(O) * sizeof(double));
  if (!ws->infer) {
    ws->dZdec = bfalloc(ws, (size_t)O * H);
    ws->gdec = (float*)dalloc(ws, (size_t)O * H * 4);
    ws->wpart = (float*)dalloc(ws, (size_t)dec_head_warps(O) * (H * IO_DOUT + IO_DOUT) * 4);
    ws->thin_part = (float*)dalloc(ws, (size_t)wgrad_thin_blocks(std::max(ws->Nmax, ws->Emax)) * IO_F_NODE * H * 4);
    ws->d_scale_dec = (float*)dalloc(ws, 2 * sizeof(float));
  }
  ws->io_ready = true;
}

static int weight_map(xmgn_workspace* ws, Prog& pr, const bf16* base, int width, long long rows) {
  if (pr.next_map >= MAX_MAPS) throw Fail{set_error(XMGN_ESTATE, "internal: out of tensor-map slots")};
  const int NB = (ws->H < 256 ? ws->H : 256) / 2;
  pr.p.maps[pr.next_map] = tmap16(base, width, rows, width, 64, NB, ws->f16);
  return pr.next_map++;
}

// encoder blk (0 node, 1 edge) over rows [0, rows) of its 16-bit inputs X: forward (bwd = false:
// y = LN(MLP(X)) -> h^0 / e^0) or recompute + backward (bwd = true: dZ_j into scrZ[j], A_j / S'_j
// into scrA / scrS, column sums for gamma, beta and the biases)
static void enc_prog(xmgn_workspace* ws, int blk, const float* io, long long rows, bool bwd, cudaStream_t st) {
  if (rows <= 0) return;
  const int H = ws->H, m = ws->m;
  IoLayout Io{H, m};
  const BfBuf& X = blk ? ws->Xe : ws->Xn;
  Prog pr(ws);
  pr.p.maps[4] = map_rows(X.p, rows, IO_IN_COLS, 128, ws->f16);
  pr.p.maps[5] = pr.p.maps[4];
  const int w64 = weight_map(ws, pr, ws->wio64.p, IO_IN_COLS, 2LL * H);
  const int wH = weight_map(ws, pr, ws->wioH.p, H, (long long)ws->S3 * H);
  for (int j = 0; j < m; ++j) {
    Step& s = pr.add();
    s.a_src = j ? A_ACT : A_TMA; s.a_map0 = 4; s.K = j ? H : IO_IN_COLS;
    s.b_map = j ? wH : w64; s.b_row0 = (int)(j ? io_T(ws->m, blk, j) * H : (long long)blk * H);
    s.epi = EPI_SILU; s.bias = io + Io.b(blk, j);
    if (bwd) {
      s.flags = EF_STORE_A | EF_STORE_S; s.scr_a = ws->scrA[j].p; s.scr_s = ws->scrS[j].p; s.lo_off = 0;
      s.st_map = pr.in_map(ws->scrA[j].p, rows, H);
    }
  }
  Step& s = pr.add();
  s.a_src = m ? A_ACT : A_TMA; s.a_map0 = 4; s.K = H; s.b_map = wH; s.b_row0 = (int)(io_T(m, blk, m) * H);
  s.bias = io + Io.b(blk, m); s.gamma = io + Io.gamma(blk); s.beta = io + Io.beta(blk);
  if (!bwd) {
    s.epi = EPI_LN_FWD; s.flags = EF_NO_RES | EF_STORE_BF; s.bf_lo = 0;
    if (blk == 0) { s.flags |= EF_STORE_F32; s.f_out = ws->h_buf[0]; s.ld_out = H; s.bf_out = ws->h_ck.p; }
    else {
      s.bf_out = ws->e_ck.p;
      if (ws->e32_mode) { s.flags |= EF_STORE_F32; s.f_out = ws->e32[0]; s.ld_out = H; }
    }
    run_prog(ws, blk ? "enc_edge_fwd" : "enc_node_fwd", pr, (int)rows, nullptr, nullptr, false, st);
    return;
  }
  s.epi = EPI_LN_BWD; s.flags = blk == 0 ? EF_COLSUM_ALL : 0;   // edge rows: dgamma only (tile partials stay small)
  if (blk == 0) { s.f_in = ws->Gh; s.ld_in = H; s.valid_in = (int)rows; }
  else {
    s.flags |= EF_G16 | EF_NO_GA; s.g16 = ws->Ge[ws->gc_last].p; s.g16_lo = 0; s.valid_in = (int)rows;
    s.in_map = pr.in_map(ws->Ge[ws->gc_last].p, rows, H);
  }
  s.scr_z = ws->scrZ[m].p; s.lo_off = 0; s.st_map = pr.in_map(ws->scrZ[m].p, rows, H);
  for (int j = m; j >= 1; --j) {
    Step& d = pr.add();
    d.a_src = A_ACT; d.K = H; d.b_map = wH; d.b_row0 = (int)(io_D(m, blk, j) * H);
    d.epi = EPI_DSILU; d.flags = (blk == 0 ? EF_COLSUM_ALL : 0) | EF_DISCARD; d.vec0 = 3 + (m - j);
    d.scr_s = ws->scrS[j - 1].p; d.scr_z = ws->scrZ[j - 1].p; d.lo_off = 0;
    d.in_map = pr.in_map(ws->scrS[j - 1].p, rows, H);
    if (j > 1) d.st_map = pr.in_map(ws->scrZ[j - 1].p, rows, H);
    else d.flags |= EF_NO_ACT;   // dZ_0 by row stores: the program must not end writing ACT
  }
  run_prog(ws, blk ? "enc_edge_bwd" : "enc_node_bwd", pr, (int)rows, nullptr, nullptr, true, st);
}

}  // namespace xmgn

extern "C" size_t xmgn_io_param_count(const xmgn_model_cfg* c) {
  if (!c || c->hidden <= 0 || c->mlp_hidden_layers < 1) return 0;
  return (size_t)IoLayout{c->hidden, c->mlp_hidden_layers}.count();
}

extern "C" xmgn_status xmgn_model_fwd(xmgn_workspace* ws, int part, const float* params, const float* io_params,
                                      const float* pos, const float* nrm, const float* stats, const float* targets,
                                      int64_t n_global, float* pred, float* loss, void* stream) {
  return guarded("xmgn_model_fwd", [&]() -> xmgn_status {
    if (!ws || !params || !io_params || !pos || !nrm || !stats || !pred)
      return set_error(XMGN_EINVAL, "xmgn_model_fwd: null argument");
    if (part < 0 || part >= (int)ws->g->parts.size())
      return set_error(XMGN_EINVAL, "xmgn_model_fwd: part=%d outside [0,%d)", part, (int)ws->g->parts.size());
    if (ws->split) return set_error(XMGN_EUNSUPPORTED, "xmgn_model_fwd: the FP32 check mode covers the processor only");
    const Part& P = ws->g->parts[part];
    if (targets && (!loss || n_global < P.n_owned || n_global <= 0))
      return set_error(XMGN_EINVAL, "xmgn_model_fwd: targets need loss != NULL and n_global=%lld >= n_owned=%lld > 0",
                       (long long)n_global, (long long)P.n_owned);
    XMGN_CUDA(cudaSetDevice(ws->dev), "xmgn_model_fwd: cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    ensure_io(ws);
    const DPart& dp = ws->dparts[part];
    const int H = ws->H, L = ws->L, m = ws->m;
    IoLayout Io{H, m};
    const float* io = io_params;
    launch_pack(ws->f16, io, ws->d_jobs_io, ws->njobs_io, st);
    const int64_t n0 = n_at(P, L, 0), e1 = e_at(P, L, 1), no = P.n_owned;
    // inputs and encoders -> h^0, e^0
    launch_node_inputs(ws->f16, pos, nrm, stats, n0, ws->Xn.p, st);
    launch_edge_inputs(ws->f16, pos, dp.src, dp.dst, stats, e1, ws->Xe.p, st);
    enc_prog(ws, 0, io, n0, false, st);
    enc_prog(ws, 1, io, e1, false, st);
    // processor (h^L of the owned rows also in 16 bits for the decoder)
    proc_fwd(ws, part, params, ws->h_buf[0], ws->e32_mode ? ws->e32[0] : nullptr, ws->h_buf[L & 1], true, ws->hL16.p,
             st);
    // decoder hidden layers on the tensor cores -> zdec = A_{m-1} W_{m-1} (bias added by the head)
    const bool train = !ws->infer && targets;
    {
      Prog pr(ws);
      set_a(ws, pr, 4, ws->hL16, no, H);
      const int wH = weight_map(ws, pr, ws->wioH.p, H, (long long)ws->S3 * H);
      for (int j = 0; j < m; ++j) {
        Step& s = pr.add();
        s.a_src = j ? A_ACT : A_TMA; s.a_map0 = 4; s.K = H; s.b_map = wH; s.b_row0 = (int)(io_T(m, 2, j) * H);
        if (j < m - 1) {
          s.epi = EPI_SILU; s.bias = io + Io.b(2, j);
          if (train && no > 0) {
            s.flags = EF_STORE_A | EF_STORE_S; s.scr_a = ws->scrA[j].p; s.scr_s = ws->scrS[j].p; s.lo_off = 0;
            s.st_map = pr.in_map(ws->scrA[j].p, no, H);
          }
        } else {
          s.epi = EPI_STORE; s.f_out = ws->zdec; s.ld_out = H; s.col0 = 0;
        }
      }
      run_prog(ws, "dec_fwd", pr, (int)no, nullptr, nullptr, false, st);
    }
    // output layer + owned-row MSE (+ its adjoint for the backward)
    const double nd = (double)IO_DOUT * (double)(n_global > 0 ? n_global : 1);
    const float inv_nd = (float)(1.0 / nd);
    const float S = (float)std::ldexp(1.0, (int)std::floor(std::log2(nd)));   // dy S = O(y - t)
    ws->head_warps = dec_head_warps(std::max<int64_t>(no, 1));
    launch_dec_head(ws->f16, H, ws->zdec, no, io + Io.b(2, m - 1), io + Io.W(2, m), io + Io.b(2, m), targets, inv_nd, S,
                    pred, ws->sse_part, train ? ws->dZdec.p : nullptr, ws->wpart, st);
    if (targets && no > 0) launch_loss_reduce(ws->sse_part, ws->head_warps, inv_nd, loss, st);
    if (train) {
      launch_set_scale(ws->d_scale_dec, S, 1.0f / S, st);
      ws->last_model_fwd = part;
    } else {
      ws->last_model_fwd = -1;
    }
    return XMGN_OK;
  });
}

extern "C" xmgn_status xmgn_model_bwd(xmgn_workspace* ws, int part, const float* params, const float* io_params,
                                      float* grad_params, float* grad_io, void* stream) {
  return guarded("xmgn_model_bwd", [&]() -> xmgn_status {
    if (!ws || !params || !io_params || !grad_params || !grad_io)
      return set_error(XMGN_EINVAL, "xmgn_model_bwd: null argument");
    if (ws->infer) return set_error(XMGN_ESTATE, "xmgn_model_bwd: inference workspace");
    if (part != ws->last_model_fwd || part != ws->last_fwd)
      return set_error(XMGN_ESTATE, "xmgn_model_bwd: part=%d is not the last xmgn_model_fwd with targets (%d)", part,
                       ws->last_model_fwd);
    XMGN_CUDA(cudaSetDevice(ws->dev), "xmgn_model_bwd: cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    const Part& P = ws->g->parts[part];
    const int H = ws->H, L = ws->L, m = ws->m;
    IoLayout Io{H, m};
    const float* io = io_params;
    const int64_t no = P.n_owned;
    const BfBuf none{};
    // decoder backward: S dZ_{m-1} (head) -> dgrad chain -> S dL/dh^L (FP32)
    {
      Prog pr(ws);
      set_a(ws, pr, 4, ws->dZdec, no, H);
      const int wH = weight_map(ws, pr, ws->wioH.p, H, (long long)ws->S3 * H);
      for (int j = m - 1; j >= 0; --j) {
        Step& s = pr.add();
        s.a_src = j == m - 1 ? A_TMA : A_ACT; s.a_map0 = 4; s.K = H; s.b_map = wH; s.b_row0 = (int)(io_D(m, 2, j) * H);
        if (j > 0) {
          s.epi = EPI_DSILU; s.scr_s = ws->scrS[j - 1].p; s.scr_z = ws->scrZ[j - 1].p; s.lo_off = 0;
          if (no > 0) { s.in_map = pr.in_map(ws->scrS[j - 1].p, no, H); s.st_map = pr.in_map(ws->scrZ[j - 1].p, no, H); }
        } else {
          s.epi = EPI_STORE; s.f_out = ws->gdec; s.ld_out = H; s.col0 = 0;
        }
      }
      run_prog(ws, "dec_bwd", pr, (int)no, nullptr, nullptr, true, st);
    }
    auto dZ = [&](int j) { return j == m - 1 ? ws->dZdec : ws->scrZ[j]; };
    const float* inv_dec = ws->d_scale_dec + 1;
    for (int j = m - 1; j >= 1; --j)   // dW_j = A_{j-1}^T dZ_j, db_j (ones tile)
      wgrad(ws, ws->scrA[j - 1], none, H, H / 128, dZ(j), H, 0, no, H, grad_io, Io.W(2, j), st, Io.b(2, j), inv_dec);
    wgrad(ws, ws->hL16, none, H, H / 128, dZ(0), H, 0, no, H, grad_io, Io.W(2, 0), st, Io.b(2, 0), inv_dec);
    if (no > 0) {
      const long long nw = (long long)H * IO_DOUT + IO_DOUT;   // dW_m [H x 4] then db_m [4]
      launch_reduce_part(ws->wpart, ws->head_warps, nw, nw, grad_io + Io.W(2, m), st, nullptr);
      launch_scale_copy(ws->gdec, no * H, inv_dec, ws->gdec, st);
    }
    // processor backward (its own exact loss scale S_p: Gh, G_e come out x S_p)
    xmgn_status r = xmgn_processor_bwd(ws, part, params, ws->gdec, grad_params, nullptr, nullptr, stream);
    if (r != XMGN_OK) return r;
    // encoders: upstream dL/dh^0 (Gh) and dL/de^0 (G_e), both x S_p
    const int64_t n0 = n_at(P, L, 0), e1 = e_at(P, L, 1);
    for (int blk = 0; blk < 2; ++blk) {
      const long long rows = blk ? e1 : n0;
      if (rows <= 0) continue;
      enc_prog(ws, blk, io, rows, true, st);
      ColsumDst d;
      for (int v = 0; v < NV_MAX; ++v) d.off[v] = -1;
      d.off[0] = Io.gamma(blk); d.off[1] = Io.beta(blk); d.off[2] = Io.b(blk, m); d.off[3] = Io.b(blk, m - 1);
      if (m >= 2) d.off[4] = Io.b(blk, m - 2);
      if (blk == 1) for (int v = 1; v < NV_MAX; ++v) d.off[v] = -1;   // edge rows: dgamma only
      reduce_colsums(ws, d, grad_io, st);
      for (int j = 1; j <= m; ++j)   // (edge rows: the biases ride on the weight-gradient GEMMs)
        wgrad(ws, ws->scrA[j - 1], none, H, H / 128, ws->scrZ[j], H, 0, rows, H, grad_io, Io.W(blk, j), st,
              blk == 1 ? Io.b(blk, j) : -1);
      if (blk == 1) {
        wgrad(ws, none, none, H, 0, ws->scrZ[0], H, 0, rows, 0, grad_io, 0, st, Io.b(blk, 0));        // db_0
        wgrad(ws, none, none, H, 0, ws->Ge[ws->gc_last], H, 0, rows, 0, grad_io, 0, st, Io.beta(blk));  // dbeta
      }
      const BfBuf& X = blk ? ws->Xe : ws->Xn;
      const long long nf = (long long)Io.fin(blk) * H;
      launch_wgrad_thin(ws->f16, Io.fin(blk), X.p, ws->scrZ[0].p, rows, H, ws->thin_part, st);
      launch_reduce_part(ws->thin_part, wgrad_thin_blocks(rows), nf, nf, grad_io + Io.W(blk, 0), st, ws->d_scale + 1);
    }
    return XMGN_OK;
  });
}

extern "C" xmgn_status xmgn_scatter_rows(const float* src, const int64_t* idx, int64_t n, int64_t row_elems,
                                         float* dst, void* stream) {
  return guarded("xmgn_scatter_rows", [&]() -> xmgn_status {
    if (n < 0 || row_elems <= 0 || (n && (!src || !idx || !dst)))
      return set_error(XMGN_EINVAL, "xmgn_scatter_rows: bad arguments (n=%lld row_elems=%lld)", (long long)n,
                       (long long)row_elems);
    launch_scatter_rows(src, (const long long*)idx, n, row_elems, dst, (cudaStream_t)stream);
    XMGN_CUDA(cudaGetLastError(), "xmgn_scatter_rows launch");
    return XMGN_OK;
  });
}

extern "C" xmgn_status xmgn_check_finite(const float* dev, size_t n, void* stream) {
  return guarded("xmgn_check_finite", [&]() -> xmgn_status {
    cudaStream_t st = (cudaStream_t)stream;
    int* flag = nullptr;
    XMGN_CUDA(cudaMallocAsync((void**)&flag, 4, st), "xmgn_check_finite");
    XMGN_CUDA(cudaMemsetAsync(flag, 0, 4, st), "xmgn_check_finite");
    launch_nonfinite(dev, (long long)n, flag, st);
    int h = 0;
    XMGN_CUDA(cudaMemcpyAsync(&h, flag, 4, cudaMemcpyDeviceToHost, st), "xmgn_check_finite");
    XMGN_CUDA(cudaStreamSynchronize(st), "xmgn_check_finite");
    cudaFreeAsync(flag, st);
    if (h) return set_error(XMGN_ENONFINITE, "xmgn_check_finite: non-finite value among %zu floats", n);
    return XMGN_OK;
  });
}
