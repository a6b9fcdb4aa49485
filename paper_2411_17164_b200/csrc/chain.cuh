// The fused per-tile GEMM-chain kernel: every MLP of the processor (forward,
// recompute, dgrad) runs through it.
//
// One persistent CTA per SM walks 128-row tiles.  For each tile it executes a
// short PROGRAM of steps; step s computes acc[128, N] = A_s[128, K_s] * B_s^T
// on tcgen05 (BF16 operands, FP32 accumulator in TMEM, N = H <= 512 columns)
// followed by a fused epilogue.  A_s is either
//   * A_TMA: rows of one or two global BF16 tensors (concatenated along K),
//     streamed by TMA through the A ring, or
//   * A_ACT: the previous step's epilogue output kept on chip in the ACT tile
//     (128 x H BF16 in shared memory, 128-byte-swizzled K-major) -- so an
//     MLP's hidden activations never touch HBM.
// B_s (weights, K-major = W^T or W) is streamed by TMA through the B ring.
//
// Warp roles (256 threads): warp 0 = TMA producer, warp 1 = MMA issuer
// (one elected lane), warp 2 = TMEM allocator, warps 4..7 = epilogue (thread
// = tile row = TMEM lane).  The A ring aliases the ACT tile: a program never
// needs both at once (A_TMA steps only start after the previous step's MMAs
// retired, and an epilogue that writes ACT is always followed by an A_ACT step).
//
// FP32 check mode (SPLIT): every operand is carried as hi + lo BF16 and each
// k-step issues hi*hi + lo*hi + hi*lo (FP32-class products, north_star's
// "FP32 check mode").
#pragma once
#include <cuda_bf16.h>
#include <cuda.h>
#include "tc.cuh"

namespace xmgn {

enum : int { A_TMA = 0, A_ACT = 1 };
enum : int {
  EPI_SILU = 0,    // v = acc + b (+ P[src] + P[dst]) -> SiLU -> ACT (+ scratch A, S')
  EPI_LN_FWD = 1,  // v = acc + b -> LN -> out = res + y (fp32 + bf16 [+ ACT])
  EPI_STORE = 2,   // out[:, col0 + c] = acc
  EPI_LN_BWD = 3,  // recompute LN, dY = G (+ Ga[dst]) -> dZ -> ACT + scratch; dgamma, dbeta, db
  EPI_DSILU = 4,   // dZ = acc * S' -> ACT + scratch; db
  EPI_ADD = 5      // out = (r < valid ? in : 0) (+ Ga[dst]) + acc
};
enum : int {
  EF_GATHER_P = 1,     // EPI_SILU: add P[src][c] + P[dst][H + c]
  EF_STORE_A = 2,      // EPI_SILU: scratch A = SiLU(v)
  EF_STORE_S = 4,      // EPI_SILU: scratch S = SiLU'(v)
  EF_WRITE_ACT = 8,    // EPI_LN_FWD: also write the BF16 output into ACT
  EF_GATHER_G = 16,    // EPI_LN_BWD / EPI_ADD: add Ga[dst][c]
  EF_STORE_BF = 32,    // EPI_LN_FWD: write bf16 output (checkpoint)
  EF_RES16 = 64,       // EPI_LN_FWD: residual input is the 16-bit tensor res16 (else fp32 f_in)
  EF_STORE_F32 = 128,  // EPI_LN_FWD: write the fp32 output f_out
  EF_OUT16 = 256,      // EPI_STORE: write 16-bit bf_out (ld_out, col0) instead of fp32 f_out
  EF_COLSUM_ALL = 1024,  // EPI_LN_BWD / EPI_DSILU: also accumulate dbeta / db column sums here
                         // (else only dgamma; the bias sums come from the wgrad GEMMs)
  EF_G16 = 512,        // EPI_LN_BWD / EPI_ADD: the gradient stream is the 16-bit g16 (edge programs):
                       // LN_BWD writes dY = g16 (+ ga16[dst]) back into g16; ADD does g16 += acc
  EF_DISCARD = 2048,   // EPI_DSILU: this is the last read of S' -- drop its L2 lines afterwards
  EF_STORE_Z = 8192,   // EPI_SILU (16-bit modes): round z to 16 bits, store it to scr_z, SiLU the rounded z
  EF_FROM_IN = 16384,  // EPI_SILU (16-bit modes): z is the TMA row input in ACT (a K = 0 step, no MMA)
  EF_NO_RES = 32768,   // EPI_LN_FWD (16-bit modes): y = LN(z), no residual (the encoders, NEXT-1)
  EF_NO_ACT = 65536,   // EPI_DSILU (16-bit modes): dZ leaves by row stores only, ACT untouched (last step)
  EF_NO_GA = 131072,   // EPI_LN_BWD + EF_G16: dY = G rows only (no G_a[dst] term, no write-back)
  EF_OUT_HALF = 262144,  // EPI_STORE + EF_OUT16 (16-bit modes): write FP16 whatever the operand type
                         // (the node pre-projections P are epilogue addends, not MMA operands)
  EF_STORE_LO = 524288,  // EPI_LN_FWD (16-bit modes): also write lo = y - rnd16(y) to lo_out (2 x 16-bit
                         // GEMM operands of the BF16 mode)
  EF_ST_SAVE = 1048576,  // EPI_LN_FWD (16-bit modes): write the row's (mean, rstd) to ln_st[row]
  EF_ST_LOAD = 2097152   // EPI_LN_BWD (16-bit modes): read (mean, rstd) from ln_st[row] (the forward's,
                         // bitwise those the recompute would give) instead of a statistics pass
};

enum : int {
  CTL_WAIT_ACT = 1,      // A_ACT step whose A was just written by the previous epilogue
  CTL_NEED_ACT_FREE = 2  // A_TMA step that must wait until no MMA reads ACT (A ring aliases ACT)
};

struct Step {
  int a_src, a_map0, a_map1, a_ksplit;  // A source; tensor-map slots (hi; lo = slot+1 in SPLIT)
  int ctl;                               // CTL_* (derived on the host from the program)
  int b_map, b_row0, K;                  // weight map slot, first weight row, reduction length
  int epi, flags, col0, vec0;            // epilogue op, flags, output column offset, colsum vector
  int valid_in;                          // rows of f_in that are valid (EPI_LN_BWD / EPI_ADD)
  const float* bias;
  const float* gamma;
  const float* beta;
  const float* f_in;    // residual input / incoming gradient  [rows][ld_in]
  float* f_out;         // fp32 output [rows][ld_out]
  int ld_in, ld_out;
  const float* gather;  // P [N][2H] (EF_GATHER_P) or Ga [N][H] (EF_GATHER_G)
  __nv_bfloat16* bf_out;     // bf16 row output hi [rows][H]; lo at bf_out + bf_lo_off
  __nv_bfloat16* scr_a;      // scratch SiLU(v)
  __nv_bfloat16* scr_s;      // scratch SiLU'(v) (written by EPI_SILU, read by EPI_DSILU)
  __nv_bfloat16* scr_z;      // scratch dZ
  long long lo_off;          // element offset of the lo half of the scratch buffers (SPLIT)
  long long bf_lo;           // element offset of the lo half of bf_out (SPLIT)
  const __nv_bfloat16* res16;  // 16-bit residual rows [rows][H] (EF_RES16); lo at res16 + res16_lo
  long long res16_lo;
  const __nv_bfloat16* gather16;  // 16-bit P [N][2H] (EF_GATHER_P); lo at + gather16_lo
  long long gather16_lo;
  __nv_bfloat16* g16;             // 16-bit gradient stream [rows][H] (EF_G16)
  long long g16_lo;
  __nv_bfloat16* g16_out;         // EPI_ADD + EF_G16 output (same lo offset as g16)
  __nv_bfloat16* lo_out;          // EPI_LN_FWD + EF_STORE_LO: lo rows [rows][H]
  float2* ln_st;                  // EF_ST_SAVE / EF_ST_LOAD: per-row LayerNorm (mean, rstd) [rows]
  const __nv_bfloat16* ga16;      // 16-bit aggregation adjoint G_a [N][H] gathered by dst (EF_G16)
  long long ga16_lo;
  // 16-bit modes: the epilogue's contiguous 16-bit row input (S', G_e, G_e', residual) is
  // bulk-loaded by TMA into the ACT tile once the accumulator is ready (ACT is dead then:
  // the step's MMAs have read it); map slot, -1 = read rows from global instead
  int in_map;
  // EPI_SILU + EF_GATHER_P: the P[src] rows are TMA-gathered (tile::gather4) into ACT at
  // accumulator-ready; map over P with 1-row boxes of 64 columns (-1 = row loads)
  int gsrc_map;
  // outputs equal to the ACT tile this epilogue writes (A_j, dZ_j scratch) leave by TMA
  // bulk stores straight from ACT (map slot, -1 = row stores)
  int st_map;
};

// does the epilogue of step st read or write the ACT tile (outputs, TMA-staged inputs, stores)?
// does the epilogue of step st write the ACT tile (the next step's A operand)?
__host__ __device__ inline bool step_writes_act(const Step& st) {
  return st.epi == EPI_SILU || st.epi == EPI_LN_BWD || (st.epi == EPI_DSILU && !(st.flags & EF_NO_ACT)) ||
         (st.epi == EPI_LN_FWD && (st.flags & EF_WRITE_ACT));
}
__host__ __device__ inline bool step_uses_act(const Step& st) {
  return step_writes_act(st) || st.in_map >= 0 || st.gsrc_map >= 0 || st.st_map >= 0;
}

// epilogue ops a kernel instantiation contains (OPS template mask): the hot programs get kernels
// without the code of ops they never run (smaller instruction footprint)
enum : int {
  OPB_SILU = 1, OPB_LNF16 = 2, OPB_LNF32 = 4, OPB_STORE = 8, OPB_ADD16 = 16, OPB_ADD32 = 32, OPB_LNB16 = 64,
  OPB_LNB32 = 128, OPB_DSILU = 256, OPS_ALL = 511,
  OPS_EDGE_FWD = OPB_SILU | OPB_LNF16,
  OPS_EDGE_BWD = OPB_SILU | OPB_LNB16 | OPB_DSILU | OPB_ADD16
};
__host__ __device__ inline int step_opbit(const Step& st) {
  switch (st.epi) {
    case EPI_SILU: return OPB_SILU;
    case EPI_LN_FWD: return (st.flags & EF_RES16) ? OPB_LNF16 : OPB_LNF32;
    case EPI_STORE: return OPB_STORE;
    case EPI_ADD: return (st.flags & EF_G16) ? OPB_ADD16 : OPB_ADD32;
    case EPI_LN_BWD: return (st.flags & EF_G16) ? OPB_LNB16 : OPB_LNB32;
    case EPI_DSILU: return OPB_DSILU;
    default: return OPS_ALL;
  }
}

constexpr int MAX_STEPS = 8;
constexpr int MAX_MAPS = 24;
constexpr int NV_MAX = 5;  // column-sum vectors per kernel
// Epilogue: EW warps per TMEM lane quadrant, each owning H/EW columns of its 32
// rows (row statistics are exchanged through shared memory).  The 16-bit modes
// use four column groups (16 epilogue warps, latency tolerance); the FP32 check
// mode keeps two (its hi/lo operands need the registers).
#ifndef XMGN_CTRL_REGS
#define XMGN_CTRL_REGS 32   // control warps need < 32; the epilogue gets 112 (no spills), profiles/r02e_ab_ctrl_regs.jsonl
#endif
#ifndef XMGN_EPI_GROUPS
#define XMGN_EPI_GROUPS 4
#endif
// H = 128 (16-bit modes): four CTAs per SM (four pair-tiles in flight per SM pair, so one tile's
// TMA / MMA / epilogue latency chain overlaps the others'), one column group each (all four
// fit: 4 x 128 TMEM columns, 4 x 56 KB smem with a 2-slot B ring).  CFG2 step (1 B200, FP16):
// 1 CTA/SM 42.3 ms, 2 (two groups) 33.6 ms, 3 31.1 ms, 4 30.7 ms (profiles/r03e_ab_ctas128.txt).
#ifndef XMGN_CTAS128
#define XMGN_CTAS128 4
#endif
#ifndef XMGN_EW128
#define XMGN_EW128 1
#endif
#ifndef XMGN_CTRL_REGS_128
#define XMGN_CTRL_REGS_128 24   // H = 128: epilogue 104 instead of 96 (fewer spills), CFG2 -2.5% (profiles/r03p_ab_ctrl24_128.txt)
#endif
template <int H, bool SPLIT>
struct EpiShape {
  static constexpr int MINB = (H == 128 && !SPLIT) ? XMGN_CTAS128 : 1;   // CTAs per SM
  static constexpr int EW = SPLIT ? 2 : (MINB > 1 ? XMGN_EW128 : XMGN_EPI_GROUPS);
  static constexpr int THREADS = 128 + 128 * EW;
  // setmaxnreg split.  The CTA owns exactly THREADS x LAUNCH_REGS registers (the
  // count ptxas derives from __launch_bounds__); setmaxnreg.inc can only take what
  // the control warpgroup released with setmaxnreg.dec, or it blocks forever.
  static constexpr int LAUNCH_REGS = (65536 / (THREADS * MINB)) & ~7;
  static constexpr int CTRL_REGS = MINB > 1 ? XMGN_CTRL_REGS_128 : XMGN_CTRL_REGS;   // control warps after setmaxnreg.dec
  static constexpr int EPI_REGS_FIT = (LAUNCH_REGS + (LAUNCH_REGS - CTRL_REGS) / EW) & ~7;
  static constexpr int EPI_REGS = EPI_REGS_FIT > 224 ? 224 : EPI_REGS_FIT;
  static_assert(128 * CTRL_REGS + 128 * EW * EPI_REGS <= THREADS * LAUNCH_REGS, "register pool");
};

struct ChainParams {
  CUtensorMap maps[MAX_MAPS];
  Step steps[MAX_STEPS];
  int n_steps;
  int M;              // rows
  const int* src;     // [M] source local id of each edge row (edge programs)
  const int* dst;     // [M] destination local id
  float* colsum;      // partial column sums (backward): [slot][CTA tile 2 t + rank][quadrant][H]
  long long cs_vstride;   // elements per slot (= CTA tiles x 4 x H)
  int cs_slot[NV_MAX];    // column-sum vector -> slot (-1: the program never writes it)
  float eps;          // LayerNorm epsilon
  int* tile_counter;  // dynamic tile scheduler: zeroed before the launch (null = static tiles)
  // static parameter table (16-bit modes): when the program's distinct bias / gamma / beta
  // vectors fit the PRM region (n_prm > 0), they are staged in shared memory ONCE per launch
  // (prm_src[i] -> table row i, null = zeros) and step s reads rows prm_slot[s][0..2]; else
  // (n_prm = 0) every step re-stages its three vectors before waiting for its accumulator
  int n_prm;
  const float* prm_src[6];
  signed char prm_slot[MAX_STEPS][3];
};
constexpr int TQ = 2;   // tile-queue slots per cluster (the producer claims at most one tile ahead)

template <int H, bool SPLIT>
struct ChainCfg {
  static constexpr int F = SPLIT ? 2 : 1;
  static constexpr int NB = H < 256 ? H : 256;                 // MMA N (columns per N-half)
  static constexpr int NBH = NB / 2;                           // B rows held by each CTA of the pair
  static constexpr uint32_t ACT_HALF = 128u * H * 2u;          // one BF16 copy of the ACT tile
  static constexpr uint32_t ACT_BYTES = F * ACT_HALF;
  static constexpr uint32_t A_SLOT_HALF = 128u * 64u * 2u;     // 16 KiB
  static constexpr uint32_t A_SLOT = F * A_SLOT_HALF;
  static constexpr int SA = ACT_BYTES / A_SLOT;
  static constexpr uint32_t B_SLOT_HALF = NBH * 128u;
  static constexpr uint32_t B_SLOT = F * B_SLOT_HALF;
  static constexpr uint32_t SMEM_LIMIT =
      EpiShape<H, SPLIT>::MINB > 1 ? 228u * 1024u / EpiShape<H, SPLIT>::MINB - 1024u : 227u * 1024u;
  static constexpr uint32_t PRM_BYTES = 2u * 3u * H * 4u;        // per-step bias/gamma/beta, double-buffered
  static constexpr int SB_FIT = (int)((SMEM_LIMIT - 1536u - 1024u * EpiShape<H, SPLIT>::EW - PRM_BYTES - ACT_BYTES) / B_SLOT);
  static constexpr int SB = SB_FIT > 8 ? 8 : SB_FIT;
  static constexpr uint32_t BAR_OFF = ACT_BYTES + SB * B_SLOT;
  static constexpr uint32_t RED_OFF = BAR_OFF + 512;             // row-reduction exchange [2][EW][128] f32
  static constexpr uint32_t PRM_OFF = RED_OFF + 2 * EpiShape<H, SPLIT>::EW * 128 * 4;
  static constexpr uint32_t SMEM_BYTES = PRM_OFF + PRM_BYTES + 1024;  // + alignment slack
  static constexpr uint32_t TMEM_COLS = H;
  static_assert(SB >= 2, "B ring too small");
  static_assert(SMEM_BYTES <= 232448, "shared memory budget");
  static_assert(EpiShape<H, SPLIT>::MINB * (SMEM_BYTES + 1024u) <= 228u * 1024u,
                "the resident CTAs per SM (MINB) must fit the SM's shared memory");
};

__device__ __forceinline__ float sigmoid_fast(float v) {
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * v));
  return fmaf(0.5f, t, 0.5f);
}
template <bool ACCURATE>
__device__ __forceinline__ float sigmoid_(float v) {
  if constexpr (ACCURATE) return 1.0f / (1.0f + __expf(-v));
  else return sigmoid_fast(v);
}
// SiLU(x) = x*sigmoid(x) = h + h*tanh(h), h = x/2 (one MUFU op on the fast path)
template <bool ACCURATE>
__device__ __forceinline__ float silu_(float x) {
  if constexpr (ACCURATE) {
    return x / (1.0f + __expf(-x));
  } else {
    const float h = 0.5f * x;
    float t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(h));
    return fmaf(h, t, h);
  }
}
// SiLU and SiLU' = s (1 + x (1 - s)), s = sigmoid(x)
template <bool ACCURATE>
__device__ __forceinline__ void silu_and_grad(float x, float& y, float& dy) {
  const float sg = sigmoid_<ACCURATE>(x);
  y = x * sg;
  dy = sg * fmaf(x, 1.0f - sg, 1.0f);
}

// Store 32 consecutive values (cols c0..c0+31) of row `row` into a swizzled
// K-major BF16 tile [H/64 blocks][128 rows][64]; lo = residual in SPLIT mode.
template <int H, bool SPLIT, bool F16>
__device__ __forceinline__ void store_tile32(uint8_t* tile, uint32_t lo_off, int row, int c0, const float* v) {
  uint8_t* blk = tile + (c0 >> 6) * (128 * 128);
  const int q0 = (c0 & 63) >> 3;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t hi[4], lo[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) split2<F16, SPLIT>(v[q * 8 + 2 * i], v[q * 8 + 2 * i + 1], hi[i], lo[i]);
    const uint32_t a = smem_u32(blk) + sw128_off(row, q0 + q);
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(hi[0]), "r"(hi[1]), "r"(hi[2]), "r"(hi[3])
                 : "memory");
    if constexpr (SPLIT)
      asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a + lo_off), "r"(lo[0]), "r"(lo[1]), "r"(lo[2]),
                   "r"(lo[3])
                   : "memory");
  }
}

// 32 values -> global BF16 row segment (hi, and lo at +lo_off elements in SPLIT).
template <bool SPLIT, bool F16>
__device__ __forceinline__ void store_bf32(__nv_bfloat16* p, long long lo_off, const float* v) {
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    uint32_t hi[8], lo[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) split2<F16, SPLIT>(v[q * 16 + 2 * i], v[q * 16 + 2 * i + 1], hi[i], lo[i]);
    stg256(p + 16 * q, hi);
    if constexpr (SPLIT) stg256(p + lo_off + 16 * q, lo);
  }
}
template <bool SPLIT, bool F16>
__device__ __forceinline__ void load_bf32(const __nv_bfloat16* p, long long lo_off, float* v) {
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    uint32_t u[8];
    ldg256(p + 16 * q, u);
    unpack8<F16>(make_uint4(u[0], u[1], u[2], u[3]), v + q * 16);
    unpack8<F16>(make_uint4(u[4], u[5], u[6], u[7]), v + q * 16 + 8);
    if constexpr (SPLIT) {
      uint32_t w[8];
      ldg256(p + lo_off + 16 * q, w);
      float t[16];
      unpack8<false>(make_uint4(w[0], w[1], w[2], w[3]), t);
      unpack8<false>(make_uint4(w[4], w[5], w[6], w[7]), t + 8);
#pragma unroll
      for (int i = 0; i < 16; ++i) v[q * 16 + i] += t[i];
    }
  }
}
// v <- value as stored by store_bf32 (16-bit hi [+ lo]) -- keeps passes bitwise consistent
template <bool SPLIT, bool F16>
__device__ __forceinline__ void load_bf32_regs(float* v) {
#pragma unroll
  for (int i = 0; i < 32; i += 2) {
    uint32_t hi, lo;
    split2<F16, SPLIT>(v[i], v[i + 1], hi, lo);
    float t[8];
    uint4 u = make_uint4(hi, 0, 0, 0);
    unpack8<F16 && !SPLIT>(u, t);
    float a = t[0], b = t[1];
    if constexpr (SPLIT) {
      uint4 w = make_uint4(lo, 0, 0, 0);
      unpack8<false>(w, t);
      a += t[0];
      b += t[1];
    }
    v[i] = a;
    v[i + 1] = b;
  }
}
__device__ __forceinline__ void load_f32x32(const float* p, float* v) {
#pragma unroll
  for (int q = 0; q < 4; ++q) ldg256(p + 8 * q, reinterpret_cast<uint32_t*>(v + 8 * q));
}
__device__ __forceinline__ void load_f32x32_ro(const float* p, float* v) {
#pragma unroll
  for (int q = 0; q < 4; ++q) ldg256_nc(p + 8 * q, reinterpret_cast<uint32_t*>(v + 8 * q));
}
__device__ __forceinline__ void store_f32x32(float* p, const float* v) {
#pragma unroll
  for (int q = 0; q < 4; ++q) stg256(p + 8 * q, reinterpret_cast<const uint32_t*>(v + 8 * q));
}

// Column sums of 32 values over the 32 lanes of a warp: afterwards lane l
// holds the sum of column l (transpose-reduce, 31 shuffles, fixed order).
__device__ __forceinline__ float warp_colsum32(float* v) {
  const int lane = lane_id();
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
#pragma unroll
    for (int i = 0; i < w; ++i) {
      bool up = (lane & w) != 0;
      float send = up ? v[i] : v[i + w];
      float keep = up ? v[i + w] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, w);
    }
  }
  return v[0];
}

// SiLU(x) = h + h tanh(h), h = x/2.  FP16 mode: tanh on packed f16x2 (one MUFU op per
// two elements; its ~2^-11 error is at the FP16 rounding of the stored activation).
template <bool F16>
__device__ __forceinline__ void tanh2(float a, float b, float& ta, float& tb) {
  if constexpr (F16) {
    uint32_t hh = pack16<true>(a, b), tt;
    asm("tanh.approx.f16x2 %0, %1;" : "=r"(tt) : "r"(hh));
    const __half2 t2 = *reinterpret_cast<const __half2*>(&tt);
    ta = __low2float(t2);
    tb = __high2float(t2);
  } else {
    asm("tanh.approx.f32 %0, %1;" : "=f"(ta) : "f"(a));
    asm("tanh.approx.f32 %0, %1;" : "=f"(tb) : "f"(b));
  }
}
// dY of the LayerNorm backward: incoming gradient rows (< valid_in) plus the
// aggregation adjoint G_a[dst] for edge programs.
__device__ __forceinline__ void load_dy(const Step& st, bool has_g, bool valid, int r, int dst, int c0, float* dy) {
  if (has_g) load_f32x32(st.f_in + (size_t)r * st.ld_in + c0, dy);
  else {
#pragma unroll
    for (int i = 0; i < 32; ++i) dy[i] = 0.f;
  }
  if (valid && (st.flags & EF_GATHER_G)) {
    float ga[32];
    load_f32x32(st.gather + (size_t)dst * st.ld_in + c0, ga);
#pragma unroll
    for (int i = 0; i < 32; ++i) dy[i] += ga[i];
  }
}

}  // namespace xmgn
#include "epi16.cuh"
namespace xmgn {

// Tile schedule of the chain kernel (see k_chain): static, or dynamic through a queue the
// leader's producer fills from an atomic counter.
// The dynamic queue is compiled out by default: on B200 its extra live state made the epilogue
// spill (edge bwd +5%, profiles/r02d_ab_tiles.jsonl), more than the end-of-kernel tail it removes.
// Build with -DXMGN_STATIC_TILES=0 and run with XMGN_DYN=1 to use it.
#ifndef XMGN_STATIC_TILES
#define XMGN_STATIC_TILES 1
#endif
// The OPS-specialised edge-forward kernel compiles the dynamic queue in even so (it does not
// spill there); it runs dynamic when the launch passes a tile counter (XMGN_DYN_FWD=0: static).
#ifndef XMGN_DYN_EDGE_FWD
#define XMGN_DYN_EDGE_FWD 1
#endif
// H = 128 (16-bit modes): every chain program on the dynamic queue (balances the 4-CTA/SM grid).
// Off: the queue's state makes the 96-register H = 128 epilogue spill more -- CFG2 +5%
// (profiles/r03r_ab_dyn128_rejected.txt)
#ifndef XMGN_DYN128
#define XMGN_DYN128 0
#endif
template <bool DYN>
struct TileSched {   // everything but the queue base is re-derived at each call (few live registers)
  const ChainParams* p;
  uint64_t* base;        // tq_full[TQ], tq_empty[TQ], then int q[TQ]
  __device__ __forceinline__ int at(int i) const {   // every role
    if (!DYN || !p->tile_counter) {
      const int t = (int)cluster_id_x() + i * (int)n_clusters_x();
      return t < (p->M + 255) / 256 ? t : -1;
    }
    mbar_wait_cluster(&base[i % TQ], (i / TQ) & 1);
    return *reinterpret_cast<volatile int*>(reinterpret_cast<int*>(base + 2 * TQ) + i % TQ);
  }
  __device__ __forceinline__ int claim(int i) const {   // the leader's producer (one lane)
    if (!DYN || !p->tile_counter) return at(i);
    const int slot = i % TQ;
    if (i >= TQ) mbar_wait_cluster(&base[TQ + slot], ((i / TQ) - 1) & 1);
    const int t = atomicAdd(p->tile_counter, 1);
    const int tile = t < (p->M + 255) / 256 ? t : -1;
    int* q = reinterpret_cast<int*>(base + 2 * TQ) + slot;
    *q = tile;
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(mapa_shared(smem_u32(q), 1)), "r"(tile) : "memory");
    mbar_arrive(&base[slot]);
    mbar_arrive_cluster(mapa_shared(smem_u32(&base[slot]), 1));
    return tile;
  }
  __device__ __forceinline__ void done(int i) const {   // hand-off warps, lane 0, after the tile
    if (!DYN || !p->tile_counter) return;
    if (cluster_ctarank() == 0) mbar_arrive(&base[TQ + i % TQ]);
    else mbar_arrive_cluster(mapa_shared(smem_u32(&base[TQ + i % TQ]), 0));
  }
};

// Z1: backward programs whose first edge step reloads the forward's z_1 checkpoint
// (a separate instantiation so the regular backward kernel's register allocation is
// unaffected)
//
// PIPE (H = 512, 16-bit modes, every step K = H): the step's accumulator is produced as two
// N-halves (TMEM columns [0,256) and [256,512)) in the order nh = 0 over all K, then nh = 1
// with K-half 0 before K-half 1.  The epilogue warps of column groups 0-1 own N-half 0 and
// those of groups 2-3 own N-half 1, each half with its own barriers, so
//   * half 0's epilogue runs while the MMA computes N-half 1 (it may rewrite ACT half 0 as
//     soon as N-half 1's K-half-0 MMAs have read it: act_rd[0]);
//   * the next step's N-half-0 MMAs over K-half 0 start as soon as half 0's epilogue has
//     written ACT half 0 and drained TMEM half 0, while half 1's epilogue still runs.
// An A_TMA step stages its A chunk kc straight into ACT block kc (all K = H resident, read by
// both N-halves).  LayerNorm steps still need both halves' row statistics (row_sum).
template <int H, bool SPLIT, bool BWD, bool F16, bool Z1 = false, bool PIPE = false, int OPS = OPS_ALL>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(EpiShape<H, SPLIT>::THREADS, EpiShape<H, SPLIT>::MINB)
    k_chain(const __grid_constant__ ChainParams p) {
  static_assert(!PIPE || (H == 512 && !SPLIT && !Z1 && EpiShape<H, SPLIT>::EW == 4), "PIPE: H = 512, 16-bit, 4 groups");
  using C = ChainCfg<H, SPLIT>;
  constexpr int NB = C::NB;
  constexpr int NH = H / NB;           // N-halves per step
  using ES = EpiShape<H, SPLIT>;
  constexpr int EW = ES::EW;
  constexpr int HC = H / EW;           // columns per epilogue warp
  constexpr int NC = HC / 32;          // 32-column chunks per epilogue warp
  constexpr int NEPI = 128 * EW;       // epilogue threads
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* act = smem;                       // ACT tile (and A ring)
  uint8_t* bring = smem + C::ACT_BYTES;      // B ring
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* a_full = bars;                   // [SA]
  uint64_t* a_empty = a_full + C::SA;        // [SA]
  uint64_t* b_full = a_empty + C::SA;        // [SB]
  uint64_t* b_empty = b_full + C::SB;        // [SB]
  uint64_t* acc_full = b_empty + C::SB;      // MMA -> epilogue
  uint64_t* acc_empty = acc_full + 1;        // epilogue -> MMA (TMEM drained)
  uint64_t* act_full = acc_empty + 1;        // epilogue -> MMA (ACT written)
  uint64_t* act_free = act_full + 1;         // MMA -> producer (no MMA reads ACT any more)
  uint64_t* mma_idle = act_free + 1;         // MMA -> itself (all issued MMAs retired)
  uint64_t* in_full = mma_idle + 1;          // [H/64] epilogue input boxes landed in ACT
  // PIPE: per N-half barriers
  uint64_t* acc_full2 = in_full + H / 64;    // [2] MMA -> epilogue half h (TMEM half h ready)
  uint64_t* acc_empty2 = acc_full2 + 2;      // [2] epilogue half h (both CTAs) -> MMA (TMEM half drained)
  uint64_t* act_full2 = acc_empty2 + 2;      // [2] epilogue half h (both CTAs) -> MMA (ACT half written)
  uint64_t* act_rd = act_full2 + 2;          // [2] MMA -> epilogue / producer: ACT half no longer read
  uint64_t* act_idle = act_rd + 2;           // [2] local epilogue half -> local producer: ACT half idle
  uint64_t* tq_full = act_idle + 2;          // [TQ] tile-queue entry written (both CTAs)
  uint64_t* tq_empty = tq_full + TQ;         // [TQ] leader: entry consumed by every role of both CTAs
  int* tq = reinterpret_cast<int*>(tq_empty + TQ);   // [TQ] queued pair-tile ids (-1: no more)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tq + TQ);
  static_assert(8 * (2 * C::SA + 2 * C::SB + 5 + H / 64 + 10 + 2 * TQ) + 4 * TQ + 4 <= 512,
                "barrier region overflows RED_OFF");
  float* red = reinterpret_cast<float*>(smem + C::RED_OFF);
  float* prm_base = reinterpret_cast<float*>(smem + C::PRM_OFF);

  const int w = warp_id();
  const uint32_t rank = cluster_ctarank();
  const int cid = (int)cluster_id_x(), ncl = (int)n_clusters_x();
  const int n_tiles = (p.M + 255) / 256;     // pair tiles of 256 rows (128 per CTA)
  constexpr int EPI_ARRIVALS = 1;   // warp 3, once per CTA and step
  if (threadIdx.x == 0) {
    for (int i = 0; i < C::SA; ++i) { mbar_init(&a_full[i], 1); mbar_init(&a_empty[i], 1); }
    for (int i = 0; i < C::SB; ++i) { mbar_init(&b_full[i], 1); mbar_init(&b_empty[i], 1); }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 2 * EPI_ARRIVALS);   // epilogue arrivals of both CTAs
    mbar_init(act_full, 2 * EPI_ARRIVALS);
    mbar_init(act_free, 1);
    mbar_init(mma_idle, 1);
    for (int i = 0; i < H / 64; ++i) mbar_init(&in_full[i], 1);
    for (int i = 0; i < TQ; ++i) {
      mbar_init(&tq_full[i], 1);
      mbar_init(&tq_empty[i], 2 * (PIPE ? 2 : 1));   // the hand-off warps of both CTAs
    }
    if constexpr (PIPE) {
      for (int h = 0; h < 2; ++h) {
        mbar_init(&acc_full2[h], 1);
        mbar_init(&acc_empty2[h], 2);
        mbar_init(&act_full2[h], 2);
        mbar_init(&act_rd[h], 1);
        mbar_init(&act_idle[h], 1);
      }
    }
    fence_barrier_init();
  }
  if (w == 0 && lane_id() == 0)
    for (int i = 0; i < MAX_MAPS; ++i) tma_prefetch(&p.maps[i]);
  if (!SPLIT && p.n_prm > 0)
    for (int i = threadIdx.x; i < p.n_prm * H; i += blockDim.x) {
      const float* v = p.prm_src[i / H];
      prm_base[i] = v ? __ldg(v + (i % H)) : 0.f;
    }
  if (w == 2) tmem_alloc_cg2(tslot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  // ---- tile schedule.  Static: cluster cid takes tiles cid, cid + ncl, ...  Dynamic (tile_counter):
  // the leader's producer claims pair tiles with an atomic counter and queues them in both
  // CTAs' tq[] (TQ slots); every role reads the same sequence.  A slot is reused only after the
  // hand-off warps of both CTAs finished its tile, by which time every role has read it.
  constexpr bool DYN = !XMGN_STATIC_TILES || (XMGN_DYN_EDGE_FWD && PIPE && !BWD && OPS == OPS_EDGE_FWD) ||
                       (XMGN_DYN128 && H == 128 && !SPLIT);
  const TileSched<DYN> ts{&p, tq_full};

  // register split (setmaxnreg, per warpgroup): control warps 0-3 need few registers,
  // the epilogue warpgroups get the rest
  if (w < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(ES::CTRL_REGS) : "memory");
  if (w == 0 && PIPE) {
    // ============================ PIPE TMA producer: B in MMA order (nh outer, k inner);
    // A_TMA chunk kc -> ACT block kc once the previous step is done with that ACT half
    if (elect_one()) {
      int bi = 0, g = 0;
      int nid0 = 0, nid1 = 0;   // act_idle waits per ACT half (each matched by one hand-off arrive)
      for (int it = 0, tile; (tile = rank == 0 ? ts.claim(it) : ts.at(it)) >= 0; ++it) {
        const int row0 = tile * 256 + (int)rank * 128;
        for (int s = 0; s < p.n_steps; ++s, ++g) {
          const Step& st = p.steps[s];
          const bool tma_a = st.a_src == A_TMA;
          constexpr int NK = H / 64;
          for (int nh = 0; nh < 2; ++nh) {
            for (int kc = 0; kc < NK; ++kc) {
              if (tma_a && nh == 0) {
                const int kh = kc / (NK / 2);
                if (g > 0 && kc % (NK / 2) == 0) {
                  mbar_wait(&act_rd[kh], (g - 1) & 1);     // the previous step's MMAs read it
                  // the previous step's epilogue used it (skipped when that epilogue never touches
                  // ACT: the A loads then overlap it)
                  const Step& pv = p.steps[s > 0 ? s - 1 : p.n_steps - 1];
                  if (step_uses_act(pv)) {
                    if (kh == 0) mbar_wait(&act_idle[0], nid0++ & 1);
                    else mbar_wait(&act_idle[1], nid1++ & 1);
                  }
                }
                if (rank == 0) mbar_expect_tx(&a_full[kc], 2 * C::A_SLOT);
                const uint32_t fb = mapa_shared(smem_u32(&a_full[kc]), 0);
                const int k = kc * 64;
                // A = [map a_map0 | map a_map0 + d | map a_map0 + 2d | ...], a_ksplit columns each
                const int seg = st.a_map1 >= 0 ? k / st.a_ksplit : 0;
                const int mi = st.a_map0 + seg * (st.a_map1 - st.a_map0), kk = k - seg * st.a_ksplit;
                tma_load_2d_cg2(act + kc * C::A_SLOT, &p.maps[mi], fb, kk, row0);
              }
              const int slot = bi % C::SB;
              if (bi >= C::SB) mbar_wait(&b_empty[slot], ((bi / C::SB) - 1) & 1);
              if (rank == 0) mbar_expect_tx(&b_full[slot], 2 * C::B_SLOT);
              const uint32_t fb = mapa_shared(smem_u32(&b_full[slot]), 0);
              const int brow = st.b_row0 + nh * NB + (int)rank * C::NBH;
              tma_load_2d_cg2(bring + slot * C::B_SLOT, &p.maps[st.b_map], fb, kc * 64, brow);
              ++bi;
            }
          }
        }
      }
    }
  } else if (w == 1 && PIPE) {
    // ============================ PIPE MMA issuer (leader CTA): per step nh = 0 (all K), then
    // nh = 1 (K-half 0, commit act_rd[0], K-half 1, commit act_rd[1])
    if (rank == 0) {
      constexpr uint32_t idesc = idesc_pair(NB, F16);
      constexpr int NK = H / 64;
      int bi = 0, g = 0, na = 0;
      for (int it = 0, tile; (tile = ts.at(it)) >= 0; ++it) {
        for (int s = 0; s < p.n_steps; ++s, ++g) {
          const Step& st = p.steps[s];
          const bool tma_a = st.a_src == A_TMA;
          for (int nh = 0; nh < 2; ++nh) {
            if (g > 0) mbar_wait(&acc_empty2[nh], (g - 1) & 1);   // TMEM half nh drained
            for (int kc = 0; kc < NK; ++kc) {
              const int kh = kc / (NK / 2);
              if (nh == 0) {
                if (tma_a) mbar_wait(&a_full[kc], na & 1);
                else if (g > 0 && kc % (NK / 2) == 0) mbar_wait(&act_full2[kh], (g - 1) & 1);
              }
              tc_fence_after();
              const uint32_t a_base = smem_u32(act + kc * (128 * 128));
              const int bslot = bi % C::SB;
              mbar_wait(&b_full[bslot], (bi / C::SB) & 1);
              tc_fence_after();
              const uint32_t b_base = smem_u32(bring + bslot * C::B_SLOT);
              if (elect_one()) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  uint64_t ad = sdesc_sw128(a_base + k * 32, 16, 1024);
                  uint64_t bd = sdesc_sw128(b_base + k * 32, 16, 1024);
                  mma_f16_cg2(tmem + nh * NB, ad, bd, idesc, (kc | k) != 0);
                }
                mma_commit_cg2_mc(&b_empty[bslot], 3);
                if (nh == 1 && kc % (NK / 2) == NK / 2 - 1) mma_commit_cg2_mc(&act_rd[kh], 3);
              }
              __syncwarp();
              ++bi;
            }
            if (elect_one()) mma_commit_cg2_mc(&acc_full2[nh], 3);
            __syncwarp();
          }
          if (tma_a) ++na;
        }
      }
    }
  } else if (w == 0) {
    // ============================ TMA producer (both CTAs: own A rows, own half of B)
    if (elect_one()) {
      int ai = 0, bi = 0, g = 0, naf = 0;  // A / B ring fills, global step, act_free phases
      for (int it = 0, tile; (tile = rank == 0 ? ts.claim(it) : ts.at(it)) >= 0; ++it) {
        const int row0 = tile * 256 + (int)rank * 128;
        for (int s = 0; s < p.n_steps; ++s, ++g) {
          const Step& st = p.steps[s];
          const bool tma_a = st.a_src == A_TMA;
          if (tma_a && g > 0 && (st.ctl & CTL_NEED_ACT_FREE)) { mbar_wait(act_free, naf & 1); ++naf; }
          for (int kc = 0; kc < st.K / 64; ++kc) {
            if (tma_a) {
              const int slot = ai % C::SA;
              if (ai >= C::SA) mbar_wait(&a_empty[slot], ((ai / C::SA) - 1) & 1);
              if (rank == 0) mbar_expect_tx(&a_full[slot], 2 * C::A_SLOT);
              const uint32_t fb = mapa_shared(smem_u32(&a_full[slot]), 0);
              uint8_t* dstp = act + slot * C::A_SLOT;
              const int k = kc * 64;
              const int seg = st.a_map1 >= 0 ? k / st.a_ksplit : 0;   // A segments, see the PIPE producer
              const int mi = st.a_map0 + seg * (st.a_map1 - st.a_map0), kk = k - seg * st.a_ksplit;
              tma_load_2d_cg2(dstp, &p.maps[mi], fb, kk, row0);
              if constexpr (SPLIT) tma_load_2d_cg2(dstp + C::A_SLOT_HALF, &p.maps[mi + 1], fb, kk, row0);
              ++ai;
            }
            for (int nh = 0; nh < NH; ++nh) {
              const int slot = bi % C::SB;
              if (bi >= C::SB) mbar_wait(&b_empty[slot], ((bi / C::SB) - 1) & 1);
              if (rank == 0) mbar_expect_tx(&b_full[slot], 2 * C::B_SLOT);
              const uint32_t fb = mapa_shared(smem_u32(&b_full[slot]), 0);
              uint8_t* dstp = bring + slot * C::B_SLOT;
              const int brow = st.b_row0 + nh * NB + (int)rank * C::NBH;
              tma_load_2d_cg2(dstp, &p.maps[st.b_map], fb, kc * 64, brow);
              if constexpr (SPLIT) tma_load_2d_cg2(dstp + C::B_SLOT_HALF, &p.maps[st.b_map + 1], fb, kc * 64, brow);
              ++bi;
            }
          }
        }
      }
    }
  } else if (w == 1) {
    // ============================ MMA issuer (leader CTA only; M = 256 pair MMAs)
    if (rank == 0) {
      constexpr uint32_t idesc = idesc_pair(NB, F16);
      const uint32_t act_free_peer = mapa_shared(smem_u32(act_free), 1);
      int ai = 0, bi = 0, g = 0, nact = 0, nidle = 0;
      for (int it = 0, tile; (tile = ts.at(it)) >= 0; ++it) {
        for (int s = 0; s < p.n_steps; ++s, ++g) {
          const Step& st = p.steps[s];
          const bool tma_a = st.a_src == A_TMA;
          // the previous epilogue must be done (it may still read its input out of ACT)
          // before ACT can become A-ring space again
          if (g > 0) mbar_wait(acc_empty, (g - 1) & 1);
          if (tma_a && g > 0 && (st.ctl & CTL_NEED_ACT_FREE)) {
            // let every issued MMA (the ones reading ACT) retire, then hand both
            // CTAs' ACT tiles to their producers as A-ring space.
            if (elect_one()) mma_commit_cg2_mc(mma_idle, 1);
            __syncwarp();
            mbar_wait(mma_idle, nidle & 1);
            ++nidle;
            if (elect_one()) { mbar_arrive(act_free); mbar_arrive_cluster(act_free_peer); }
            __syncwarp();
          }
          if (st.ctl & CTL_WAIT_ACT) { mbar_wait(act_full, nact & 1); ++nact; }
          tc_fence_after();
          for (int kc = 0; kc < st.K / 64; ++kc) {
            int aslot = 0;
            uint32_t a_base;
            if (tma_a) {
              aslot = ai % C::SA;
              mbar_wait(&a_full[aslot], (ai / C::SA) & 1);
              a_base = smem_u32(act + aslot * C::A_SLOT);
            } else {
              a_base = smem_u32(act + kc * (128 * 128));
            }
            const uint32_t a_lo = tma_a ? C::A_SLOT_HALF : C::ACT_HALF;
            for (int nh = 0; nh < NH; ++nh) {
              const int bslot = bi % C::SB;
              mbar_wait(&b_full[bslot], (bi / C::SB) & 1);
              tc_fence_after();
              const uint32_t b_base = smem_u32(bring + bslot * C::B_SLOT);
              if (elect_one()) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  const uint32_t acc = (kc | k) != 0;
                  const uint32_t d = tmem + nh * NB;
                  uint64_t ad = sdesc_sw128(a_base + k * 32, 16, 1024);
                  uint64_t bd = sdesc_sw128(b_base + k * 32, 16, 1024);
                  mma_f16_cg2(d, ad, bd, idesc, acc);
                  if constexpr (SPLIT) {
                    uint64_t adl = sdesc_sw128(a_base + a_lo + k * 32, 16, 1024);
                    uint64_t bdl = sdesc_sw128(b_base + C::B_SLOT_HALF + k * 32, 16, 1024);
                    mma_f16_cg2(d, adl, bd, idesc, 1);
                    mma_f16_cg2(d, ad, bdl, idesc, 1);
                  }
                }
                mma_commit_cg2_mc(&b_empty[bslot], 3);
              }
              __syncwarp();
              ++bi;
            }
            if (tma_a) {
              if (elect_one()) mma_commit_cg2_mc(&a_empty[aslot], 3);
              __syncwarp();
              ++ai;
            }
          }
          if (elect_one()) mma_commit_cg2_mc(acc_full, 3);
          __syncwarp();
        }
      }
    }
  } else if (PIPE && (w == 3 || w == 2)) {
    // ============================ PIPE step hand-off of N-half h (warp 3: h = 0, warp 2: h = 1,
    // idle after the TMEM allocation): joins that half's end-of-step barrier, then arrives on
    // the leader's acc_empty2[h] / act_full2[h] and on the local act_idle[h]
    const int h = w == 3 ? 0 : 1;
    const uint32_t ae_l = mapa_shared(smem_u32(&acc_empty2[h]), 0);
    const uint32_t af_l = mapa_shared(smem_u32(&act_full2[h]), 0);
    for (int it = 0, tile; (tile = ts.at(it)) >= 0; ++it) {
      for (int s = 0; s < p.n_steps; ++s) {
        named_bar(7 + h, 256 + 32);
        if (lane_id() == 0) {
          // act_idle only when the producer will wait for it (the next step stages its A by TMA
          // into ACT and this step used ACT): every phase is waited on, and it is arrived first so
          // it has completed by the time the MMA sees this step's acc_empty
          if (p.steps[s + 1 < p.n_steps ? s + 1 : 0].a_src == A_TMA && step_uses_act(p.steps[s]))
            mbar_arrive(&act_idle[h]);
          if (rank == 0) {
            mbar_arrive(&acc_empty2[h]);
            mbar_arrive(&act_full2[h]);
          } else {
            mbar_arrive_cluster(ae_l);
            mbar_arrive_cluster(af_l);
          }
        }
        __syncwarp();
      }
      if (lane_id() == 0) ts.done(it);
      __syncwarp();
    }
  } else if (w == 3) {
    // ============================ step hand-off: joins the epilogue's end-of-step barrier and
    // arrives on the leader's acc_empty / act_full.  A release at cluster scope waits for
    // the arriving thread's own outstanding global stores (MEMBAR.GPU); this warp has none,
    // the epilogue warps (which store) would stall the hand-off by ~2 us per step.
    const uint32_t acc_empty_l = mapa_shared(smem_u32(acc_empty), 0);
    const uint32_t act_full_l = mapa_shared(smem_u32(act_full), 0);
    int g = 0;
    for (int it = 0, tile; (tile = ts.at(it)) >= 0; ++it) {
      for (int s = 0; s < p.n_steps; ++s, ++g) {
        const Step& st = p.steps[s];
        const bool wa = step_writes_act(st);
        named_bar(8, NEPI + 32);
        if (lane_id() == 0) {
          if (rank == 0) {          // the leader's own barriers: CTA-scope release suffices
            mbar_arrive(acc_empty);
            if (wa) mbar_arrive(act_full);
          } else {
            mbar_arrive_cluster(acc_empty_l);
            if (wa) mbar_arrive_cluster(act_full_l);
          }
        }
        __syncwarp();
      }
      if (lane_id() == 0) ts.done(it);
      __syncwarp();
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(ES::EPI_REGS) : "memory");
    // ============================ epilogue: thread = tile row (TMEM lane) x HC columns
    const int q = w & 3;                 // TMEM lane quadrant
    const int eg = (w - 4) >> 2;         // column group
    const int lane = lane_id();
    const int trow = q * 32 + lane;
    const int cb = eg * HC;              // first column of this thread
    const int hh = PIPE ? (eg >> 1) : 0; // PIPE: the N-half this warp's columns belong to
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16) + cb;
    // full-row sum of a per-thread partial, identical bits in every group
    auto row_sum = [&](float x) -> float {
      if constexpr (EW == 1) {
        return x;
      } else {
        red[eg * 128 + trow] = x;
        named_bar(1 + q, 32 * EW);
        float t = red[trow];
#pragma unroll
        for (int j = 1; j < EW; ++j) t += red[j * 128 + trow];
        named_bar(1 + q, 32 * EW);
        return t;
      }
    };
    // two row sums in one exchange (the same per-value order as two row_sum calls: same bits)
    auto row_sum2 = [&](float& a, float& b) {
      if constexpr (EW > 1) {
        red[eg * 128 + trow] = a;
        red[(EW + eg) * 128 + trow] = b;
        named_bar(1 + q, 32 * EW);
        float ta = red[trow], tb = red[EW * 128 + trow];
#pragma unroll
        for (int j = 1; j < EW; ++j) {
          ta += red[j * 128 + trow];
          tb += red[(EW + j) * 128 + trow];
        }
        named_bar(1 + q, 32 * EW);
        a = ta;
        b = tb;
      }
    };
    // per-(CTA tile, quadrant) column-sum partials in global memory: lane l of this warp owns
    // column c0 + l of every chunk; each entry is written exactly once per launch (by the one
    // warp that runs that tile and quadrant), so the partials do not depend on the CTA <-> tile
    // assignment and k_reduce_colsum sums them in a fixed order.
    float* colsum_base = nullptr;
    auto colsum_add = [&](int vec, int c0, float* vals) {
      const float cs = warp_colsum32(vals);
      colsum_base[(size_t)p.cs_slot[vec] * p.cs_vstride + c0 + lane] = cs;
    };
    int g = 0, nin = 0;   // nin: steps whose input came through in_full (its phase)
    const uint64_t pol_last = policy_evict_last();
    // TMA stores of ACT boxes: with HC >= 64 each column group stores its own boxes
    // (barrier 9 + eg over its 4 warps, issuer = lane 0 of its quadrant-0 warp); with
    // narrower groups all epilogue warps share barrier 9 and thread 128 issues.
    constexpr bool GROUP_STORES = HC >= 64;
    const int sbar = GROUP_STORES ? 9 + eg : 9;
    constexpr int SBAR_THREADS = GROUP_STORES ? 128 : NEPI;
    const bool issuer = GROUP_STORES ? (q == 0 && lane == 0) : (threadIdx.x == 128);
    bool st_pending = false;   // TMA stores out of ACT may still be reading it
    for (int it = 0, tile; (tile = ts.at(it)) >= 0; ++it) {
      const int r = tile * 256 + (int)rank * 128 + trow;
      const bool valid = r < p.M;
      const int rr = valid ? r : 0;
      const int src = p.src ? p.src[rr] : 0;
      const int dst = p.dst ? p.dst[rr] : 0;
      colsum_base = p.colsum ? p.colsum + ((size_t)(2 * tile + (int)rank) * 4 + q) * H : nullptr;
      for (int s = 0; s < p.n_steps; ++s, ++g) {
        const Step& st = p.steps[s];
        float* prm = prm_base + (g & 1) * 3 * H;
        bool wrote_act = false;
        if constexpr (SPLIT) {
        mbar_wait(acc_full, g & 1);
        tc_fence_after();
        float v[32], pb[32];
        if (st.epi == EPI_SILU && !(st.flags & (EF_GATHER_P | EF_STORE_S | EF_STORE_A))) {
          // plain SiLU epilogue, software-pipelined one chunk ahead (TMEM + bias)
          uint32_t ta[32];
          float bn[32];
          tmem_ld32_async(tl, ta);
          load_f32x32_ro(st.bias + cb, bn);
#pragma unroll 1
          for (int cc = 0; cc < NC; ++cc) {
            const int c0 = cb + cc * 32;
            tmem_wait32(ta);
            float x[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) x[i] = __uint_as_float(ta[i]) + bn[i];
            if (cc + 1 < NC) {
              tmem_ld32_async(tl + (cc + 1) * 32, ta);
              load_f32x32_ro(st.bias + c0 + 32, bn);
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) x[i] = silu_<SPLIT>(x[i]);
            store_tile32<H, SPLIT, F16>(act, C::ACT_HALF, trow, c0, x);
          }
          wrote_act = true;
        } else if (st.epi == EPI_SILU) {
#pragma unroll 1
          for (int cc = 0; cc < NC; ++cc) {
            const int c0 = cb + cc * 32;
            tmem_ld32(tl + cc * 32, v);
            load_f32x32_ro(st.bias + c0, pb);
            if (st.flags & EF_GATHER_P) {
              float g1[32];
              load_bf32<SPLIT, F16>(st.gather16 + (size_t)src * 2 * H + c0, st.gather16_lo, g1);
#pragma unroll
              for (int i = 0; i < 32; ++i) pb[i] += g1[i];
              load_bf32<SPLIT, F16>(st.gather16 + (size_t)dst * 2 * H + H + c0, st.gather16_lo, g1);
#pragma unroll
              for (int i = 0; i < 32; ++i) pb[i] += g1[i];
            }
            float sv[32];
            if (st.flags & EF_STORE_S) {
              float dv[32];
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const float x = v[i] + pb[i];
                silu_and_grad<SPLIT>(x, sv[i], dv[i]);
              }
              if (valid) store_bf32<SPLIT, F16>(st.scr_s + (size_t)r * H + c0, st.lo_off, dv);
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i) sv[i] = silu_<SPLIT>(v[i] + pb[i]);
            }
            store_tile32<H, SPLIT, F16>(act, C::ACT_HALF, trow, c0, sv);
            if (valid && (st.flags & EF_STORE_A)) store_bf32<SPLIT, F16>(st.scr_a + (size_t)r * H + c0, st.lo_off, sv);
          }
          wrote_act = true;
        } else if (st.epi == EPI_LN_FWD || st.epi == EPI_LN_BWD) {
          // z = acc + b; mean and variance over the H columns of this row in one TMEM pass
          // (shifted partial moments per thread + exact group combination, as ln_stats16)
          float sum = 0.f, sq = 0.f, kz = 0.f;
#pragma unroll 1
          for (int cc = 0; cc < NC; ++cc) {
            tmem_ld32(tl + cc * 32, v);
            load_f32x32_ro(st.bias + cb + cc * 32, pb);
            if (cc == 0) kz = v[0] + pb[0];
#pragma unroll
            for (int i = 0; i < 32; ++i) { const float z = v[i] + pb[i] - kz; sum += z; sq = fmaf(z, z, sq); }
          }
          const float mg = kz + sum * (1.0f / HC);
          const float m2 = fmaxf(sq - sum * sum * (1.0f / HC), 0.f);
          const float mean = row_sum(mg) * (1.0f / EW);
          const float dmg = mg - mean;
          const float var = row_sum(fmaf((float)HC * dmg, dmg, m2)) * (1.0f / H);
          const float rstd = rsqrtf(var + p.eps);
          if (st.epi == EPI_LN_FWD) {
#pragma unroll 1
            for (int cc = 0; cc < NC; ++cc) {
              const int c0 = cb + cc * 32;
              tmem_ld32(tl + cc * 32, v);
              float res[32], gm[32], bt[32];
              load_f32x32_ro(st.bias + c0, pb);
              load_f32x32_ro(st.gamma + c0, gm);
              load_f32x32_ro(st.beta + c0, bt);
              if (valid && (st.flags & EF_RES16)) load_bf32<SPLIT, F16>(st.res16 + (size_t)r * H + c0, st.res16_lo, res);
              else if (valid) load_f32x32(st.f_in + (size_t)r * st.ld_in + c0, res);
              else {
#pragma unroll
                for (int i = 0; i < 32; ++i) res[i] = 0.f;
              }
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                float xh = (v[i] + pb[i] - mean) * rstd;
                v[i] = res[i] + fmaf(gm[i], xh, bt[i]);
              }
              if (valid) {
                if (st.flags & EF_STORE_F32) store_f32x32(st.f_out + (size_t)r * st.ld_out + c0, v);
                if (st.flags & EF_STORE_BF) store_bf32<SPLIT, F16>(st.bf_out + (size_t)r * H + c0, st.bf_lo, v);
              }
              if (st.flags & EF_WRITE_ACT) store_tile32<H, SPLIT, F16>(act, C::ACT_HALF, trow, c0, v);
            }
            wrote_act = (st.flags & EF_WRITE_ACT) != 0;
          } else if constexpr (BWD) {
            // LayerNorm backward: dx^ = dY*gamma; dz = rstd (dx^ - mean(dx^) - x^ mean(dx^ x^))
            const bool has_g = valid && r < st.valid_in;
            float s1 = 0.f, s2 = 0.f;
#pragma unroll 1
            for (int cc = 0; cc < NC; ++cc) {
              const int c0 = cb + cc * 32;
              tmem_ld32(tl + cc * 32, v);
              float dy[32], gm[32];
              load_f32x32_ro(st.bias + c0, pb);
              load_f32x32_ro(st.gamma + c0, gm);
              if (st.flags & EF_G16) {
                // dY = G_e (rows < valid_in) + G_a[dst]; written back as G_e' for pass B and dX
                float ga[32];
                if (has_g) load_bf32<SPLIT, F16>(st.g16 + (size_t)r * H + c0, st.g16_lo, dy);
                else {
#pragma unroll
                  for (int i = 0; i < 32; ++i) dy[i] = 0.f;
                }
                if (valid) {
                  load_bf32<SPLIT, F16>(st.ga16 + (size_t)dst * H + c0, st.ga16_lo, ga);
#pragma unroll
                  for (int i = 0; i < 32; ++i) dy[i] += ga[i];
                  store_bf32<SPLIT, F16>(st.g16 + (size_t)r * H + c0, st.g16_lo, dy);
                  // use the stored (rounded) value so pass B and this pass agree
                  load_bf32_regs<SPLIT, F16>(dy);
                }
              } else {
                load_dy(st, has_g, valid, r, dst, c0, dy);
              }
              float t1[32], t2[32];
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                float xh = (v[i] + pb[i] - mean) * rstd;
                float dxh = dy[i] * gm[i];
                s1 += dxh;
                s2 += dxh * xh;
                t1[i] = valid ? dy[i] * xh : 0.f;
                t2[i] = valid ? dy[i] : 0.f;
              }
              colsum_add(0, c0, t1);                               // dgamma
              if (st.flags & EF_COLSUM_ALL) colsum_add(1, c0, t2);  // dbeta
            }
            s1 = row_sum(s1) * (1.0f / H);
            s2 = row_sum(s2) * (1.0f / H);
#pragma unroll 1
            for (int cc = 0; cc < NC; ++cc) {
              const int c0 = cb + cc * 32;
              tmem_ld32(tl + cc * 32, v);
              float dy[32], gm[32];
              load_f32x32_ro(st.bias + c0, pb);
              load_f32x32_ro(st.gamma + c0, gm);
              if (st.flags & EF_G16) {
                if (valid) load_bf32<SPLIT, F16>(st.g16 + (size_t)r * H + c0, st.g16_lo, dy);
                else {
#pragma unroll
                  for (int i = 0; i < 32; ++i) dy[i] = 0.f;
                }
              } else {
                load_dy(st, has_g, valid, r, dst, c0, dy);
              }
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                float xh = (v[i] + pb[i] - mean) * rstd;
                float dxh = dy[i] * gm[i];
                v[i] = valid ? rstd * (dxh - s1 - xh * s2) : 0.f;
              }
              store_tile32<H, SPLIT, F16>(act, C::ACT_HALF, trow, c0, v);
              if (valid) store_bf32<SPLIT, F16>(st.scr_z + (size_t)r * H + c0, st.lo_off, v);
              if (st.flags & EF_COLSUM_ALL) colsum_add(2, c0, v);   // db_{m+1}
            }
            wrote_act = true;
          }
        } else if (st.epi == EPI_DSILU) {
          if constexpr (BWD) {
            // S' rows are software-pipelined one chunk ahead (raw 16-bit registers)
            uint32_t cur[16], nxt[16];
            const __nv_bfloat16* srow = st.scr_s + (size_t)r * H + cb;
            if (!SPLIT && valid) { ldg256(srow, cur); ldg256(srow + 16, cur + 8); }
#pragma unroll 1
            for (int cc = 0; cc < NC; ++cc) {
              const int c0 = cb + cc * 32;
              if (!SPLIT && valid && cc + 1 < NC) {
                ldg256(srow + (cc + 1) * 32, nxt);
                ldg256(srow + (cc + 1) * 32 + 16, nxt + 8);
              }
              tmem_ld32(tl + cc * 32, v);
              float sd[32];
              if constexpr (SPLIT) {
                if (valid) load_bf32<SPLIT, F16>(st.scr_s + (size_t)r * H + c0, st.lo_off, sd);
              } else {
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4)
                  unpack8<F16>(make_uint4(cur[4 * q4], cur[4 * q4 + 1], cur[4 * q4 + 2], cur[4 * q4 + 3]), sd + 8 * q4);
#pragma unroll
                for (int i = 0; i < 16; ++i) cur[i] = nxt[i];
              }
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = valid ? v[i] * sd[i] : 0.f;
              store_tile32<H, SPLIT, F16>(act, C::ACT_HALF, trow, c0, v);
              if (valid) store_bf32<SPLIT, F16>(st.scr_z + (size_t)r * H + c0, st.lo_off, v);
              if (st.flags & EF_COLSUM_ALL) colsum_add(st.vec0, c0, v);  // db_m (3) / db_{m-1} (4)
            }
            wrote_act = true;
          }
        } else if (st.epi == EPI_STORE) {
#pragma unroll 1
          for (int cc = 0; cc < NC; ++cc) {
            tmem_ld32(tl + cc * 32, v);
            if (valid) {
              if (st.flags & EF_OUT16)
                store_bf32<SPLIT, F16>(st.bf_out + (size_t)r * st.ld_out + st.col0 + cb + cc * 32, st.bf_lo, v);
              else
                store_f32x32(st.f_out + (size_t)r * st.ld_out + st.col0 + cb + cc * 32, v);
            }
          }
        } else if (st.epi == EPI_ADD && (st.flags & EF_G16)) {
#pragma unroll 1
          for (int cc = 0; cc < NC; ++cc) {
            const int c0 = cb + cc * 32;
            tmem_ld32(tl + cc * 32, v);
            if (valid) {
              float t[32];
              load_bf32<SPLIT, F16>(st.g16 + (size_t)r * H + c0, st.g16_lo, t);
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] += t[i];
              store_bf32<SPLIT, F16>(st.g16_out + (size_t)r * H + c0, st.g16_lo, v);
            }
          }
        } else if (st.epi == EPI_ADD) {
          const bool has_in = valid && r < st.valid_in;
#pragma unroll 1
          for (int cc = 0; cc < NC; ++cc) {
            const int c0 = cb + cc * 32;
            tmem_ld32(tl + cc * 32, v);
            if (valid) {
              float t[32];
              if (has_in) {
                load_f32x32(st.f_in + (size_t)r * st.ld_in + c0, t);
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] += t[i];
              }
              if (st.flags & EF_GATHER_G) {
                load_f32x32(st.gather + (size_t)dst * H + c0, t);
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] += t[i];
              }
              store_f32x32(st.f_out + (size_t)r * st.ld_out + c0, v);
            }
          }
        }
        } else {
          // ---------------- 16-bit operand modes: ops of epi16.cuh.  Each op issues its
          // MMA-independent row loads, then calls wait(): stage this step's bias / gamma /
          // beta in shared memory, wait for the accumulator.
          auto wait = [&]() {
            if constexpr (PIPE) {
              // this N-half's 256 threads stage its 256 columns of bias / gamma / beta
              if (p.n_prm == 0) {
                const int et = threadIdx.x - 128 - 256 * hh;
                for (int i = et; i < 3 * 256; i += 256) {
                  const int vec = i >> 8, c = 256 * hh + (i & 255);
                  const float* srcv = vec == 0 ? st.bias : (vec == 1 ? st.gamma : st.beta);
                  prm[vec * H + c] = srcv ? __ldg(srcv + c) : 0.f;
                }
                named_bar(5 + hh, 256);
              }
              mbar_wait(&acc_full2[hh], g & 1);
              tc_fence_after();
              mbar_wait(&act_rd[hh], g & 1);   // this step's MMAs no longer read ACT half hh
              if (st_pending) {   // the previous step's TMA stores out of ACT half hh have read it
                if (issuer) bulk_wait_read0();
                named_bar(14 + hh, 256);
                st_pending = false;
              }
            } else {
            if (p.n_prm == 0) {
              const int et = threadIdx.x - 128;
              for (int i = et; i < 3 * H; i += NEPI) {
                const float* srcv = i < H ? st.bias : (i < 2 * H ? st.gamma : st.beta);
                prm[i] = srcv ? __ldg(srcv + (i % H)) : 0.f;
              }
              named_bar(7, NEPI);
            }
            mbar_wait(acc_full, g & 1);
            tc_fence_after();
            if (st_pending) {   // the previous step's stores must have read ACT before anything rewrites it
              if (issuer) bulk_wait_read0();
              named_bar(13, NEPI);
              st_pending = false;
            }
            }
            if (st.gsrc_map >= 0) {
              // P[src] rows of this warp's 32 tile rows, this column group's boxes: lane j
              // issues box first + j for each group of 4 rows (src ids by shuffle)
              if (threadIdx.x == (PIPE ? 128 + 256 * hh : 128))
                for (int b = (PIPE ? 4 * hh : 0); b < (PIPE ? 4 * hh + 4 : H / 64); ++b)
                  mbar_expect_tx(&in_full[b], 128 * 128);
              const bool owner = (cb & 63) == 0;                  // narrow groups share a box
              const int first = cb >> 6, nb = HC >= 64 ? HC / 64 : 1;
#pragma unroll 1
              for (int gi = 0; gi < 8; ++gi) {
                const int s0 = __shfl_sync(0xffffffffu, src, 4 * gi), s1 = __shfl_sync(0xffffffffu, src, 4 * gi + 1);
                const int s2 = __shfl_sync(0xffffffffu, src, 4 * gi + 2), s3 = __shfl_sync(0xffffffffu, src, 4 * gi + 3);
                if (owner && lane < nb) {
                  const int b = first + lane;
                  tma_gather4(act + b * (128 * 128) + (q * 32 + 4 * gi) * 128, &p.maps[st.gsrc_map], &in_full[b], b * 64,
                              s0, s1, s2, s3);
                }
              }
            }
            if (st.in_map >= 0 && threadIdx.x == (PIPE ? 128 + 256 * hh : 128)) {
              // the step's MMAs have read ACT: bulk-load the row input over it, in the order
              // the column groups consume the 64-column boxes (PIPE: this half's groups only)
              const int row0 = tile * 256 + (int)rank * 128;
              constexpr int BPG = HC >= 64 ? HC / 64 : 1;          // boxes per column group
              constexpr int NG = HC >= 64 ? EW : H / 64;
              const int g0 = PIPE ? 2 * hh : 0, g1 = PIPE ? 2 * hh + 2 : NG;
              for (int j = 0; j < BPG; ++j)
                for (int gi = g0; gi < g1; ++gi) {
                  const int b = gi * BPG + j;
                  mbar_expect_tx(&in_full[b], 128 * 128);
                  tma_load_2d(act + b * (128 * 128), &p.maps[st.in_map], &in_full[b], b * 64, row0);
                }
            }
          };
          Epi e;
          e.act = act; e.tl = tl; e.trow = trow; e.cb = cb; e.r = r; e.src = src; e.dst = dst; e.valid = valid;
          if (p.n_prm > 0) {
            e.sb = prm_base + p.prm_slot[s][0] * H + cb;
            e.sg = prm_base + p.prm_slot[s][1] * H + cb;
            e.sbt = prm_base + p.prm_slot[s][2] * H + cb;
          } else {
            e.sb = prm + cb; e.sg = prm + H + cb; e.sbt = prm + 2 * H + cb;
          } e.colsum = colsum_base; e.cs_vstride = (size_t)p.cs_vstride; e.cs_slot = p.cs_slot; e.eps = p.eps;
          e.in_full = in_full; e.in_par = nin & 1; e.pol_last = pol_last;
          constexpr int NC16 = HC / 16;
          const int op = st.epi;
          const int ob = step_opbit(st);
          if (ob == OPB_SILU) {
            if constexpr ((OPS & OPB_SILU) != 0) {
              if constexpr (Z1) {
                if (st.flags & EF_FROM_IN) op_silu_in<H, NC16, F16>(e, st, wait);
                else op_silu<H, NC16, F16, false>(e, st, wait);
              } else {
                op_silu<H, NC16, F16, !BWD>(e, st, wait);
              }
              wrote_act = true;
            }
          } else if (ob == OPB_LNF16) {
            if constexpr ((OPS & OPB_LNF16) != 0) {
              op_ln_fwd<H, NC16, F16, false>(e, st, wait, row_sum);
              wrote_act = (st.flags & EF_WRITE_ACT) != 0;
            }
          } else if (ob == OPB_LNF32) {
            if constexpr ((OPS & OPB_LNF32) != 0) {
              op_ln_fwd<H, NC16, F16, true>(e, st, wait, row_sum);
              wrote_act = (st.flags & EF_WRITE_ACT) != 0;
            }
          } else if (ob == OPB_STORE) {
            if constexpr ((OPS & OPB_STORE) != 0) op_store<H, NC16, F16>(e, st, wait);
          } else if (ob == OPB_ADD16) {
            if constexpr ((OPS & OPB_ADD16) != 0) op_add16<H, NC16, F16>(e, st, wait);
          } else if (ob == OPB_ADD32) {
            if constexpr ((OPS & OPB_ADD32) != 0) op_add32<H, NC16, F16>(e, st, wait);
          } else if constexpr (BWD) {
            if (ob == OPB_LNB16) {
              if constexpr ((OPS & OPB_LNB16) != 0) {
                op_ln_bwd16<H, NC16, F16>(e, st, wait, row_sum, row_sum2);
                wrote_act = true;
              }
            } else if (ob == OPB_LNB32) {
              if constexpr ((OPS & OPB_LNB32) != 0) {
                op_ln_bwd32<H, NC16, F16>(e, st, wait, row_sum, row_sum2);
                wrote_act = true;
              }
            } else if (ob == OPB_DSILU) {
              if constexpr ((OPS & OPB_DSILU) != 0) {
                op_dsilu<H, NC16, F16>(e, st, wait);
                wrote_act = !(st.flags & EF_NO_ACT);
              }
            }
          }
          if constexpr (OPS != OPS_ALL) {
            if ((ob & OPS) == 0) __trap();   // the host picked a kernel without this op
          }
          // rows this step wrote with ordinary stores that a later step of this kernel reads
          // back by TMA (S' -> the dSiLU steps, G_e' -> the dX step): order the generic-proxy
          // writes before those async-proxy reads (the end-of-step barrier carries the order
          // to the TMA-issuing thread)
          if ((op == EPI_SILU && (st.flags & EF_STORE_S)) || (op == EPI_LN_BWD && (st.flags & EF_G16)))
            fence_proxy_async_global();
          if (st.in_map >= 0 || st.gsrc_map >= 0) ++nin;
          if (st.st_map >= 0) {
            // this thread-set's ACT boxes -> global rows [row0, row0 + 128) by TMA
            fence_proxy_async_smem();
            named_bar(sbar, SBAR_THREADS);
            if (issuer) {
              const int row0 = tile * 256 + (int)rank * 128;
              const int b0 = GROUP_STORES ? cb / 64 : 0, nb = GROUP_STORES ? HC / 64 : H / 64;
              for (int b = b0; b < b0 + nb; ++b) tma_store_2d(&p.maps[st.st_map], act + b * (128 * 128), b * 64, row0);
              bulk_commit();
            }
            st_pending = true;
          }
          // the next step refills the A ring (aliases ACT): drain before arriving.  PIPE: only
          // when the next step loads its A into ACT by TMA; otherwise the next step's MMA may read
          // ACT while the stores still read it, and its epilogue drains them before rewriting ACT
          {
            const Step& nx = p.steps[s + 1 < p.n_steps ? s + 1 : 0];
            if (st_pending && (PIPE ? nx.a_src == A_TMA : (nx.a_src == A_TMA && (nx.ctl & CTL_NEED_ACT_FREE)))) {
              if (issuer) bulk_wait_read0();
              st_pending = false;
            }
          }
        }
        tc_fence_before();
        if (wrote_act) fence_proxy_async_smem();
        __syncwarp();
        // warp 3 (PIPE: warp 3 / 2 for N-half 0 / 1) arrives on the leader's barriers once
        // every epilogue warp (of the half) is here
        if constexpr (PIPE) named_bar(7 + hh, 256 + 32);
        else named_bar(8, NEPI + 32);
      }
    }
    if (issuer) bulk_wait0();   // no TMA store may outlive the CTA's shared memory
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (w == 2) tmem_dealloc_cg2(tmem, C::TMEM_COLS);
}

}  // namespace xmgn
