// Epilogue ops of the chain kernel for the 16-bit operand modes (BF16 / FP16).
//
// Thread = one tile row (TMEM lane) x HC = H / EW columns, walked in
// 16-column chunks.  Latency tolerance comes from three places:
//   * the op's global row inputs for chunks 0 and 1 are requested BEFORE the
//     thread waits for the step's accumulator (they do not depend on the MMA),
//   * every 16-bit input stream is double-buffered two chunks ahead (the chunk
//     loop is unrolled by two so the buffers alternate without register moves),
//   * the TMEM accumulator is read one chunk ahead (tcgen05.ld is asynchronous
//     until tcgen05.wait::ld).
// Column sums (dgamma, dbeta, db) use a fixed-order 16-column transpose-reduce
// over the warp followed by a fixed-order read-modify-write of per-(CTA,
// quadrant) global partials, so results are bitwise run-to-run stable.
#pragma once
#ifndef XMGN_ROWSUM2
#define XMGN_ROWSUM2 1
#endif
#include "tc.cuh"


namespace xmgn {

// ---- 16-column helpers
__device__ __forceinline__ void tmem_ld16_async(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait16(uint32_t* r) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15])::"memory");
}
// 16 x 16-bit = 32 bytes = one 256-bit access
__device__ __forceinline__ void ld16(const void* p, uint32_t* r) { ldg256(p, r); }
template <bool F16>
__device__ __forceinline__ void cvt16(const uint32_t* r, float* v) {
  unpack8<F16>(make_uint4(r[0], r[1], r[2], r[3]), v);
  unpack8<F16>(make_uint4(r[4], r[5], r[6], r[7]), v + 8);
}
// v += the 16 16-bit values in r (unpacked word by word: no temporary array)
template <bool F16>
__device__ __forceinline__ void add16(const uint32_t* r, float* v) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float t[2];
    unpack2<F16>(r[i], t);
    v[2 * i] += t[0];
    v[2 * i + 1] += t[1];
  }
}
template <bool F16>
__device__ __forceinline__ void pack16x16(const float* v, uint32_t* h) {
#pragma unroll
  for (int i = 0; i < 8; ++i) h[i] = pack16<F16>(v[2 * i], v[2 * i + 1]);
}
template <bool F16>
__device__ __forceinline__ void st16(void* p, const float* v) {
  uint32_t h[8];
  pack16x16<F16>(v, h);
  stg256(p, h);
}
// v <- the value it has once stored in 16 bits (keeps passes bitwise consistent)
template <bool F16>
__device__ __forceinline__ void round16(float* v) {
  uint32_t h[8];
  pack16x16<F16>(v, h);
  cvt16<F16>(h, v);
}
// 16 FP32 values = 64 bytes = two 256-bit accesses
__device__ __forceinline__ void ld32x16(const float* p, uint32_t* r) {
  ldg256(p, r);
  ldg256(p + 8, r + 8);
}
__device__ __forceinline__ void st32x16(float* p, const float* v) {
  stg256(p, reinterpret_cast<const uint32_t*>(v));
  stg256(p + 8, reinterpret_cast<const uint32_t*>(v + 8));
}
__device__ __forceinline__ void lds16(const float* p, float* v) {  // broadcast read of 16 floats
  const uint32_t a = smem_u32(p);
#pragma unroll
  for (int q = 0; q < 4; ++q)
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v[4 * q]), "=f"(v[4 * q + 1]), "=f"(v[4 * q + 2]), "=f"(v[4 * q + 3])
                 : "r"(a + 16 * q));
}
// 16 values of row `row`, columns c0..c0+15 (c0 % 16 == 0), into / out of the
// 128-byte-swizzled K-major 16-bit tile [H/64 blocks][128 rows][64].
__device__ __forceinline__ uint32_t tile_addr16(uint8_t* tile, int row, int c0) {
  return smem_u32(tile + (c0 >> 6) * (128 * 128)) + sw128_off(row, (c0 & 63) >> 3);
}
template <bool F16>
__device__ __forceinline__ void sts_tile16(uint8_t* tile, int row, int c0, const float* v) {
  uint32_t h[8];
  pack16x16<F16>(v, h);
  const uint32_t a0 = tile_addr16(tile, row, c0), a1 = tile_addr16(tile, row, c0 + 8);
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a0), "r"(h[0]), "r"(h[1]), "r"(h[2]), "r"(h[3])
               : "memory");
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a1), "r"(h[4]), "r"(h[5]), "r"(h[6]), "r"(h[7])
               : "memory");
}
// the same from already packed 16-bit words
__device__ __forceinline__ void sts_tile16_packed(uint8_t* tile, int row, int c0, const uint32_t* h) {
  const uint32_t a0 = tile_addr16(tile, row, c0), a1 = tile_addr16(tile, row, c0 + 8);
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a0), "r"(h[0]), "r"(h[1]), "r"(h[2]), "r"(h[3])
               : "memory");
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a1), "r"(h[4]), "r"(h[5]), "r"(h[6]), "r"(h[7])
               : "memory");
}
template <bool F16>
__device__ __forceinline__ void lds_tile16(uint8_t* tile, int row, int c0, float* v) {
  uint32_t h[8];
  const uint32_t a0 = tile_addr16(tile, row, c0), a1 = tile_addr16(tile, row, c0 + 8);
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(h[0]), "=r"(h[1]), "=r"(h[2]), "=r"(h[3]) : "r"(a0)
               : "memory");
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(h[4]), "=r"(h[5]), "=r"(h[6]), "=r"(h[7]) : "r"(a1)
               : "memory");
  cvt16<F16>(h, v);
}
// SiLU(x) = h + h tanh(h), h = x/2 (FP16 mode: tanh on packed f16x2)
template <bool F16>
__device__ __forceinline__ void silu16(float* x) {
#pragma unroll
  for (int i = 0; i < 16; i += 2) {
    const float ha = 0.5f * x[i], hb = 0.5f * x[i + 1];
    float ta, tb;
    tanh2<F16>(ha, hb, ta, tb);
    x[i] = fmaf(ha, ta, ha);
    x[i + 1] = fmaf(hb, tb, hb);
  }
}
// x <- SiLU(x), d <- SiLU'(x) = s + x s (1 - s), s = (1 + tanh(x/2)) / 2
template <bool F16>
__device__ __forceinline__ void silu_grad16(float* x, float* d) {
#pragma unroll
  for (int i = 0; i < 16; i += 2) {
    const float ha = 0.5f * x[i], hb = 0.5f * x[i + 1];
    float ta, tb;
    tanh2<F16>(ha, hb, ta, tb);
    const float sa = fmaf(0.5f, ta, 0.5f), sb = fmaf(0.5f, tb, 0.5f);
    d[i] = fmaf(x[i] * sa, 1.0f - sa, sa);
    d[i + 1] = fmaf(x[i + 1] * sb, 1.0f - sb, sb);
    x[i] = fmaf(ha, ta, ha);
    x[i + 1] = fmaf(hb, tb, hb);
  }
}
// Column sums of 16 values over the 32 lanes of a warp (fixed order): afterwards
// lanes l and l + 16 both hold the sum of column (l & 15).
__device__ __forceinline__ float warp_colsum16(float* v) {
  const int lane = lane_id();
#pragma unroll
  for (int w = 8; w >= 1; w >>= 1) {
#pragma unroll
    for (int i = 0; i < w; ++i) {
      const bool up = (lane & w) != 0;
      const float send = up ? v[i] : v[i + w];
      const float keep = up ? v[i + w] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, w);
    }
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 16);
}

// ---- per-thread context of one epilogue step
struct Epi {
  uint8_t* act;      // ACT tile (this CTA)
  uint32_t tl;       // TMEM address of (this thread's lane quadrant, first column cb)
  int trow, cb, r;   // tile row, first column, global row
  int src, dst;      // edge endpoints of row r (0 for node programs / invalid rows)
  bool valid;        // r < M
  const float* sb;   // bias  [cb ..] in shared memory
  const float* sg;   // gamma [cb ..]
  const float* sbt;  // beta  [cb ..]
  float* colsum;     // this (CTA tile, quadrant)'s column-sum partials, vector slot stride cs_vstride
  size_t cs_vstride;
  const int* cs_slot;  // vector -> slot of the partial buffer
  float eps;
  uint64_t* in_full; // [H/64] mbarriers: TMA-loaded input boxes in ACT (Step::in_map)
  uint32_t in_par;   // their phase parity for this step
  uint64_t pol_last; // L2 evict_last policy (in-kernel scratch)
};

// 16 values of this row's TMA-loaded input (ACT, columns c0 .. c0+15), after the box landed
template <bool F16>
// (chunks are consumed in increasing column order: the box's barrier is waited on at the box's
// first chunk, or at this thread's first chunk when it starts inside a box)
__device__ __forceinline__ void in16(const Epi& e, int c0, float* v) {
  if ((c0 & 63) == 0 || c0 == e.cb) mbar_wait(&e.in_full[c0 >> 6], e.in_par);
  lds_tile16<F16>(e.act, e.trow, c0, v);
}

// Column sums of this warp's 32 rows for columns c0 .. c0+15 -> this tile's partial of vector
// `vec` (written once: every (tile, quadrant, column) has exactly one writer, so no
// read-modify-write and no dependence on which CTA runs the tile)
template <int H>
__device__ __forceinline__ void colsum16_add(const Epi& e, int vec, int c0, float* vals) {
  const float cs = warp_colsum16(vals);
  const int lane = lane_id();
  if (lane < 16) e.colsum[(size_t)e.cs_slot[vec] * e.cs_vstride + c0 + lane] = cs;
}

// Row statistics (mean, rstd) of z = acc + b over the H columns of this row, in
// one TMEM pass without the cancellation of E[z^2] - mean^2: each thread sums its
// HC columns shifted by its own first value k (S1 = sum(z - k), S2 = sum(z - k)^2,
// so its partial M2 = S2 - S1^2 / HC loses nothing when |mean| >> sigma), and the
// EW column groups are combined exactly (Chan et al.): mean = avg of the group
// means, M2 = sum_g (M2_g + HC (mean_g - mean)^2); var = M2 / H (biased).
// row_sum combines the groups in a fixed order.
template <int H, int NC, class RowSum>
__device__ __forceinline__ void ln_stats16(const Epi& e, float eps, RowSum row_sum, float& mean, float& rstd) {
  constexpr int HC = NC * 16;          // columns of this thread
  constexpr int EW = H / HC;           // column groups per row
  float s1 = 0.f, s2 = 0.f, k = 0.f;
  uint32_t ta[16];
  tmem_ld16_async(e.tl, ta);
#pragma unroll 1
  for (int cc = 0; cc < NC; ++cc) {
    float b[16];
    lds16(e.sb + cc * 16, b);
    tmem_wait16(ta);
#pragma unroll
    for (int i = 0; i < 16; ++i) b[i] += __uint_as_float(ta[i]);
    if (cc + 1 < NC) tmem_ld16_async(e.tl + (cc + 1) * 16, ta);
    if (cc == 0) k = b[0];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float d = b[i] - k;
      s1 += d;
      s2 = fmaf(d, d, s2);
    }
  }
  const float mg = k + s1 * (1.0f / HC);
  const float m2 = fmaxf(s2 - s1 * s1 * (1.0f / HC), 0.f);
  mean = row_sum(mg) * (1.0f / EW);
  const float dm = mg - mean;
  const float var = row_sum(fmaf((float)HC * dm, dm, m2)) * (1.0f / H);
  rstd = rsqrtf(var + eps);
}

// ================================================================ ops
// Every op receives `wait`, which blocks until the step's accumulator is in TMEM;
// loads that do not depend on it are issued first.

// EPI_SILU: x = acc + b (+ P[src][c] + P[dst][H + c]) -> SiLU -> ACT (+ scratch A, S')
template <int H, int NC, bool F16, bool STZ, class Wait>
__device__ __forceinline__ void op_silu(const Epi& e, const Step& st, Wait wait) {
  const bool gp = (st.flags & EF_GATHER_P) != 0;
  // A leaves by TMA from ACT when st_map is set, else by row stores
  const bool sa = e.valid && (st.flags & EF_STORE_A) != 0 && st.st_map < 0, ss = (st.flags & EF_STORE_S) != 0;
  const __nv_bfloat16* ps = st.gather16 + (size_t)e.src * 2 * H + e.cb;
  const __nv_bfloat16* pd = st.gather16 + (size_t)e.dst * 2 * H + H + e.cb;
  __nv_bfloat16* oa = st.scr_a + (size_t)e.r * H + e.cb;
  __nv_bfloat16* os = st.scr_s + (size_t)e.r * H + e.cb;
  const bool tsrc = gp && st.gsrc_map >= 0;   // P[src] rows arrive in ACT by TMA gather
  const bool rz = STZ && (st.flags & EF_STORE_Z) != 0;   // keep z (16-bit) for the backward (fwd kernels)
  __nv_bfloat16* oz = st.scr_z + (size_t)e.r * H + e.cb;
  uint32_t s0[8], d0[8], s1[8], d1[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) s0[i] = d0[i] = s1[i] = d1[i] = 0u;
  if (gp) {
    if (!tsrc) { ld16(ps, s0); ld16(ps + 16, s1); }
    ld16(pd, d0);
    ld16(pd + 16, d1);
  }
  wait();
  uint32_t ta[16];
  tmem_ld16_async(e.tl, ta);
  auto body = [&](int cc, uint32_t* gs, uint32_t* gd) {
    float x[16];
    lds16(e.sb + cc * 16, x);
    if (gp) {
      if (tsrc) {
        float t[16];
        in16<true>(e, e.cb + cc * 16, t);   // P is stored FP16 in every 16-bit mode (EF_OUT_HALF)
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] += t[i];
      } else {
        add16<true>(gs, x);
      }
      add16<true>(gd, x);
      if (cc + 2 < NC) {
        if (!tsrc) ld16(ps + (cc + 2) * 16, gs);
        ld16(pd + (cc + 2) * 16, gd);
      }
    }
    tmem_wait16(ta);
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] += __uint_as_float(ta[i]);
    if (cc + 1 < NC) tmem_ld16_async(e.tl + (cc + 1) * 16, ta);
    if constexpr (STZ) {
      if (rz) {                         // the SiLU sees exactly the z the backward will reload
        round16<F16>(x);
        if (e.valid) st16<F16>(oz + cc * 16, x);
      }
    }
    if (ss) {
      float dv[16];
      silu_grad16<F16>(x, dv);
      if (e.valid) {                    // S': read again in this kernel -> keep in L2
        uint32_t h[8];
        pack16x16<F16>(dv, h);
        stg256_pol(os + cc * 16, h, e.pol_last);
      }
    } else {
      silu16<F16>(x);
    }
    sts_tile16<F16>(e.act, e.trow, e.cb + cc * 16, x);
    if (sa) st16<F16>(oa + cc * 16, x);
  };
#pragma unroll 1
  for (int cc = 0; cc < NC; cc += 2) {
    body(cc, s0, d0);
    body(cc + 1, s1, d1);
  }
}

// EPI_SILU + EF_FROM_IN: a step without MMA whose z is the forward's 16-bit z_1
// checkpoint, TMA-loaded into ACT (in_map): SiLU (+ SiLU') in place, A / S' out.
// Compiled only into the Z1 variant of the backward kernel.
template <int H, int NC, bool F16, class Wait>
__device__ __forceinline__ void op_silu_in(const Epi& e, const Step& st, Wait wait) {
  const bool sa = e.valid && (st.flags & EF_STORE_A) != 0 && st.st_map < 0, ss = (st.flags & EF_STORE_S) != 0;
  __nv_bfloat16* oa = st.scr_a + (size_t)e.r * H + e.cb;
  __nv_bfloat16* os = st.scr_s + (size_t)e.r * H + e.cb;
  wait();
#pragma unroll 1
  for (int cc = 0; cc < NC; ++cc) {
    float x[16];
    in16<F16>(e, e.cb + cc * 16, x);
    if (ss) {
      float dv[16];
      silu_grad16<F16>(x, dv);
      if (e.valid) {
        uint32_t h[8];
        pack16x16<F16>(dv, h);
        stg256_pol(os + cc * 16, h, e.pol_last);
      }
    } else {
      silu16<F16>(x);
    }
    sts_tile16<F16>(e.act, e.trow, e.cb + cc * 16, x);
    if (sa) st16<F16>(oa + cc * 16, x);
  }
}

// EPI_LN_FWD: y = res + gamma * LN(acc + b) + beta; res = 16-bit res16 rows
// (IN32 = false) or FP32 f_in rows (IN32 = true)
template <int H, int NC, bool F16, bool IN32, class Wait, class RowSum>
__device__ __forceinline__ void op_ln_fwd(const Epi& e, const Step& st, Wait wait, RowSum row_sum) {
  constexpr int W = IN32 ? 16 : 8;
  const bool w32 = e.valid && (st.flags & EF_STORE_F32) != 0;
  const bool w16 = e.valid && (st.flags & EF_STORE_BF) != 0, wact = (st.flags & EF_WRITE_ACT) != 0;
  const bool wlo = e.valid && (st.flags & EF_STORE_LO) != 0;
  __nv_bfloat16* oplo = st.lo_out + (size_t)e.r * H + e.cb;
  const bool has_res = e.valid && !(st.flags & EF_NO_RES);
  const __nv_bfloat16* rp16 = st.res16 + (size_t)e.r * H + e.cb;
  const float* rp32 = st.f_in + (size_t)e.r * st.ld_in + e.cb;
  float* op32 = st.f_out + (size_t)e.r * st.ld_out + e.cb;
  __nv_bfloat16* op16 = st.bf_out + (size_t)e.r * H + e.cb;
  // 16-bit residual rows: two chunks ahead in alternating buffers; FP32 rows: one
  // chunk ahead in a single buffer (q1 unused) to stay within the register budget
  constexpr int AHEAD = IN32 ? 1 : 2;
  uint32_t q0[W], q1[IN32 ? 1 : W];
#pragma unroll
  for (int i = 0; i < W; ++i) q0[i] = 0u;
#pragma unroll
  for (int i = 0; i < (IN32 ? 1 : W); ++i) q1[i] = 0u;
  auto load = [&](int cc, uint32_t* q) {
    if constexpr (IN32) ld32x16(rp32 + cc * 16, q);
    else ld16(rp16 + cc * 16, q);
  };
  const bool tin = !IN32 && st.in_map >= 0;    // residual rows arrive in ACT by TMA
  if (has_res && !tin) { load(0, q0); if (!IN32) load(1, q1); }
  wait();
  float mean, rstd;
  ln_stats16<H, NC>(e, e.eps, row_sum, mean, rstd);
  if ((st.flags & EF_ST_SAVE) && e.valid && e.cb == 0) st.ln_st[e.r] = make_float2(mean, rstd);
  uint32_t ta[16];
  tmem_ld16_async(e.tl, ta);
  auto body = [&](int cc, uint32_t* q) {
    float y[16], res[16];
    if constexpr (IN32) {
#pragma unroll
      for (int i = 0; i < 16; ++i) res[i] = __uint_as_float(q[i]);
    } else {
      if (tin) in16<F16>(e, e.cb + cc * 16, res);   // rows >= M read zero (OOB fill)
      else cvt16<F16>(q, res);
    }
    if (has_res && !tin && cc + AHEAD < NC) load(cc + AHEAD, q);
    lds16(e.sb + cc * 16, y);
    tmem_wait16(ta);
#pragma unroll
    for (int i = 0; i < 16; ++i) y[i] = (y[i] + __uint_as_float(ta[i]) - mean) * rstd;
    if (cc + 1 < NC) tmem_ld16_async(e.tl + (cc + 1) * 16, ta);
    float gm[16];
    lds16(e.sg + cc * 16, gm);
#pragma unroll
    for (int i = 0; i < 16; ++i) y[i] = fmaf(gm[i], y[i], res[i]);
    lds16(e.sbt + cc * 16, gm);
#pragma unroll
    for (int i = 0; i < 16; ++i) y[i] += gm[i];
    if (w32) st32x16(op32 + cc * 16, y);
    if (w16) st16<F16>(op16 + cc * 16, y);
    if (wlo) {                      // y = hi + lo, both 16-bit (hi = the EF_STORE_BF rounding)
      uint32_t hw[8];
      float lo[16];
      pack16x16<F16>(y, hw);
      cvt16<F16>(hw, lo);
#pragma unroll
      for (int i = 0; i < 16; ++i) lo[i] = y[i] - lo[i];
      st16<F16>(oplo + cc * 16, lo);
    }
    if (wact) sts_tile16<F16>(e.act, e.trow, e.cb + cc * 16, y);
  };
#pragma unroll 1
  for (int cc = 0; cc < NC; cc += 2) {
    body(cc, q0);
    body(cc + 1, IN32 ? q0 : q1);
  }
}

// Both LN backward forms rely on dY = 0 on rows >= M (TMA out-of-bounds fill, unloaded
// registers, no G_a gather): every product with dY then vanishes there (x^ is finite: those
// rows' accumulators are finite), so no per-element row mask is needed.
// EPI_LN_BWD, edge form (EF_G16): dY = G_e (rows < valid_in) + G_a[dst], written
// back (16-bit) as G_e'; LayerNorm backward dz = rstd (dY*g - mean(dY*g) - x^ mean(dY*g x^))
// -> ACT + scratch dZ; dgamma (and with EF_COLSUM_ALL dbeta, db) column sums.
// Pass A stashes the rounded dY in ACT at the position pass B overwrites with dz.
template <int H, int NC, bool F16, class Wait, class RowSum, class RowSum2>
__device__ __forceinline__ void op_ln_bwd16(const Epi& e, const Step& st, Wait wait, RowSum row_sum, RowSum2 row_sum2) {
  const bool csall = (st.flags & EF_COLSUM_ALL) != 0;
  const bool has_g = e.valid && e.r < st.valid_in;
  const bool ga = e.valid && !(st.flags & EF_NO_GA);   // G_a[dst] term + G_e' write-back
  __nv_bfloat16* gp16 = st.g16 + (size_t)e.r * H + e.cb;
  const __nv_bfloat16* ap16 = st.ga16 + (size_t)e.dst * H + e.cb;
  __nv_bfloat16* zp = st.scr_z + (size_t)e.r * H + e.cb;
  uint32_t g0[8], g1[8], a0[8], a1[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) g0[i] = g1[i] = a0[i] = a1[i] = 0u;
  const bool tin = st.in_map >= 0;   // G_e rows arrive in ACT by TMA (rows >= valid_in read zero)
  if (has_g && !tin) { ld16(gp16, g0); ld16(gp16 + 16, g1); }
  if (ga) { ld16(ap16, a0); ld16(ap16 + 16, a1); }
  // the forward's statistics (EF_ST_LOAD): issued before the accumulator wait; rows >= M
  // (no forward row) take finite dummies, their dY is 0
  const bool ldst = (st.flags & EF_ST_LOAD) != 0;
  float2 ms = make_float2(0.f, 1.f);
  if (ldst && e.valid) ms = __ldg(st.ln_st + e.r);
  wait();
  float mean = ms.x, rstd = ms.y;
  if (!ldst) ln_stats16<H, NC>(e, e.eps, row_sum, mean, rstd);
  float s1 = 0.f, s2 = 0.f;
  uint32_t ta[16];
  tmem_ld16_async(e.tl, ta);
  auto passA = [&](int cc, uint32_t* gq, uint32_t* aq) {
    const int c0 = e.cb + cc * 16;
    float dy[16], xh[16];
    if (tin) in16<F16>(e, c0, dy);
    else cvt16<F16>(gq, dy);
    if (ga) add16<F16>(aq, dy);
    if (cc + 2 < NC) {
      if (has_g && !tin) ld16(gp16 + (cc + 2) * 16, gq);
      if (ga) ld16(ap16 + (cc + 2) * 16, aq);
    }
    {                                                // dy <- dy as stored (G_e'), packed once
      uint32_t h[8];
      pack16x16<F16>(dy, h);
      cvt16<F16>(h, dy);
      if (ga) stg256(gp16 + cc * 16, h);
      sts_tile16_packed(e.act, e.trow, c0, h);       // stash for pass B
    }
    lds16(e.sb + cc * 16, xh);
    tmem_wait16(ta);
#pragma unroll
    for (int i = 0; i < 16; ++i) xh[i] = (xh[i] + __uint_as_float(ta[i]) - mean) * rstd;
    if (cc + 1 < NC) tmem_ld16_async(e.tl + (cc + 1) * 16, ta);
    float gm[16];
    lds16(e.sg + cc * 16, gm);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float dxh = dy[i] * gm[i];
      s1 += dxh;
      s2 += dxh * xh[i];
      gm[i] = dy[i] * xh[i];                       // dgamma terms (dy = 0 on rows >= M)
    }
    colsum16_add<H>(e, 0, c0, gm);
    if (csall) {
#pragma unroll
      for (int i = 0; i < 16; ++i) xh[i] = dy[i];
      colsum16_add<H>(e, 1, c0, xh);                 // dbeta
    }
  };
#pragma unroll 1
  for (int cc = 0; cc < NC; cc += 2) {
    passA(cc, g0, a0);
    passA(cc + 1, g1, a1);
  }
#if XMGN_ROWSUM2
  row_sum2(s1, s2);                                  // one exchange for both sums (same bits)
  s1 *= (1.0f / H);
  s2 *= (1.0f / H);
#else
  (void)row_sum2;
  s1 = row_sum(s1) * (1.0f / H);
  s2 = row_sum(s2) * (1.0f / H);
#endif
  tmem_ld16_async(e.tl, ta);
#pragma unroll 1
  for (int cc = 0; cc < NC; ++cc) {
    const int c0 = e.cb + cc * 16;
    float dy[16], xh[16];
    lds_tile16<F16>(e.act, e.trow, c0, dy);
    lds16(e.sb + cc * 16, xh);
    tmem_wait16(ta);
#pragma unroll
    for (int i = 0; i < 16; ++i) xh[i] = (xh[i] + __uint_as_float(ta[i]) - mean) * rstd;
    if (cc + 1 < NC) tmem_ld16_async(e.tl + (cc + 1) * 16, ta);
    float gm[16];
    lds16(e.sg + cc * 16, gm);
#pragma unroll
    for (int i = 0; i < 16; ++i) dy[i] = rstd * (dy[i] * gm[i] - s1 - xh[i] * s2);
    sts_tile16<F16>(e.act, e.trow, c0, dy);
    if (e.valid && st.st_map < 0) st16<F16>(zp + cc * 16, dy);
    if (csall) colsum16_add<H>(e, 2, c0, dy);        // db_{m+1}
  }
}

// EPI_LN_BWD, node form: dY = G_h rows (FP32 f_in, rows < valid_in); same math.
template <int H, int NC, bool F16, class Wait, class RowSum, class RowSum2>
__device__ __forceinline__ void op_ln_bwd32(const Epi& e, const Step& st, Wait wait, RowSum row_sum, RowSum2 row_sum2) {
  const bool csall = (st.flags & EF_COLSUM_ALL) != 0;
  const bool has_g = e.valid && e.r < st.valid_in;
  const float* gp32 = st.f_in + (size_t)e.r * st.ld_in + e.cb;
  __nv_bfloat16* zp = st.scr_z + (size_t)e.r * H + e.cb;
  uint32_t g0[16];   // FP32 rows: one chunk ahead (register budget)
#pragma unroll
  for (int i = 0; i < 16; ++i) g0[i] = 0u;
  if (has_g) ld32x16(gp32, g0);
  // the forward's statistics (EF_ST_LOAD): issued before the accumulator wait; rows >= M
  // (no forward row) take finite dummies, their dY is 0
  const bool ldst = (st.flags & EF_ST_LOAD) != 0;
  float2 ms = make_float2(0.f, 1.f);
  if (ldst && e.valid) ms = __ldg(st.ln_st + e.r);
  wait();
  float mean = ms.x, rstd = ms.y;
  if (!ldst) ln_stats16<H, NC>(e, e.eps, row_sum, mean, rstd);
  float s1 = 0.f, s2 = 0.f;
  uint32_t ta[16];
  tmem_ld16_async(e.tl, ta);
  auto passA = [&](int cc, uint32_t* gq) {
    const int c0 = e.cb + cc * 16;
    float dy[16], xh[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) dy[i] = __uint_as_float(gq[i]);
    if (has_g && cc + 1 < NC) ld32x16(gp32 + (cc + 1) * 16, gq);
    lds16(e.sb + cc * 16, xh);
    tmem_wait16(ta);
#pragma unroll
    for (int i = 0; i < 16; ++i) xh[i] = (xh[i] + __uint_as_float(ta[i]) - mean) * rstd;
    if (cc + 1 < NC) tmem_ld16_async(e.tl + (cc + 1) * 16, ta);
    float gm[16];
    lds16(e.sg + cc * 16, gm);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float dxh = dy[i] * gm[i];
      s1 += dxh;
      s2 += dxh * xh[i];
      gm[i] = dy[i] * xh[i];
    }
    colsum16_add<H>(e, 0, c0, gm);
    if (csall) {
#pragma unroll
      for (int i = 0; i < 16; ++i) xh[i] = dy[i];
      colsum16_add<H>(e, 1, c0, xh);
    }
  };
#pragma unroll 1
  for (int cc = 0; cc < NC; cc += 2) {
    passA(cc, g0);
    passA(cc + 1, g0);
  }
#if XMGN_ROWSUM2
  row_sum2(s1, s2);                                  // one exchange for both sums (same bits)
  s1 *= (1.0f / H);
  s2 *= (1.0f / H);
#else
  (void)row_sum2;
  s1 = row_sum(s1) * (1.0f / H);
  s2 = row_sum(s2) * (1.0f / H);
#endif
  if (has_g) ld32x16(gp32, g0);
  tmem_ld16_async(e.tl, ta);
  auto passB = [&](int cc, uint32_t* gq) {
    const int c0 = e.cb + cc * 16;
    float dy[16], xh[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) dy[i] = __uint_as_float(gq[i]);
    if (has_g && cc + 1 < NC) ld32x16(gp32 + (cc + 1) * 16, gq);
    lds16(e.sb + cc * 16, xh);
    tmem_wait16(ta);
#pragma unroll
    for (int i = 0; i < 16; ++i) xh[i] = (xh[i] + __uint_as_float(ta[i]) - mean) * rstd;
    if (cc + 1 < NC) tmem_ld16_async(e.tl + (cc + 1) * 16, ta);
    float gm[16];
    lds16(e.sg + cc * 16, gm);
#pragma unroll
    for (int i = 0; i < 16; ++i) dy[i] = rstd * (dy[i] * gm[i] - s1 - xh[i] * s2);
    sts_tile16<F16>(e.act, e.trow, c0, dy);
    if (e.valid && st.st_map < 0) st16<F16>(zp + cc * 16, dy);
    if (csall) colsum16_add<H>(e, 2, c0, dy);
  };
#pragma unroll 1
  for (int cc = 0; cc < NC; cc += 2) {
    passB(cc, g0);
    passB(cc + 1, g0);
  }
}

// EPI_DSILU: dZ = acc * S' -> ACT + scratch dZ (+ db column sums)
template <int H, int NC, bool F16, class Wait>
__device__ __forceinline__ void op_dsilu(const Epi& e, const Step& st, Wait wait) {
  const bool csall = (st.flags & EF_COLSUM_ALL) != 0;
  const bool noact = (st.flags & EF_NO_ACT) != 0;   // last step of a program: rows out, ACT untouched
  const __nv_bfloat16* sp = st.scr_s + (size_t)e.r * H + e.cb;
  __nv_bfloat16* zp = st.scr_z + (size_t)e.r * H + e.cb;
  uint32_t q0[8], q1[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) q0[i] = q1[i] = 0u;   // invalid rows: S' = 0
  const bool tin = st.in_map >= 0;   // S' rows arrive in ACT by TMA
  if (e.valid && !tin) { ld16(sp, q0); ld16(sp + 16, q1); }
  wait();
  uint32_t ta[16];
  tmem_ld16_async(e.tl, ta);
  auto body = [&](int cc, uint32_t* q) {
    const int c0 = e.cb + cc * 16;
    float x[16];
    if (tin) in16<F16>(e, c0, x);       // rows >= M read zero
    else cvt16<F16>(q, x);
    if (e.valid && !tin && cc + 2 < NC) ld16(sp + (cc + 2) * 16, q);
    tmem_wait16(ta);
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] *= __uint_as_float(ta[i]);
    if (cc + 1 < NC) tmem_ld16_async(e.tl + (cc + 1) * 16, ta);
    if (!noact) sts_tile16<F16>(e.act, e.trow, c0, x);
    if (e.valid && (st.st_map < 0 || noact)) st16<F16>(zp + cc * 16, x);
    if (csall) colsum16_add<H>(e, st.vec0, c0, x);
  };
#pragma unroll 1
  for (int cc = 0; cc < NC; cc += 2) {
    body(cc, q0);
    body(cc + 1, q1);
  }
  if (e.valid && (st.flags & EF_DISCARD)) {   // last read of S' (consumed above): drop its lines
#pragma unroll
    for (int i = 0; i < NC * 16 * 2 / 128; ++i) discard_l2_line(reinterpret_cast<const uint8_t*>(sp) + 128 * i);
  }
}

// EPI_STORE: out[:, col0 + c] = acc (16-bit bf_out with EF_OUT16, else FP32 f_out)
template <int H, int NC, bool F16, class Wait>
__device__ __forceinline__ void op_store(const Epi& e, const Step& st, Wait wait) {
  const bool o16 = (st.flags & EF_OUT16) != 0, oh = o16 && (st.flags & EF_OUT_HALF) != 0;
  __nv_bfloat16* op16 = st.bf_out + (size_t)e.r * st.ld_out + st.col0 + e.cb;
  float* op32 = st.f_out + (size_t)e.r * st.ld_out + st.col0 + e.cb;
  wait();
  uint32_t ta[16];
  tmem_ld16_async(e.tl, ta);
#pragma unroll 1
  for (int cc = 0; cc < NC; ++cc) {
    tmem_wait16(ta);
    float x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = __uint_as_float(ta[i]);
    if (cc + 1 < NC) tmem_ld16_async(e.tl + (cc + 1) * 16, ta);
    if (e.valid) {
      if (oh) st16<true>(op16 + cc * 16, x);
      else if (o16) st16<F16>(op16 + cc * 16, x);
      else st32x16(op32 + cc * 16, x);
    }
  }
}

// EPI_ADD, edge form (EF_G16): g16_out = g16 + acc (16-bit gradient stream)
template <int H, int NC, bool F16, class Wait>
__device__ __forceinline__ void op_add16(const Epi& e, const Step& st, Wait wait) {
  const __nv_bfloat16* ip = st.g16 + (size_t)e.r * H + e.cb;
  __nv_bfloat16* op = st.g16_out + (size_t)e.r * H + e.cb;
  uint32_t q0[8], q1[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) q0[i] = q1[i] = 0u;
  const bool tin = st.in_map >= 0;   // G_e' rows arrive in ACT by TMA
  if (e.valid && !tin) { ld16(ip, q0); ld16(ip + 16, q1); }
  wait();
  uint32_t ta[16];
  tmem_ld16_async(e.tl, ta);
  auto body = [&](int cc, uint32_t* q) {
    float x[16];
    if (tin) in16<F16>(e, e.cb + cc * 16, x);
    else cvt16<F16>(q, x);
    if (e.valid && !tin && cc + 2 < NC) ld16(ip + (cc + 2) * 16, q);
    tmem_wait16(ta);
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] += __uint_as_float(ta[i]);
    if (cc + 1 < NC) tmem_ld16_async(e.tl + (cc + 1) * 16, ta);
    if (e.valid) st16<F16>(op + cc * 16, x);
  };
#pragma unroll 1
  for (int cc = 0; cc < NC; cc += 2) {
    body(cc, q0);
    body(cc + 1, q1);
  }
}

// EPI_ADD, node form: f_out = (rows < valid_in ? f_in : 0) (+ gather[dst] with EF_GATHER_G) + acc (FP32)
template <int H, int NC, bool F16, class Wait>
__device__ __forceinline__ void op_add32(const Epi& e, const Step& st, Wait wait) {
  const bool has_in = e.valid && e.r < st.valid_in, gg = e.valid && (st.flags & EF_GATHER_G) != 0;
  const float* ip = st.f_in + (size_t)e.r * st.ld_in + e.cb;
  const float* gp = st.gather + (size_t)e.dst * H + e.cb;
  float* op = st.f_out + (size_t)e.r * st.ld_out + e.cb;
  uint32_t q0[16], q1[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) q0[i] = q1[i] = 0u;
  if (has_in) { ld32x16(ip, q0); ld32x16(ip + 16, q1); }
  wait();
  uint32_t ta[16];
  tmem_ld16_async(e.tl, ta);
  auto body = [&](int cc, uint32_t* q) {
    float x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = __uint_as_float(q[i]);
    if (has_in && cc + 2 < NC) ld32x16(ip + (cc + 2) * 16, q);
    if (gg) {
      uint32_t t[16];
      ld32x16(gp + cc * 16, t);
#pragma unroll
      for (int i = 0; i < 16; ++i) x[i] += __uint_as_float(t[i]);
    }
    tmem_wait16(ta);
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] += __uint_as_float(ta[i]);
    if (cc + 1 < NC) tmem_ld16_async(e.tl + (cc + 1) * 16, ta);
    if (e.valid) st32x16(op + cc * 16, x);
  };
#pragma unroll 1
  for (int cc = 0; cc < NC; cc += 2) {
    body(cc, q0);
    body(cc + 1, q1);
  }
}

}  // namespace xmgn
